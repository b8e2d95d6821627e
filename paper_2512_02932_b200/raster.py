"""Forward rendering API -- drop-in for the reference's ``hybridsplat.raster``
(raster/render.py:83-118, raster/project.py:34-90).

``render(scene, camera, settings)`` runs the whole hot path on the B200 through
libhgs.so: float64 preprocess, onesweep depth sort, tile binning, and the
per-tile compositor.  It accepts the reference-style host ``GaussianSet``
(float64 numpy; outputs come back as float64 numpy, like the reference) or a
device-resident ``DeviceGaussians`` (float32 CUDA tensors; outputs stay on the
GPU as torch tensors).  There is no CPU backend.
"""

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .core import CameraView, DeviceGaussians, GaussianSet
from .errors import ConfigError, DegenerateIntersection, IntegrityError
from .settings import (ALPHA_CLAMP, EARLY_STOP_T, LOWPASS_SIGMA, MIN_ALPHA, SCREEN_DILATION,
                       TILE_SIZE, RenderSettings)

HAVE_EXT = _lib.available()

# raster/__init__.py:12-19 of the reference, in the same order
__all__ = ["ALPHA_CLAMP", "DegenerateIntersection", "EARLY_STOP_T", "LOWPASS_SIGMA",
           "MIN_ALPHA", "ProjectedSplat", "RenderSettings", "SCREEN_DILATION",
           "SplatFrame", "build_frame", "evaluate_contribution",
           "project_gaussian_3d", "ray_splat_intersect",
           "HAVE_EXT", "BlendLog", "RenderOutput", "active_backend", "render",
           "render_naive", "scene_fingerprint"]

TILE_SIZES = (8, 16, 32, 64)  # RenderSettings.tile_size values SplatFrame can export
_OVERLAP = os.environ.get("HGS_OVERLAP", "1") != "0"  # A/B switch of the preprocess side stream


def active_backend(settings: RenderSettings):
    """Backend selection (raster/render.py:20-27).  Only the sm_100a kernels
    exist here; the reference's CPU backends are rejected rather than
    silently substituted."""
    b = settings.backend
    if b in ("auto", "cuda"):
        _lib.lib()
        return "cuda"
    if b in ("cython", "python"):
        raise ConfigError("backend %r is a CPU backend of the reference; this package only "
                          "provides the sm_100a CUDA rasterizer" % b)
    raise ConfigError("backend must be auto or cuda")


def scene_fingerprint(scene):
    """Identity of the scene a RenderOutput was produced from
    (raster/render.py:67-70).  Host scenes use the reference's sums; device
    scenes use tensor version counters (no device sync)."""
    if isinstance(scene, DeviceGaussians):
        return ("device", scene.count) + scene.versions()
    # deterministic block sums on all host cores (numpy's sums are
    # single-threaded: 5 ms at 1M); render takes the same sums during the
    # scene's upload (DeviceGaussians.from_host(fingerprint=True))
    from ._hostio import fingerprint_sum
    return (scene.count,) + tuple(fingerprint_sum(a) for a in (scene.center, scene.opacity_logit, scene.log_scale))


@dataclass
class ProjectedSplat:
    """raster/project.py:48-57"""
    gaussian_index: int
    type_spec: int
    screen_center: np.ndarray
    depth_key: float
    radius: float
    conic: Optional[np.ndarray] = None
    plane_params: Optional[np.ndarray] = None


@dataclass
class BlendLog:
    """Per-pixel ordered record of every composited contribution
    (raster/render.py:30-51); materialised on demand from the GPU frame."""
    offsets: np.ndarray
    position: np.ndarray
    gaussian_index: np.ndarray
    alpha: np.ndarray
    u: np.ndarray
    v: np.ndarray

    def entries(self, ix, iy, width):
        lo = self.offsets[iy * width + ix]
        hi = self.offsets[iy * width + ix + 1]
        return [(int(self.gaussian_index[e]), float(self.alpha[e]),
                 (float(self.u[e]), float(self.v[e]))) for e in range(lo, hi)]


_FRAME_FIELDS = ("idx", "typ", "depth", "center2d", "cov2d", "conic", "mrow", "alpha_eff",
                 "color", "radius", "normal", "bbox", "tile_offsets", "tile_ids", "pixel_count",
                 "t_cam", "alpha", "view_dir", "cam_dist")
# per-splat (length m) fields; "valid" is all True after build_frame's cull
_PER_SPLAT = ("idx", "typ", "depth", "center2d", "cov2d", "conic", "mrow", "alpha_eff", "color",
              "radius", "normal", "bbox", "t_cam", "alpha", "view_dir", "cam_dist")


class SplatFrame:
    """The device frame of one render: sorted splat records, tile lists and
    per-pixel replay state, living in one caller-owned CUDA buffer.  The
    reference's SplatFrame arrays (raster/project.py:60-90) are exported on
    first access (float64, exactly the values the binning used)."""

    def __init__(self, scene, camera, settings, buf, info, flags):
        self.scene = scene
        self.camera = camera
        self.settings = settings
        self.buf = buf
        self.info = info
        self.flags = flags
        self.height = camera.height
        self.width = camera.width
        self.tile_size = settings.tile_size
        self._host = None

    @property
    def count(self):
        self.sync()
        return int(self.info.m)

    @property
    def pair_count(self):
        """Tile/splat pairs of the compositor's 16 x 16 tile lists (the
        reference's bbox lists, ``len(tile_ids)``, also keep the pairs whose
        support cannot reach the tile)."""
        self.sync()
        return int(self.info.k)

    @property
    def pending(self):
        """True for a frame rendered with async=True whose counts are still
        on the device."""
        return self.info.m < 0

    def sync(self):
        """Read M, K and the status of an asynchronous frame (one stream
        synchronisation); raises the status as the reference exception
        (ConfigError for an exhausted pair capacity)."""
        if self.info.m >= 0:
            return self
        rc = _lib.lib().hgs_frame_sync_info(_lib.ptr(self.buf), self.info,
                                            _lib.current_stream_handle(self.buf.device))
        if rc == _lib.HGS_ERR_PAIR_CAPACITY:
            key = (self.info.n, self.width, self.height)
            _pair_hint[key] = max(_pair_hint.get(key, 0), int(self.info.k * 1.25) + 1024)
            raise ConfigError("frame pair capacity exceeded (K = %d); render again" % self.info.k)
        _lib.check(rc, "hgs_forward")
        return self

    def export(self):
        """Dict of float64 / int numpy arrays (reference SplatFrame fields)."""
        if self._host is not None:
            return self._host
        import torch
        m, k = self.count, self.pair_count
        dev = self.buf.device
        W, H = self.width, self.height
        d = dict(
            idx=torch.empty(max(m, 1), dtype=torch.int32, device=dev),
            typ=torch.empty(max(m, 1), dtype=torch.uint8, device=dev),
            depth=torch.empty(max(m, 1), dtype=torch.float64, device=dev),
            center2d=torch.empty((max(m, 1), 2), dtype=torch.float64, device=dev),
            cov2d=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            conic=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            mrow=torch.empty((max(m, 1), 3, 4), dtype=torch.float64, device=dev),
            alpha_eff=torch.empty(max(m, 1), dtype=torch.float64, device=dev),
            color=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            radius=torch.empty(max(m, 1), dtype=torch.float64, device=dev),
            normal=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            bbox=torch.empty((max(m, 1), 4), dtype=torch.int32, device=dev),
            tile_offsets=torch.empty(int(self.info.n_tiles) + 1, dtype=torch.int64, device=dev),
            tile_ids=torch.empty(max(k, 1), dtype=torch.int32, device=dev),
            pixel_count=torch.empty((H, W), dtype=torch.int32, device=dev),
            t_cam=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            alpha=torch.empty(max(m, 1), dtype=torch.float64, device=dev),
            view_dir=torch.empty((max(m, 1), 3), dtype=torch.float64, device=dev),
            cam_dist=torch.empty(max(m, 1), dtype=torch.float64, device=dev),
        )
        if self.flags & _lib.HGS_FLAG_FRAME_ONLY:
            d["pixel_count"] = None  # nothing was composited
        ex = _lib.FrameExport(*(_lib.ptr(d[f]) for f in _FRAME_FIELDS))
        ds = self.scene
        sc = _lib.scene_struct(ds)
        _lib.check(_lib.lib().hgs_frame_export_arrays(
            sc, _lib.camera_struct(self.camera), _lib.settings_struct(self.settings, self.flags),
            _lib.ptr(self.buf), self.info, ex, _lib.current_stream_handle(dev)), "frame export")
        if not (self.flags & _lib.HGS_FLAG_NAIVE):
            # the reference's lists (bbox-based, project.py:329-357) at the
            # settings' tile size; the compositor's own 16 x 16 lists drop the
            # tiles its support cannot reach (hgs_frame_tile_bins)
            d["tile_offsets"], d["tile_ids"] = self._rebin(self.tile_size)
            k = int(d["tile_ids"].shape[0])
        out = {f: (t.cpu().numpy() if t is not None else None) for f, t in d.items()}
        for f in _PER_SPLAT:
            out[f] = out[f][:m]
        out["tile_ids"] = out["tile_ids"][:k]
        out["valid"] = np.ones(m, dtype=bool)
        self._host = out
        return out

    def _rebin(self, tile):
        """Tile lists at another tile size (project.py:329-357) on the GPU."""
        import torch
        L = _lib.lib()
        dev = self.buf.device
        stream = _lib.current_stream_handle(dev)
        W, H = self.width, self.height
        n_tiles = ((W + tile - 1) // tile) * ((H + tile - 1) // tile)
        offsets = torch.empty(n_tiles + 1, dtype=torch.int64, device=dev)
        # the compositor's lists are culled: the bbox lists are longer (~1.5x)
        cap = max(2 * self.pair_count * max(16 // tile, 1) ** 2 + self.count, 1)
        for _ in range(2):
            nb = L.hgs_tile_bins_scratch_bytes(self.count, W, H, tile, cap)
            scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
            ids = torch.empty(cap, dtype=torch.int32, device=dev)
            k = _lib._i64(0)
            rc = L.hgs_frame_tile_bins(_lib.ptr(self.buf), self.info, tile, _lib.ptr(offsets),
                                       _lib.ptr(ids), cap, _lib.ptr(scratch), nb, ctypes.byref(k),
                                       stream)
            if rc == _lib.HGS_ERR_PAIR_CAPACITY:
                cap = int(k.value)
                continue
            _lib.check(rc, "hgs_frame_tile_bins")
            return offsets, ids[:int(k.value)]
        raise ConfigError("could not size the tile-bin buffer")

    def __getattr__(self, name):
        if name in _FRAME_FIELDS or name == "valid":
            return self.export()[name]
        raise AttributeError(name)

    def splat(self, k):
        f = self.export()
        typ = int(f["typ"][k])
        c = f["conic"][k]
        return ProjectedSplat(
            gaussian_index=int(f["idx"][k]), type_spec=typ, screen_center=f["center2d"][k].copy(),
            depth_key=float(f["depth"][k]), radius=float(f["radius"][k]),
            conic=np.array([[c[0], c[1]], [c[1], c[2]]]) if typ == 1 else None,
            plane_params=f["mrow"][k].copy() if typ == 0 else None)


class RenderOutput:
    """raster/render.py:54-65.  ``color``/``depth``/``transmittance`` are numpy
    float64 for host scenes and float32 CUDA tensors for device scenes;
    ``alpha`` (1 - T) and ``normal`` are the extension images (for host
    scenes they are downloaded on first access: the reference has no such
    outputs, so a drop-in caller never pays for them)."""

    def __init__(self, color, depth, transmittance, alpha, normal, frame, fingerprint,
                 host_scene=None, lazy=None):
        self.color = color
        self.depth = depth
        self.transmittance = transmittance
        self._alpha = alpha
        self._normal = normal
        self._lazy = lazy or {}  # name -> device tensor still to download
        self.frame = frame
        self.scene_fingerprint = fingerprint
        self._host_scene = host_scene
        self._log = None

    def _extension(self, name):
        t = self._lazy.pop(name, None)
        if t is not None:
            from ._hostio import download
            setattr(self, "_" + name, download([t], tag="ext")[0])
        return getattr(self, "_" + name)

    @property
    def alpha(self):
        return self._extension("alpha")

    @alpha.setter
    def alpha(self, v):
        self._lazy.pop("alpha", None)
        self._alpha = v

    @property
    def normal(self):
        return self._extension("normal")

    @normal.setter
    def normal(self, v):
        self._lazy.pop("normal", None)
        self._normal = v

    def check_scene(self, scene):
        if scene_fingerprint(scene) != self.scene_fingerprint:
            raise IntegrityError("blend log does not match this scene")

    @property
    def blend_log(self):
        if self._log is None:
            self._log = _materialise_log(self.frame)
        return self._log


def _materialise_log(frame):
    import torch
    fx = frame.export()
    counts = fx["pixel_count"].reshape(-1).astype(np.int64)
    offsets = np.zeros(counts.size + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    tot = int(offsets[-1])
    dev = frame.buf.device
    d_off = torch.from_numpy(offsets).to(dev)
    pos = torch.empty(max(tot, 1), dtype=torch.int32, device=dev)
    al = torch.empty(max(tot, 1), dtype=torch.float32, device=dev)
    u = torch.empty_like(al)
    v = torch.empty_like(al)
    _lib.check(_lib.lib().hgs_blend_log(
        _lib.scene_struct(frame.scene), _lib.camera_struct(frame.camera),
        _lib.settings_struct(frame.settings, frame.flags), _lib.ptr(frame.buf), frame.info,
        _lib.ptr(d_off), _lib.ptr(pos), _lib.ptr(al), _lib.ptr(u), _lib.ptr(v),
        _lib.current_stream_handle(dev)), "blend log")
    pos = pos.cpu().numpy()[:tot]
    idx = fx["idx"]
    return BlendLog(offsets, pos, idx[pos] if tot else pos,
                    al.double().cpu().numpy()[:tot], u.double().cpu().numpy()[:tot],
                    v.double().cpu().numpy()[:tot])


# pair-capacity hints per (n, W, H): K of the last frame, so steady-state
# frames allocate once and never retry.
_pair_hint = {}


def _check_camera(camera):
    if not isinstance(camera, CameraView):
        for a in ("fx", "fy", "cx", "cy", "width", "height", "world_to_camera"):
            if not hasattr(camera, a):
                raise ConfigError("camera lacks %s" % a)
    if int(camera.width) > 65535 or int(camera.height) > 65535:
        raise ConfigError("image dimensions above 65535 are not supported")


def rasterize(ds, camera, settings, flags=0, outputs=None, events=None, async_=False, frame_buf=None,
              overlap=None):
    """Device-level forward: DeviceGaussians -> (images dict, SplatFrame).

    ``outputs`` may pass preallocated image tensors (keys color, depth,
    transmittance, alpha, normal) to avoid per-frame allocation; ``events``
    (5 torch.cuda.Event) are recorded at the library's stage boundaries.
    ``async_=True``: no host round trip at all (HGS_FLAG_ASYNC; capturable in
    a CUDA graph); the frame's counts and status are read by
    ``SplatFrame.sync()`` (a backward can run before that).  ``frame_buf``:
    a preallocated uint8 CUDA buffer to render into (its size sets the pair
    capacity).  ``overlap``: run the float64 preprocess on a side stream
    beside the depth sort (hgs_settings.aux_stream)."""
    import torch
    L = _lib.lib()
    _check_camera(camera)
    if settings.tile_size not in TILE_SIZES:
        raise ConfigError("tile_size must be one of %s (the compositor bins at %d; SplatFrame "
                          "re-bins its tile lists at the requested size)" % (TILE_SIZES, TILE_SIZE))
    dev = ds.device
    W, H = int(camera.width), int(camera.height)
    n = ds.count
    if outputs is None and flags & _lib.HGS_FLAG_FRAME_ONLY:
        outputs = {}
    if outputs is None:
        outputs = dict(
            color=torch.empty((H, W, 3), dtype=torch.float32, device=dev),
            depth=torch.empty((H, W), dtype=torch.float32, device=dev),
            transmittance=torch.empty((H, W), dtype=torch.float32, device=dev),
            alpha=torch.empty((H, W), dtype=torch.float32, device=dev),
            normal=torch.empty((H, W, 3), dtype=torch.float32, device=dev))
    _check_outputs(outputs, H, W, dev)
    imgs = _lib.Images(*(_lib.ptr(outputs.get(k)) for k in
                         ("color", "depth", "transmittance", "alpha", "normal")))
    if flags & _lib.HGS_FLAG_FRAME_ONLY:
        imgs = _lib.Images(None, None, None, None, None)
    if async_:
        flags |= _lib.HGS_FLAG_ASYNC
    if overlap is None:
        overlap = _OVERLAP
    sc = _lib.scene_struct(ds)
    cam = _lib.camera_struct(camera)
    # the float64 preprocess runs on a side stream beside the depth sort
    st = _lib.settings_struct(settings, flags, events, aux=_lib.aux_handles(dev) if overlap else None)
    stream = _lib.current_stream_handle(dev)
    key = (n, W, H)
    if async_:
        if frame_buf is None:
            frame_buf = torch.empty(frame_bytes(n, W, H), dtype=torch.uint8, device=dev)
        info = _lib.FrameInfo()
        _lib.check(L.hgs_forward(sc, cam, st, _lib.ptr(frame_buf), frame_buf.numel(), imgs, info, stream),
                   "hgs_forward")
        return outputs, SplatFrame(ds, camera, settings, frame_buf, info, flags)
    cap = _pair_hint.get(key, max(8 * n, 1 << 16))
    for _ in range(3):
        nbytes = L.hgs_frame_bytes(n, W, H, TILE_SIZE, cap)
        if frame_buf is not None and frame_buf.numel() >= nbytes:
            buf = frame_buf
            nbytes = frame_buf.numel()
        else:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        info = _lib.FrameInfo()
        rc = L.hgs_forward(sc, cam, st, _lib.ptr(buf), nbytes, imgs, info, stream)
        if rc == _lib.HGS_ERR_PAIR_CAPACITY:
            cap = int(info.k * 1.25) + 1024
            _pair_hint[key] = cap
            continue
        _lib.check(rc, "hgs_forward")
        if info.k > cap * 0.9 or key not in _pair_hint:
            _pair_hint[key] = max(cap, int(info.k * 1.25) + 1024)
        return outputs, SplatFrame(ds, camera, settings, buf, info, flags)
    raise ConfigError("could not size the pair buffer")


_OUT_SHAPES = {"color": 3, "depth": 0, "transmittance": 0, "alpha": 0, "normal": 3}


def _check_outputs(outputs, H, W, dev):
    """Caller-provided image buffers are written through raw pointers: each
    must be a contiguous float32 tensor of this camera's shape on the scene's
    device (a buffer sized for another camera would be overrun)."""
    import torch
    for k, t in outputs.items():
        if t is None:
            continue
        if k not in _OUT_SHAPES:
            raise ConfigError("unknown output image %r" % (k,))
        want = (H, W, 3) if _OUT_SHAPES[k] else (H, W)
        if (not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or tuple(t.shape) != want
                or t.device != dev or not t.is_contiguous()):
            raise ConfigError("output %r must be a contiguous float32 %s tensor on %s" % (k, want, dev))


def frame_bytes(n, width, height, pairs=None):
    """Bytes of a frame buffer for n Gaussians at width x height with room for
    ``pairs`` tile/splat pairs (default: the capacity the last frame of this
    size needed, with 25% headroom)."""
    cap = pairs if pairs is not None else _pair_hint.get((n, width, height), max(8 * n, 1 << 16))
    return int(_lib.lib().hgs_frame_bytes(n, width, height, TILE_SIZE, cap))


def _flags(settings, naive=False, fast=False):
    active_backend(settings)
    f = 0
    if naive:
        f |= _lib.HGS_FLAG_NAIVE
    if fast:
        f |= _lib.HGS_FLAG_FAST
    return f


def _render(scene, camera, settings, naive, fast):
    if settings is None:
        settings = RenderSettings()
    flags = _flags(settings, naive, fast)
    if isinstance(scene, DeviceGaussians):
        imgs, frame = rasterize(scene, camera, settings, flags)
        return RenderOutput(imgs["color"], imgs["depth"], imgs["transmittance"], imgs["alpha"],
                            imgs["normal"], frame, scene_fingerprint(scene))
    if not isinstance(scene, GaussianSet):
        scene = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                            scene.sh_coeffs, scene.type_spec)
    ds = DeviceGaussians.from_host(scene, fingerprint=True)
    imgs, frame = rasterize(ds, camera, settings, flags)
    from ._hostio import download
    keys = ("color", "depth", "transmittance")
    host = dict(zip(keys, download([imgs[k] for k in keys], tag="images")))
    return RenderOutput(host["color"], host["depth"], host["transmittance"], None, None, frame,
                        ds.host_fingerprint, host_scene=scene,
                        lazy={"alpha": imgs["alpha"], "normal": imgs["normal"]})


def render(scene, camera, settings: RenderSettings = None, *, fast=False) -> RenderOutput:
    """Rasterize the scene for one view in a single alpha-blending pass
    (raster/render.py:83-98).  ``fast=True`` skips the float64 re-evaluation
    of near-threshold decisions (HGS_FLAG_FAST)."""
    return _render(scene, camera, settings, False, fast)


def render_naive(scene, camera, settings: RenderSettings = None) -> RenderOutput:
    """All-pairs compositor without tiles or bounding boxes, on the GPU
    (raster/render.py:101-118) -- the oracle the tile renderer is checked
    against."""
    return _render(scene, camera, settings, True, False)


def build_frame(scene, camera, settings: RenderSettings = None) -> SplatFrame:
    """Screen-space preparation only -- depth sort, float64 preprocess, bounds
    and tile bins, on the GPU, no compositing (raster/project.py:360-379).
    The returned frame exports the reference's SplatFrame arrays; it cannot
    be back-propagated (nothing was blended)."""
    if settings is None:
        settings = RenderSettings()
    flags = _flags(settings) | _lib.HGS_FLAG_FRAME_ONLY
    if isinstance(scene, DeviceGaussians):
        return rasterize(scene, camera, settings, flags)[1]
    if not isinstance(scene, GaussianSet):
        scene = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                            scene.sh_coeffs, scene.type_spec)
    return rasterize(DeviceGaussians.from_host(scene), camera, settings, flags)[1]


def _eval_pairs(splats, pixels, opacities):
    """hgs_eval_contributions over a list of ProjectedSplat / pixel / opacity
    triples -> (alpha, u, v, degenerate) numpy arrays."""
    import torch
    n = len(splats)
    typ = np.array([s.type_spec for s in splats], np.uint8)
    c2 = np.array([s.screen_center for s in splats], np.float64).reshape(n, 2)
    conic = np.zeros((n, 3))
    mrow = np.zeros((n, 12))
    for i, s in enumerate(splats):
        if s.type_spec == 1:
            c = np.asarray(s.conic, np.float64)
            conic[i] = (c[0, 0], c[0, 1], c[1, 1])
        else:
            mrow[i] = np.asarray(s.plane_params, np.float64).reshape(12)
    px = np.array(pixels, np.float64).reshape(n, 2)
    op = np.array(opacities, np.float64).reshape(n)
    dev = torch.device("cuda", torch.cuda.current_device())
    d = [torch.from_numpy(a).to(dev) for a in (typ, c2, conic, mrow, op, px)]
    alpha = torch.empty(n, dtype=torch.float64, device=dev)
    u = torch.empty_like(alpha)
    v = torch.empty_like(alpha)
    fl = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().hgs_eval_contributions(
        n, *(_lib.ptr(t) for t in d), _lib.ptr(alpha), _lib.ptr(u), _lib.ptr(v), _lib.ptr(fl),
        _lib.current_stream_handle(dev)), "hgs_eval_contributions")
    return (alpha.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy(), fl.cpu().numpy() != 0)


def ray_splat_intersect(splat: ProjectedSplat, pixel):
    """Tangent-frame coordinates (u, v) where the ray through ``pixel`` meets
    the plane of a flat splat (raster/project.py:109-126), evaluated on the
    GPU in float64; raises DegenerateIntersection when |den| < 1e-9."""
    if splat.plane_params is None:
        raise ConfigError("ray_splat_intersect needs a flat primitive")
    _, u, v, deg = _eval_pairs([splat], [(float(pixel[0]), float(pixel[1]))], [1.0])
    if deg[0]:
        raise DegenerateIntersection("pixel ray nearly parallel to splat plane")
    return float(u[0]), float(v[0])


def evaluate_contribution(splat: ProjectedSplat, pixel, opacity):
    """alpha_t = opacity * exp(-d/2) clamped to <= 0.99, d the conic distance
    (3D) or min(ray/splat, low-pass) distance (2D); 0 for a degenerate
    intersection (raster/project.py:129-152).  Evaluated on the GPU in
    float64, with the formulas of the compositors' float64 re-checks."""
    if splat.type_spec == 0 and splat.plane_params is None:
        raise ConfigError("flat splat without plane parameters")
    a, _, _, _ = _eval_pairs([splat], [(float(pixel[0]), float(pixel[1]))], [float(opacity)])
    return float(a[0])


def project_gaussian_3d(g, camera: CameraView, settings: RenderSettings = None):
    """Affine-project one volumetric primitive (raster/project.py:155-166);
    None when culled."""
    if settings is None:
        settings = RenderSettings()
    if g.type_spec != 1:
        raise ConfigError("project_gaussian_3d needs a volumetric primitive")
    scene = GaussianSet(np.asarray(g.center)[None], np.asarray(g.log_scale)[None],
                        np.asarray(g.rotation)[None], np.array([g.opacity_logit]),
                        np.asarray(g.sh_coeffs)[None], np.array([1], np.uint8))
    frame = build_frame(scene, camera, settings)
    return frame.splat(0) if frame.count else None
