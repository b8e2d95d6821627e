"""CPU oracle for the hybrid 2D/3D Gaussian rasterizer hot path.

TEST INFRASTRUCTURE ONLY.  This package is the parity checker for the CUDA
product path in ``paper_2512_02932_b200``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package never does.

It wraps ``hgs_oracle.c``: a float64 restatement of the reference package
``hybridsplat`` (``/root/reference/pkg/src/hybridsplat``):

* ``build_frame``      -- raster/project.py:360-379 (project_scene + cull +
  _bboxes + _tile_bins)
* ``render``           -- raster/render.py:83-98 / _blend_py.forward_blend
  (raster/_blend_py.py:55-123); ``naive=True`` is render_naive
  (render.py:101-118)
* ``blend_log``        -- BlendLog (render.py:30-51)
* ``backward``         -- grad/backward.py:37-181 with the
  _blend_py.backward_blend replay (raster/_blend_py.py:126-242)
* ``exchange_pass``    -- exchange.py:137-155

Parity of the restatement is pinned against fixtures produced by running the
reference itself (tests/golden/make_golden.py -> tests/golden/*.npz).  The
normal / alpha images and depth / normal / alpha upstream gradients are an
extension with no reference counterpart ("parity unpinned"; FD-checked).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhgs_oracle.so")

ACC_STRIDE = 25
ACC_COLOR, ACC_ALPHA, ACC_CTR, ACC_COV, ACC_MROW, ACC_Z, ACC_N = 0, 3, 4, 6, 9, 21, 22

FIELDS = {  # orc_frame_copy ids: name -> (id, dtype, per-splat shape); None = special
    "idx": (0, np.int32, ()), "typ": (1, np.uint8, ()), "depth": (2, np.float64, ()),
    "t_cam": (3, np.float64, (3,)), "center2d": (4, np.float64, (2,)),
    "cov2d": (5, np.float64, (3,)), "conic": (6, np.float64, (3,)),
    "mrow": (7, np.float64, (3, 4)), "alpha": (8, np.float64, ()),
    "alpha_eff": (9, np.float64, ()), "color": (10, np.float64, (3,)),
    "view_dir": (11, np.float64, (3,)), "cam_dist": (12, np.float64, ()),
    "bbox": (13, np.int32, (4,)), "radius": (14, np.float64, ()),
    "normal": (17, np.float64, (3,)),
}


class OracleError(RuntimeError):
    pass


class _Scene(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_bases", ctypes.c_int32),
                ("center", ctypes.c_void_p), ("log_scale", ctypes.c_void_p),
                ("rotation", ctypes.c_void_p), ("opacity_logit", ctypes.c_void_p),
                ("sh", ctypes.c_void_p), ("type_spec", ctypes.c_void_p)]


class _Camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("w2c", ctypes.c_double * 16), ("near_plane", ctypes.c_double),
                ("far_plane", ctypes.c_double)]


class _Settings(ctypes.Structure):
    _fields_ = [("background", ctypes.c_double * 3), ("tile_size", ctypes.c_int32),
                ("theta_z", ctypes.c_double), ("t_z", ctypes.c_double),
                ("lambda_z", ctypes.c_double)]


_lib = None


def build():
    """Compile libhgs_oracle.so with the committed Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_build_frame.restype = vp
        L.orc_build_frame.argtypes = [vp, vp, vp, ctypes.POINTER(ctypes.c_int)]
        L.orc_free_frame.argtypes = [vp]
        L.orc_frame_sizes.argtypes = [vp, vp]
        L.orc_frame_copy.argtypes = [vp, i32, vp]
        L.orc_forward.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp]
        L.orc_blend_log.argtypes = [vp, i32, vp, vp, vp, vp, vp]
        L.orc_backward_blend.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.orc_chain_rule.argtypes = [vp, vp, vp, vp, i32, vp, vp]
        L.orc_exchange.argtypes = [i64, vp, vp, vp, dp, vp, vp, vp]
        L.orc_num_threads.restype = i32
        L.orc_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def num_threads():
    return lib().orc_num_threads()


def set_num_threads(n):
    lib().orc_set_num_threads(int(n))


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class _Bound:
    """Keeps the float64 copies alive while C holds pointers into them."""

    def __init__(self, scene, camera, settings):
        self.center = np.ascontiguousarray(scene.center, np.float64)
        self.log_scale = np.ascontiguousarray(scene.log_scale, np.float64)
        self.rotation = np.ascontiguousarray(scene.rotation, np.float64)
        self.opacity_logit = np.ascontiguousarray(scene.opacity_logit, np.float64)
        self.sh = np.ascontiguousarray(scene.sh_coeffs, np.float64)
        self.type_spec = np.ascontiguousarray(scene.type_spec, np.uint8)
        n = self.center.shape[0]
        self.n = n
        self.B = self.sh.shape[2] if self.sh.ndim == 3 else 1
        self.sc = _Scene(n, self.B, _p(self.center).value, _p(self.log_scale).value,
                         _p(self.rotation).value, _p(self.opacity_logit).value,
                         _p(self.sh).value, _p(self.type_spec).value)
        w2c = np.ascontiguousarray(np.asarray(camera.world_to_camera, np.float64).reshape(16))
        self.cam = _Camera(float(camera.fx), float(camera.fy), float(camera.cx), float(camera.cy),
                           int(camera.width), int(camera.height), (ctypes.c_double * 16)(*w2c),
                           float(camera.near), float(camera.far))
        bg = [float(b) for b in settings.background]
        self.st = _Settings((ctypes.c_double * 3)(*bg), int(settings.tile_size),
                            float(settings.theta_z), float(settings.t_z), float(settings.lambda_z))
        self.bg = np.asarray(bg, np.float64)
        self.width, self.height = int(camera.width), int(camera.height)


class Frame:
    """Sorted, culled splat arrays + tile bins (mirrors reference SplatFrame)."""

    def __init__(self, bound):
        self._b = bound
        status = ctypes.c_int(0)
        L = lib()
        h = L.orc_build_frame(ctypes.byref(bound.sc), ctypes.byref(bound.cam),
                              ctypes.byref(bound.st), ctypes.byref(status))
        if status.value != 0 or not h:
            raise OracleError("orc_build_frame failed with status %d" % status.value)
        self._h = h
        sizes = np.zeros(5, np.int64)
        L.orc_frame_sizes(h, _p(sizes))
        self.count, self.k, self.n_tiles, self.tiles_x, self.tiles_y = (int(v) for v in sizes)
        m = self.count
        for name, (fid, dt, shp) in FIELDS.items():
            arr = np.zeros((m,) + shp, dt)
            if m:
                L.orc_frame_copy(h, fid, _p(arr))
            setattr(self, name, arr)
        self.tile_offsets = np.zeros(self.n_tiles + 1, np.int64)
        L.orc_frame_copy(h, 15, _p(self.tile_offsets))
        self.tile_ids = np.zeros(self.k, np.int32)
        if self.k:
            L.orc_frame_copy(h, 16, _p(self.tile_ids))
        self.width, self.height = bound.width, bound.height
        self.tile_size = int(bound.st.tile_size)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().orc_free_frame(self._h)
                self._h = None
        except Exception:
            pass


def build_frame(scene, camera, settings):
    return Frame(_Bound(scene, camera, settings))


def render(scene, camera, settings, naive=False, frame=None):
    """Forward composite.  Returns dict color, depth, transmittance, normal,
    alpha, counts (per-pixel log length) and the frame."""
    f = frame if frame is not None else build_frame(scene, camera, settings)
    H, W = f.height, f.width
    color = np.zeros((H, W, 3)); depth = np.zeros((H, W)); T = np.zeros((H, W))
    normal = np.zeros((H, W, 3)); counts = np.zeros(H * W, np.int64)
    lib().orc_forward(f._h, _p(f._b.bg), int(naive), _p(color), _p(depth), _p(T), _p(normal),
                      _p(counts))
    return dict(color=color, depth=depth, transmittance=T, normal=normal, alpha=1.0 - T,
                counts=counts.reshape(H, W), frame=f, naive=naive)


def blend_log(out):
    """(offsets, position, alpha, u, v) exactly as the reference BlendLog."""
    f = out["frame"]
    counts = out["counts"].reshape(-1)
    offsets = np.zeros(counts.size + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    tot = int(offsets[-1])
    pos = np.zeros(tot, np.int32); al = np.zeros(tot); u = np.zeros(tot); v = np.zeros(tot)
    st = lib().orc_blend_log(f._h, int(out["naive"]), _p(offsets), _p(pos), _p(al), _p(u), _p(v))
    if st != 0:
        raise OracleError("blend log size mismatch")
    return offsets, pos, al, u, v


def backward(scene, camera, settings, pixel_grad, depth_grad=None, normal_grad=None,
             alpha_grad=None, frame=None):
    """Gradients (grad/backward.py:37-181).

    Returns (grads (KG, N, P) float64 in ParamGrads.flat() row order,
    touched (N,) bool, acc (M, KG, ACC_STRIDE) screen-space accumulators)."""
    f = frame if frame is not None else build_frame(scene, camera, settings)
    b = f._b
    pg = np.asarray(pixel_grad, np.float64)
    single = pg.ndim == 3
    pg = np.ascontiguousarray(pg[None] if single else pg)
    kg = pg.shape[0]

    def _ext(a, shp):
        if a is None:
            return None
        a = np.asarray(a, np.float64)
        if a.ndim == len(shp):
            a = a[None]
        return np.ascontiguousarray(np.broadcast_to(a, (kg,) + shp))

    H, W = f.height, f.width
    dg = _ext(depth_grad, (H, W)); ng = _ext(normal_grad, (H, W, 3)); ag = _ext(alpha_grad, (H, W))
    m = f.count
    acc = np.zeros((max(m, 1), kg, ACC_STRIDE))
    touched_s = np.zeros(max(m, 1), np.uint8)
    P = 11 + 3 * b.B
    grads = np.zeros((kg, b.n, P))
    touched = np.zeros(b.n, bool)
    if m:
        L = lib()
        L.orc_backward_blend(f._h, _p(b.bg), kg, _p(pg), _p(dg), _p(ng), _p(ag), _p(acc),
                             _p(touched_s))
        L.orc_chain_rule(f._h, ctypes.byref(b.sc), ctypes.byref(b.cam), ctypes.byref(b.st), kg,
                         _p(acc), _p(grads))
        touched[f.idx[touched_s[:m].astype(bool)]] = True
    return grads, touched, acc[:m]


def split_grads(flat, B):
    """(N, P) -> dict of reference ParamGrads fields (grad/bundle.py:11-63)."""
    n = flat.shape[0]
    return dict(center=flat[:, 0:3], log_scale=flat[:, 3:6], rotation=flat[:, 6:10],
                opacity_logit=flat[:, 10], sh_coeffs=flat[:, 11:].reshape(n, 3, B))


def exchange_pass(log_scale, rotation, type_spec, theta_e=2.05):
    """In-place copies; returns (log_scale, rotation, type_spec, report dict)."""
    ls = np.array(log_scale, np.float64, order="C", copy=True)
    rot = np.array(rotation, np.float64, order="C", copy=True)
    ty = np.array(type_spec, np.uint8, order="C", copy=True)
    n = ls.shape[0]
    er = np.zeros(n); hist = np.zeros(20, np.int64); counts = np.zeros(4, np.int64)
    st = lib().orc_exchange(n, _p(ls), _p(rot), _p(ty), float(theta_e), _p(er), _p(hist),
                            _p(counts))
    if st != 0:
        raise OracleError("degenerate scales (status %d)" % st)
    rep = dict(n_3d_to_2d=int(counts[0]), n_2d_to_3d=int(counts[1]), n_2d=int(counts[2]),
               n_3d=int(counts[3]), erank_hist=hist, eranks=er)
    return ls, rot, ty, rep
