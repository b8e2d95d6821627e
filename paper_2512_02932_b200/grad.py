"""Backward API -- drop-in for the reference's ``hybridsplat.grad``
(grad/backward.py:37-181, grad/bundle.py:11-88).

``backward(scene, camera, output, pixel_grad)`` replays the GPU frame of
``output`` back to front (k_composite_bwd) and runs the float64 per-Gaussian
chain rule (k_chain_rule).  Like the reference it returns one ParamGrads (or a
list of KG) plus the per-Gaussian ``touched`` mask.  Optional extension
gradients: ``depth_grad`` (H,W), ``normal_grad`` (H,W,3), ``alpha_grad``
(H,W), each with the same leading KG dimension as ``pixel_grad`` if stacked.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DeviceGaussians, GaussianSet
from .errors import IntegrityError

# grad/__init__.py:7-8 of the reference
__all__ = ["backward", "GradientBundle", "ParamGrads", "param_labels", "FiniteDiffReport",
           "finite_diff_check"]


@dataclass
class ParamGrads:
    """Gradients for every trainable array of a scene (grad/bundle.py:11-63).
    Arrays are numpy float64 for host scenes, CUDA float32 views of one flat
    buffer for device scenes."""
    center: object
    log_scale: object
    rotation: object
    opacity_logit: object
    sh_coeffs: object

    @classmethod
    def zeros_like(cls, scene):
        if isinstance(scene, DeviceGaussians):
            import torch
            return cls(*(torch.zeros_like(getattr(scene, f)) for f in
                         ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs")))
        return cls(np.zeros_like(scene.center), np.zeros_like(scene.log_scale),
                   np.zeros_like(scene.rotation), np.zeros_like(scene.opacity_logit),
                   np.zeros_like(scene.sh_coeffs))

    @property
    def count(self):
        return self.center.shape[0]

    def flat(self):
        """(N, P) rows: center(3), log_scale(3), rotation(4), opacity(1), sh(3B)."""
        n = self.count
        parts = [self.center.reshape(n, -1), self.log_scale.reshape(n, -1),
                 self.rotation.reshape(n, -1), self.opacity_logit.reshape(n, 1),
                 self.sh_coeffs.reshape(n, -1)]
        if isinstance(self.center, np.ndarray):
            return np.concatenate(parts, axis=1)
        import torch
        return torch.cat(parts, dim=1)

    @classmethod
    def from_flat(cls, flat, template):
        n = template.count
        b = template.sh_coeffs.shape[2]
        if tuple(flat.shape) != (n, 11 + 3 * b):
            raise IntegrityError("flat gradient shape %s does not match scene" % (flat.shape,))
        return cls(flat[:, 0:3], flat[:, 3:6], flat[:, 6:10], flat[:, 10],
                   flat[:, 11:].reshape(n, 3, b))

    def assert_finite(self):
        for name in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs"):
            a = getattr(self, name)
            ok = np.all(np.isfinite(a)) if isinstance(a, np.ndarray) else bool(a.isfinite().all())
            if not ok:
                raise IntegrityError("non-finite gradient in %s" % name)


@dataclass
class GradientBundle:
    """grad/bundle.py:66-76"""
    g_color: ParamGrads
    g_low: ParamGrads
    g_high: ParamGrads

    @classmethod
    def zeros_like(cls, scene):
        return cls(ParamGrads.zeros_like(scene), ParamGrads.zeros_like(scene),
                   ParamGrads.zeros_like(scene))


def param_labels(scene):
    b = scene.sh_coeffs.shape[2]
    per = (["center.%d" % i for i in range(3)] + ["log_scale.%d" % i for i in range(3)]
           + ["rotation.%d" % i for i in range(4)] + ["opacity_logit"]
           + ["sh.%d.%d" % (c, k) for c in range(3) for k in range(b)])
    return [("g%d.%s" % (g, p)) for g in range(scene.count) for p in per]


def _views(flat_block, n, B):
    """ParamGrads views of one field-major (n*P,) block (include/hgs.h)."""
    o = 0
    out = []
    for shape in ((n, 3), (n, 3), (n, 4), (n,), (n, 3, B)):
        size = int(np.prod(shape))
        out.append(flat_block[o:o + size].reshape(shape))
        o += size
    return ParamGrads(*out)


def _as_device(a, dev, name, shape, nonfinite=None):
    """``nonfinite``: a list to which the count of non-finite float64 host
    inputs is appended when the upload could count them (None: not counted,
    the caller checks on the device)."""
    import torch
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float32)
        if nonfinite is not None:
            nonfinite.append(None)
    else:
        from ._hostio import upload
        cnt = {0: None}
        t = upload([(np.asarray(a), torch.float32)], dev, tag="grad_in." + name, nonfinite_out=cnt)[0]
        if nonfinite is not None:
            nonfinite.append(cnt[0])
    if t.dim() == len(shape) - 1:
        t = t.unsqueeze(0)
    if tuple(t.shape[1:]) != shape[1:]:
        raise IntegrityError("%s shape %s does not match the camera" % (name, tuple(a.shape)))
    return t.contiguous()


_det_hint = {}  # (n, kg, W, H) -> record capacity that sufficed last time


def backward_device(frame, pixel_grads, depth_grads=None, normal_grads=None, alpha_grads=None,
                    grads_out=None, touched_out=None, events=None, flags=None, scratch=None,
                    deterministic=False, accumulate=False, replay_only=False):
    """Device-level backward.  pixel_grads (KG,H,W,3) float32 CUDA; returns
    (grads (KG, n*P) float32, touched (n,) uint8).  ``events`` (3
    torch.cuda.Event) are recorded at the library's stage boundaries.
    ``deterministic``: fixed-order gradient reduction (HGS_FLAG_DETERMINISTIC),
    bitwise reproducible run to run, at extra memory and time.
    ``accumulate``: grads_out += this view's gradient (HGS_FLAG_ACCUMULATE).
    ``replay_only`` (KG <= 4): the back-to-front replay only; the chain rule
    follows in Gaussian ranges through ``chain_range`` with the same scratch."""
    import torch
    L = _lib.lib()
    ds = frame.scene
    dev = ds.device
    kg = pixel_grads.shape[0]
    n, B = ds.count, ds.sh_bases
    P = 11 + 3 * B
    if grads_out is None:
        grads_out = torch.empty((kg, n * P), dtype=torch.float32, device=dev)
    if touched_out is None:
        touched_out = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    fl = frame.flags if flags is None else flags
    if deterministic:
        fl |= _lib.HGS_FLAG_DETERMINISTIC
    if accumulate:
        fl |= _lib.HGS_FLAG_ACCUMULATE
    if replay_only:
        fl |= _lib.HGS_FLAG_REPLAY_ONLY
    key = (n, kg, frame.width, frame.height)
    # (only the deterministic mode sizes its records from K: an asynchronous
    # frame's counts stay on the device otherwise)
    records = _det_hint.get(key) or (2 * frame.pair_count + (1 << 16) if deterministic else 0)
    for _ in range(8):
        nscr = (L.hgs_backward_det_scratch_bytes(n, kg, records) if deterministic
                else L.hgs_backward_scratch_bytes(n, kg))
        if scratch is None or scratch.numel() < nscr:
            scratch = torch.empty(nscr, dtype=torch.uint8, device=dev)
        rc = L.hgs_backward(
            _lib.scene_struct(ds), _lib.camera_struct(frame.camera),
            _lib.settings_struct(frame.settings, fl, events), _lib.ptr(frame.buf), frame.info, kg,
            _lib.ptr(pixel_grads), _lib.ptr(depth_grads), _lib.ptr(normal_grads),
            _lib.ptr(alpha_grads), _lib.ptr(scratch), scratch.numel(), _lib.ptr(grads_out),
            _lib.ptr(touched_out), _lib.current_stream_handle(dev))
        if deterministic and rc == _lib.HGS_ERR_PAIR_CAPACITY:
            records *= 8
            continue
        _lib.check(rc, "hgs_backward")
        if deterministic:
            _det_hint[key] = records
        if replay_only:
            frame._replay = (scratch, kg, depth_grads, normal_grads, alpha_grads)
        return grads_out, touched_out[:n]
    raise _lib.ExtensionError("could not size the deterministic backward scratch")


def chain_range(frame, g0, g1, grads_out, accumulate=False):
    """The chain rule of the last ``backward_device(frame, ..., replay_only=True)``
    for Gaussians [g0, g1) into ``grads_out`` (KG, n*P) (hgs_backward_chain)."""
    rep = getattr(frame, "_replay", None)
    if rep is None:
        raise IntegrityError("chain_range needs a replay_only backward on this frame first")
    scratch, kg, dg, ng, ag = rep
    fl = frame.flags | (_lib.HGS_FLAG_ACCUMULATE if accumulate else 0)
    _lib.check(_lib.lib().hgs_backward_chain(
        _lib.scene_struct(frame.scene), _lib.camera_struct(frame.camera),
        _lib.settings_struct(frame.settings, fl), _lib.ptr(frame.buf), frame.info, kg,
        _lib.ptr(dg), _lib.ptr(ng), _lib.ptr(ag), _lib.ptr(scratch), scratch.numel(), int(g0),
        int(g1), _lib.ptr(grads_out), _lib.current_stream_handle(frame.buf.device)),
        "hgs_backward_chain")
    return grads_out


def backward(scene, camera, output, pixel_grad, depth_grad=None, normal_grad=None,
             alpha_grad=None, validate=True, deterministic=False):
    """Gradients of a scalar image loss with upstream dL/d(color image)
    (grad/backward.py:37-181).  pixel_grad (H,W,3) or (KG,H,W,3).  Returns a
    ParamGrads (or a list of KG) and the per-Gaussian touched mask."""
    import torch
    single = pixel_grad.ndim == 3
    H, W = int(camera.height), int(camera.width)
    shape = tuple(pixel_grad.shape[1:]) if not single else tuple(pixel_grad.shape)
    if shape != (H, W, 3):
        raise IntegrityError("pixel_grad shape %s does not match the camera"
                             % (tuple(pixel_grad.shape),))
    frame = output.frame
    dev = frame.scene.device
    host_bad = []  # non-finite float64 inputs counted while narrowing (None: check on the device)
    pg = _as_device(pixel_grad, dev, "pixel_grad", (0, H, W, 3), host_bad)
    dg = _as_device(depth_grad, dev, "depth_grad", (0, H, W), host_bad)
    ng = _as_device(normal_grad, dev, "normal_grad", (0, H, W, 3), host_bad)
    ag = _as_device(alpha_grad, dev, "alpha_grad", (0, H, W), host_bad)
    kg = pg.shape[0]
    for t in (dg, ng, ag):
        if t is not None and t.shape[0] != kg:
            raise IntegrityError("extension gradients must have the same KG as pixel_grad")
    if validate:
        # float64 host arrays: checked on their float64 values by the upload
        # (a finite 1e300 is accepted, as by the reference); device tensors:
        # checked on the device
        tens = [t for t in (pg, dg, ng, ag) if t is not None]
        if any(c for c in host_bad if c is not None):
            raise IntegrityError("pixel_grad contains non-finite values")
        dev_check = [t for t, c in zip(tens, host_bad) if c is None]
        if dev_check and bool(torch.stack([~torch.isfinite(t).all() for t in dev_check]).any()):
            raise IntegrityError("pixel_grad contains non-finite values")
    output.check_scene(scene)
    host = isinstance(scene, GaussianSet)
    grads, touched = backward_device(frame, pg, dg, ng, ag, deterministic=deterministic)
    n, B = frame.scene.count, frame.scene.sh_bases
    if host:
        from ._hostio import download
        g = download([grads], tag="grads")[0]
        out = []
        for k in range(kg):
            v = _views(g[k], n, B)
            out.append(ParamGrads(v.center, v.log_scale, v.rotation, v.opacity_logit,
                                  v.sh_coeffs))
        touched = touched.cpu().numpy().astype(bool)
    else:
        out = [_views(grads[k], n, B) for k in range(kg)]
        touched = touched.bool()
    return (out[0] if single else out), touched


# ---------------------------------------------------------------- finite differences

def _slot_ref(scene, gauss, slot):
    """(array, index) of flat parameter ``slot`` of Gaussian ``gauss`` in the
    canonical ParamGrads.flat() order (grad/findiff.py:27-56)."""
    b = scene.sh_coeffs.shape[2]
    if slot < 3:
        return scene.center, (gauss, slot)
    if slot < 6:
        return scene.log_scale, (gauss, slot - 3)
    if slot < 10:
        return scene.rotation, (gauss, slot - 6)
    if slot == 10:
        return scene.opacity_logit, (gauss,)
    k = slot - 11
    return scene.sh_coeffs, (gauss, k // b, k % b)


@dataclass
class FiniteDiffReport:
    """grad/findiff.py:59-75"""
    rel_err: np.ndarray        # flat over gaussians x params; nan = excluded
    excluded: np.ndarray       # parameters whose perturbation flips the depth order
    labels: list
    analytic: np.ndarray
    numeric: np.ndarray

    @property
    def max_rel_err(self):
        live = self.rel_err[~self.excluded]
        return float(np.nanmax(live)) if live.size else 0.0

    def pass_fraction(self, tol):
        live = self.rel_err[~self.excluded]
        if live.size == 0:
            return 1.0
        return float(np.mean(live <= tol))


def finite_diff_check(scene, camera, loss, loss_grad, eps, param_subset=None,
                      settings=None) -> FiniteDiffReport:
    """Central differences of loss(render(...).color) against the analytic GPU
    backward (grad/findiff.py:78-133): two GPU renders per scalar parameter;
    parameters whose perturbation changes the splat depth order are reported
    as excluded.  eps must lie in [1e-6, 1e-2].  The images are composited
    in float32, so the central differences carry ~1e-3 relative noise at
    eps = 1e-4 (the reference's float64 renders ~1e-9)."""
    from .errors import ConfigError
    from .raster import render
    from .settings import RenderSettings
    if not 1e-6 <= eps <= 1e-2:
        raise ConfigError("eps must be in [1e-6, 1e-2], got %r" % (eps,))
    if settings is None:
        settings = RenderSettings()
    if not isinstance(scene, GaussianSet):
        raise ConfigError("finite_diff_check needs a host GaussianSet")
    out = render(scene, camera, settings)
    base = loss(out.color)
    if not np.isfinite(base):
        raise ConfigError("loss is non-finite at the base point")
    pixel_grad = np.asarray(loss_grad(out.color), dtype=np.float64)
    analytic_grads, _ = backward(scene, camera, out, pixel_grad)
    analytic_flat = analytic_grads.flat()
    p = 11 + 3 * scene.sh_coeffs.shape[2]
    slots = list(range(p) if param_subset is None else param_subset)
    n = scene.count
    rel = np.full((n, p), np.nan)
    excluded = np.zeros((n, p), dtype=bool)
    numeric = np.full((n, p), np.nan)
    for gi in range(n):
        for slot in slots:
            work = scene.copy()
            arr, ix = _slot_ref(work, gi, slot)
            theta = float(arr[ix])
            arr[ix] = theta + eps
            out_p = render(work, camera, settings)
            arr[ix] = theta - eps
            out_m = render(work, camera, settings)
            if not np.array_equal(out_p.frame.idx, out_m.frame.idx):
                excluded[gi, slot] = True
                continue
            fd = (loss(out_p.color) - loss(out_m.color)) / (2.0 * eps)
            numeric[gi, slot] = fd
            rel[gi, slot] = abs(analytic_flat[gi, slot] - fd) / max(abs(fd), 1e-8)
    mask = np.zeros((n, p), dtype=bool)
    mask[:, slots] = True
    labels = param_labels(scene)
    return FiniteDiffReport(rel_err=rel[mask], excluded=excluded[mask],
                            labels=[l for l, m in zip(labels, mask.ravel()) if m],
                            analytic=analytic_flat[mask], numeric=numeric[mask])
