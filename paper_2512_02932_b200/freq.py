"""Frequency-decoupled optimisation on the B200 -- drop-in for the reference's
``hybridsplat.freq`` (freq/dwt.py, freq/ssim.py, freq/surgery.py).

Every function runs the sm_100a kernels of ``csrc/hgs_loss.cu`` /
``csrc/hgs_optim.cu`` through the C ABI (include/hgs_train.h).  Host numpy
inputs come back as float64 numpy like the reference; CUDA tensors stay on
the device (float32).  There is no CPU path.

The training step uses the device-level ``image_losses``: one call yields all
five loss values and the (3, H, W, C) upstream gradient stack
[dL_color/dI, lambda_low dL_low/dI, lambda_high dL_high/dI] that
``grad.backward_device`` consumes as KG = 3, and ``combine_gradients_device``
/ ``optim.Adam.step_combined`` apply Alg. 1 per Gaussian.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, IntegrityError

__all__ = ["DwtBands", "dwt_level1", "idwt_level1", "dwt_adjoint", "frequency_losses",
           "frequency_loss_grads", "ssim", "ssim_grad", "color_loss", "color_loss_grad",
           "LossWeights", "MODES", "project_conflicting_gradients", "combine_gradients",
           "image_losses", "combine_gradients_device"]

MODES = ("projection", "naive", "mask")
WINDOW_SIZE = 11
WINDOW_SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


@dataclass
class LossWeights:
    """freq/surgery.py:19-30"""
    lam: float = 0.2
    lambda_low: float = 0.2
    lambda_high: float = 0.4
    mode: str = "projection"

    def __post_init__(self):
        if min(self.lam, self.lambda_low, self.lambda_high) < 0:
            raise ConfigError("loss weights must be >= 0")
        if self.mode not in MODES:
            raise ConfigError("mode must be one of %s" % (MODES,))


@dataclass
class DwtBands:
    """freq/dwt.py:19-29"""
    LL: object
    LH: object
    HL: object
    HH: object
    orig_shape: tuple

    def detail_bands(self):
        return (self.LH, self.HL, self.HH)


# ---------------------------------------------------------------- plumbing
def _dev():
    import torch
    if not torch.cuda.is_available():
        from .errors import ExtensionError
        raise ExtensionError("the loss kernels need a CUDA device (no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dev=None):
    """-> (float32 contiguous CUDA tensor, was_host)."""
    import torch
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.to(_dev())
        return a.to(torch.float32).contiguous(), False
    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(a).to(dev or _dev(), torch.float32).contiguous(), True


def _hwc(shape):
    if len(shape) == 2:
        return int(shape[0]), int(shape[1]), 1
    if len(shape) == 3:
        return int(shape[0]), int(shape[1]), int(shape[2])
    raise ConfigError("images must be HxW or HxWxC, got %s" % (tuple(shape),))


def _out(t, host):
    return t.double().cpu().numpy() if host else t


def _pair(rendered, gt, what="rendered and gt"):
    r, host_r = _to_dev(rendered)
    g, host_g = _to_dev(gt, r.device)
    if tuple(r.shape) != tuple(g.shape):
        raise ConfigError("%s shapes differ: %s vs %s" % (what, tuple(r.shape), tuple(g.shape)))
    if r.numel() == 0:
        raise ConfigError("cannot transform an empty image")
    return r, g, host_r or host_g


def image_losses(rendered, gt, weights=None, grads=True, out=None):
    """Device-level loss stack of one view (hgs_image_losses).

    Returns (losses, stack): ``losses`` a float64 CUDA tensor of 5 values
    [L1, SSIM, L_low, L_high, L_color]; ``stack`` (3, H, W, C) float32 =
    [dL_color/dI, lambda_low dL_low/dI, lambda_high dL_high/dI] or None."""
    import torch
    w = weights or LossWeights()
    if not 0.0 <= w.lam <= 1.0:
        raise ConfigError("dssim mix must be in [0,1], got %r" % (w.lam,))
    r, g, _ = _pair(rendered, gt)
    H, W, C = _hwc(r.shape)
    dev = r.device
    L = _lib.lib()
    nscr = L.hgs_loss_scratch_bytes(H, W, C)
    scratch = torch.empty(nscr, dtype=torch.uint8, device=dev)
    losses = torch.empty(_lib.HGS_LOSS_COUNT, dtype=torch.float64, device=dev)
    stack = None
    if grads:
        stack = out if out is not None else torch.empty((3,) + tuple(r.shape), dtype=torch.float32,
                                                        device=dev)
    _lib.check(L.hgs_image_losses(H, W, C, _lib.ptr(r), _lib.ptr(g),
                                  _lib.LossWeights(float(w.lam), float(w.lambda_low),
                                                   float(w.lambda_high)),
                                  _lib.ptr(losses), _lib.ptr(stack), _lib.ptr(scratch), nscr,
                                  _lib.current_stream_handle(dev)), "hgs_image_losses")
    return losses, stack


# --------------------------------------------------------------------- DWT
def dwt_level1(image):
    """freq/dwt.py:55-74"""
    import torch
    x, host = _to_dev(image)
    if x.numel() == 0:
        raise ConfigError("cannot transform an empty image")
    H, W, C = _hwc(x.shape)
    bshape = ((H + 1) // 2, (W + 1) // 2) + tuple(x.shape[2:])
    bands = [torch.empty(bshape, dtype=torch.float32, device=x.device) for _ in range(4)]
    _lib.check(_lib.lib().hgs_dwt_level1(H, W, C, _lib.ptr(x), *(_lib.ptr(b) for b in bands),
                                         _lib.current_stream_handle(x.device)), "hgs_dwt_level1")
    return DwtBands(*(_out(b, host) for b in bands), tuple(x.shape))


def _inverse(bands, adjoint):
    import torch
    shape = tuple(bands.orig_shape)
    H, W, C = _hwc(shape)
    host = not isinstance(bands.LL, torch.Tensor)
    bs = [_to_dev(getattr(bands, k))[0] for k in ("LL", "LH", "HL", "HH")]
    want = ((H + 1) // 2, (W + 1) // 2) + shape[2:]
    if any(tuple(b.shape) != want for b in bs):
        raise ConfigError("band shapes do not match orig_shape %s" % (shape,))
    img = torch.empty(shape, dtype=torch.float32, device=bs[0].device)
    _lib.check(_lib.lib().hgs_dwt_inverse(H, W, C, *(_lib.ptr(b) for b in bs), int(adjoint),
                                          _lib.ptr(img), _lib.current_stream_handle(img.device)),
               "hgs_dwt_inverse")
    return _out(img, host)


def idwt_level1(bands):
    """freq/dwt.py:77-93"""
    return _inverse(bands, False)


def dwt_adjoint(bands):
    """freq/dwt.py:96-105"""
    return _inverse(bands, True)


# ------------------------------------------------------------------ losses
def _losses(rendered, gt, lam, lo=1.0, hi=1.0, grads=False):
    r, g, host = _pair(rendered, gt)
    l, st = image_losses(r, g, LossWeights(lam=lam, lambda_low=lo, lambda_high=hi), grads=grads)
    return l.cpu().numpy(), st, host


def frequency_losses(rendered, gt):
    """(L_low, L_high) (freq/dwt.py:108-119)"""
    l, _, _ = _losses(rendered, gt, 0.0)
    return float(l[_lib.HGS_LOSS_LOW]), float(l[_lib.HGS_LOSS_HIGH])


def frequency_loss_grads(rendered, gt):
    """(dL_low/dI, dL_high/dI) (freq/dwt.py:122-137)"""
    _, st, host = _losses(rendered, gt, 0.0, grads=True)
    return _out(st[1], host), _out(st[2], host)


def ssim(x, y):
    """Mean SSIM, 11x11 Gaussian window, zero padded (freq/ssim.py:39-49)"""
    l, _, _ = _losses(x, y, 1.0)
    return float(l[_lib.HGS_LOSS_SSIM])


def ssim_grad(x, y):
    """d mean(SSIM)/dx (freq/ssim.py:52-74): with lam = 1 the colour
    gradient is -0.5 * ssim_grad exactly."""
    _, st, host = _losses(x, y, 1.0, grads=True)
    return _out(st[0] * -2.0, host)


def color_loss(rendered, gt, lam):
    """(1 - lam) L1 + lam (1 - SSIM) / 2 (freq/ssim.py:77-87)"""
    if not 0.0 <= lam <= 1.0:
        raise ConfigError("dssim mix must be in [0,1], got %r" % (lam,))
    l, _, _ = _losses(rendered, gt, float(lam))
    return float(l[_lib.HGS_LOSS_COLOR])


def color_loss_grad(rendered, gt, lam):
    """freq/ssim.py:90-94"""
    _, st, host = _losses(rendered, gt, float(lam), grads=True)
    return _out(st[0], host)


# ----------------------------------------------------------------- surgery
def combine_gradients_device(g_color, g_low, g_high, type_spec, mode="projection", out=None,
                             n_conflicts=None, sh_bases=None):
    """Device-level Alg. 1 over field-major (n*P) ParamGrads blocks (the
    layout hgs_backward writes).  Returns (combined, n_conflicts u64 tensor)."""
    import torch
    if mode not in MODES:
        raise ConfigError("mode must be one of %s" % (MODES,))
    n = int(type_spec.shape[0])
    total = int(g_color.numel())
    if sh_bases is None:
        if n == 0 or (total // n - 11) % 3:
            raise IntegrityError("gradient arrays are misaligned with the scene")
        sh_bases = (total // n - 11) // 3
    if not (g_color.numel() == g_low.numel() == g_high.numel() == n * (11 + 3 * sh_bases)):
        raise IntegrityError("gradient arrays are misaligned with the scene")
    dev = g_color.device
    if out is None:
        out = torch.empty_like(g_color)
    if n_conflicts is None:
        n_conflicts = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().hgs_combine_gradients(
        n, sh_bases, _lib.ptr(g_color), _lib.ptr(g_low), _lib.ptr(g_high),
        _lib.ptr(type_spec.to(torch.uint8).contiguous()), _lib.COMBINE_MODES[mode], _lib.ptr(out),
        _lib.ptr(n_conflicts), _lib.current_stream_handle(dev)), "hgs_combine_gradients")
    return out, n_conflicts


def _rows_to_field_major(a, B):
    """(N, P) rows (grad/bundle.py:32-44 order) -> field-major flat tensor."""
    import torch
    n = a.shape[0]
    parts = [a[:, 0:3], a[:, 3:6], a[:, 6:10], a[:, 10:11], a[:, 11:11 + 3 * B]]
    return torch.cat([p.reshape(-1) for p in parts]) if n else a.reshape(-1)


def _field_major_to_rows(f, n, B):
    import torch
    o, cols = 0, []
    for w in (3, 3, 4, 1, 3 * B):
        cols.append(f[o:o + n * w].reshape(n, w))
        o += n * w
    return torch.cat(cols, dim=1)


def combine_gradients(g_color, g_low, g_high, type_spec, mode="projection"):
    """Total per-primitive update gradients plus the conflict count
    (freq/surgery.py:55-92).  Inputs are (N, P) flattened per-primitive
    gradient matrices; P = 11 + 3B (ParamGrads.flat order)."""
    import torch
    if mode not in MODES:
        raise ConfigError("mode must be one of %s" % (MODES,))
    host = not isinstance(g_color, torch.Tensor)
    gc, gl, gh = (_to_dev(x)[0] for x in (g_color, g_low, g_high))
    ts = type_spec if isinstance(type_spec, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(type_spec), dtype=np.uint8))
    ts = ts.to(gc.device, torch.uint8)
    if not (gc.shape == gl.shape == gh.shape and gc.dim() == 2 and gc.shape[0] == ts.shape[0]):
        raise IntegrityError("gradient arrays are misaligned with the scene")
    n, P = gc.shape
    if P <= 11 + 3 * 16 and (P - 11) % 3 == 0 and (P - 11) // 3 in (1, 4, 9, 16):
        B, pad = (P - 11) // 3, 0
    elif P <= 11 + 3 * 16:
        # not a ParamGrads row: opaque vectors, zero-padded (dots and norms
        # are unchanged) into a degree-3 row
        B, pad = 16, 11 + 3 * 16 - P
    else:
        raise IntegrityError("rows longer than a degree-3 ParamGrads row (59) are not supported")

    def fm(x):
        return _rows_to_field_major(torch.nn.functional.pad(x, (0, pad)) if pad else x, B)
    out, nc = combine_gradients_device(fm(gc), fm(gl), fm(gh), ts, mode, sh_bases=B)
    rows = _field_major_to_rows(out, n, B)[:, :P]
    return _out(rows, host), int(nc.item())


def project_conflicting_gradients(g_low, g_high, type_spec):
    """One primitive's band conflict (freq/surgery.py:33-52), through the same
    kernel.  Flat (t = 0): combine(g_color = -g_low, g_low, g_high) returns
    exactly g_high' ((-g_low + g_low) = 0).  Volumetric (t = 1): the same with
    the roles swapped, since Eq. 10 is Eq. 9 with the bands exchanged."""
    import torch
    host = not isinstance(g_low, torch.Tensor)
    gl = _to_dev(g_low)[0].reshape(1, -1)
    gh = _to_dev(g_high)[0].reshape(1, -1)
    flat = np.zeros(1, np.uint8)
    if int(type_spec) == 0:
        high, _ = combine_gradients(-gl, gl, gh, flat, "projection")
        low, high = gl[0], high[0]
    else:
        low, _ = combine_gradients(-gh, gh, gl, flat, "projection")
        low, high = low[0], gh[0]
    return _out(low, host), _out(high, host)
