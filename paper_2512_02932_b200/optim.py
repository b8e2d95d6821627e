"""The optimizer step and the single-view training step on the B200
(SURVEY.md 8(f) rows 1-2).

``train_step`` is the frequency-decoupled step of Alg. 1 end to end on the
device, without a host round trip:

  render (hgs_forward) -> image_losses (hgs_image_losses: L_color, L_low,
  L_high and the (3, H, W, 3) upstream stack) -> backward with KG = 3
  (hgs_backward) -> combine_gradients + Adam + quaternion renormalisation in
  one fused pass (hgs_combine_adam_step).

Multi-GPU steps (parallel.MultiViewTrainStep) combine per view, all-reduce
the combined gradient, then call ``Adam.step``.

The reference ships no trainer or optimizer (the SPEC's ``train`` module is
absent); the optimizer follows SPEC.md:424 -- a first-order adaptive-moment
method with the 3DGS per-group learning rates (center 1.6e-4 decaying
exponentially to 1.6e-6 and scaled by the scene extent, log_scale 5e-3,
rotation 1e-3, opacity 5e-2, SH 2.5e-3) -- in torch.optim.Adam's arithmetic
(pinned by tests/golden/make_freq_golden.py).
"""

import math
from dataclasses import dataclass, field

from . import _lib
from .errors import ConfigError

__all__ = ["AdamConfig", "Adam", "train_step", "TrainStepResult"]

GROUPS = ("center", "log_scale", "rotation", "opacity_logit", "sh")


@dataclass
class AdamConfig:
    lr: dict = field(default_factory=lambda: {"center": 1.6e-4, "log_scale": 5e-3,
                                              "rotation": 1e-3, "opacity_logit": 5e-2,
                                              "sh": 2.5e-3})
    center_lr_final: float = 1.6e-6
    decay_steps: int = 30000        # SPEC.md:387 / Appendix A: 30K iterations
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-15

    def lrs(self, step, extent=1.0):
        """Per-group learning rates at 1-based ``step`` (3DGS exponential
        decay of the centre rate, scaled by the scene extent)."""
        if set(self.lr) != set(GROUPS):
            raise ConfigError("lr must name exactly the groups %s" % (GROUPS,))
        t = min(max(step - 1, 0) / max(self.decay_steps, 1), 1.0)
        c0, c1 = self.lr["center"], self.center_lr_final
        center = math.exp(math.log(c0) * (1 - t) + math.log(c1) * t) if c0 > 0 and c1 > 0 else c0
        return [center * extent] + [self.lr[g] for g in GROUPS[1:]]


class Adam:
    """Adam moments for a DeviceGaussians (flat field-major float32 buffers,
    the ParamGrads layout of hgs_backward)."""

    def __init__(self, scene, config=None):
        import torch
        self.scene = scene
        self.config = config or AdamConfig()
        n, B = scene.count, scene.sh_bases
        self.n_params = n * (11 + 3 * B)
        self.exp_avg = torch.zeros(self.n_params, dtype=torch.float32, device=scene.device)
        self.exp_avg_sq = torch.zeros_like(self.exp_avg)
        self.steps = 0

    def _cfg(self):
        self.steps += 1
        lr = self.config.lrs(self.steps, self.scene.extent)
        b1, b2 = self.config.betas
        return _lib.AdamCfg((ctypes_float5())(*lr), float(b1), float(b2), float(self.config.eps),
                            self.steps)

    def _check(self):
        if self.exp_avg.numel() != self.scene.count * (11 + 3 * self.scene.sh_bases):
            raise ConfigError("optimizer state does not match the scene (densified?)")

    def step(self, grads):
        """Adam + rotation renormalisation with a flat (n*P) gradient."""
        self._check()
        dev = self.scene.device
        _lib.check(_lib.lib().hgs_adam_step(
            _lib.params_struct(self.scene), _lib.ptr(grads.contiguous()), _lib.ptr(self.exp_avg),
            _lib.ptr(self.exp_avg_sq), self._cfg(), _lib.current_stream_handle(dev)),
            "hgs_adam_step")

    def step_combined(self, g_color, g_low, g_high, mode="projection", n_conflicts=None):
        """Fused combine_gradients (Alg. 1) + Adam + renormalisation."""
        import torch
        self._check()
        if mode not in _lib.COMBINE_MODES:
            raise ConfigError("mode must be one of %s" % (tuple(_lib.COMBINE_MODES),))
        dev = self.scene.device
        if n_conflicts is None:
            n_conflicts = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().hgs_combine_adam_step(
            _lib.params_struct(self.scene), _lib.ptr(g_color), _lib.ptr(g_low), _lib.ptr(g_high),
            _lib.ptr(self.scene.type_spec), _lib.COMBINE_MODES[mode], _lib.ptr(self.exp_avg),
            _lib.ptr(self.exp_avg_sq), self._cfg(), _lib.ptr(n_conflicts),
            _lib.current_stream_handle(dev)), "hgs_combine_adam_step")
        return n_conflicts


def ctypes_float5():
    import ctypes
    return ctypes.c_float * 5


@dataclass
class TrainStepResult:
    losses: object        # float64 CUDA tensor [L1, SSIM, L_low, L_high, L_color]
    n_conflicts: object   # int64 CUDA tensor (1,)
    pair_count: int
    color: object         # the rendered (H, W, 3) image of this step: a view of the
                          # per-device workspace, overwritten by the next train_step
                          # (clone() it to keep it across steps)

    def total_loss(self, weights):
        """L = L_color + lambda_low L_low + lambda_high L_high (Eq. 8); syncs."""
        l = self.losses.cpu().tolist()
        return l[4] + weights.lambda_low * l[2] + weights.lambda_high * l[3]


class _Workspace:
    """Per-(scene, camera size) device buffers reused across steps."""

    def __init__(self, scene, H, W):
        import torch
        dev = scene.device
        n, B = scene.count, scene.sh_bases
        P = 11 + 3 * B
        L = _lib.lib()
        self.key = (n, B, H, W)
        self.grads = torch.empty((3, n * P), dtype=torch.float32, device=dev)
        self.touched = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.bwd_scratch = torch.empty(L.hgs_backward_scratch_bytes(n, 3), dtype=torch.uint8,
                                       device=dev)
        self.stack = torch.empty((3, H, W, 3), dtype=torch.float32, device=dev)
        self.imgs = dict(color=torch.empty((H, W, 3), device=dev),
                         depth=torch.empty((H, W), device=dev),
                         transmittance=torch.empty((H, W), device=dev))


_ws = {}


def train_step(scene, camera, gt, optimizer, weights=None, settings=None, flags=0, events=None,
               stats=None):
    """One frequency-decoupled training step of one view, all on the GPU
    (Alg. 1).  ``gt``: (H, W, 3) float32 CUDA image.
    ``stats`` (densify.DensifyStats) accumulates the densification
    statistics of this view.  Returns a TrainStepResult (device tensors; no
    host sync)."""
    from . import freq, grad, raster
    from .settings import RenderSettings
    w = weights or freq.LossWeights()
    st = settings or RenderSettings()
    H, W = int(camera.height), int(camera.width)
    if tuple(gt.shape) != (H, W, 3):
        raise ConfigError("gt image shape %s does not match the camera" % (tuple(gt.shape),))
    key = (scene.count, scene.sh_bases, H, W)
    ws = _ws.get(scene.device)  # one workspace per device, rebuilt when the sizes change
    if ws is None or ws.key != key:
        _ws.pop(scene.device, None)
        ws = _ws[scene.device] = _Workspace(scene, H, W)
    ev = events or [None] * 4
    if ev[0] is not None:
        ev[0].record()
    imgs, frame = raster.rasterize(scene, camera, st, flags, outputs=ws.imgs)
    if ev[1] is not None:
        ev[1].record()
    losses, stack = freq.image_losses(imgs["color"], gt, w, out=ws.stack)
    if ev[2] is not None:
        ev[2].record()
    g, _ = grad.backward_device(frame, stack, grads_out=ws.grads, touched_out=ws.touched,
                                scratch=ws.bwd_scratch)
    if stats is not None:
        from . import densify
        densify.accumulate(frame, stats, ws.bwd_scratch, 3, ws.touched)
    if ev[3] is not None:
        ev[3].record()
    nc = optimizer.step_combined(g[0], g[1], g[2], w.mode)
    return TrainStepResult(losses, nc, frame.pair_count, imgs["color"])
