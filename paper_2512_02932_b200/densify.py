"""Adaptive density control on the B200 (SPEC.md:411-419,
425-427).  The reference keeps the densification statistics on its
GaussianSet (``grad_accum``, ``obs_count``, ``keep``, ``append``,
``reset_stats``: core/types.py:48-49, 110-130) but ships no densify code;
the rule set below follows the SPEC:

* statistics (``accumulate``, after every backward): grad_accum += |NDC-space
  gradient of the projected centre| of the total loss, obs_count += 1 for
  every Gaussian the view touched;
* ``densify``: alpha < prune_opacity -> removed; else mean gradient >
  grad_threshold -> split (max scale > split_scale_frac * extent: two
  children at +-0.5 sigma along the major axis, scales / 1.6) or clone
  (parent + copy); children inherit type_spec; statistics reset; Adam
  moments carried for survivors, zero for new rows.

Everything runs as GPU stream compaction (csrc/hgs_densify.cu); the only host
sync is reading the new count.
"""

from dataclasses import dataclass

from . import _lib
from .core import DeviceGaussians
from .errors import ConfigError

__all__ = ["DensifyConfig", "DensifyStats", "DensifyReport", "accumulate", "densify"]


@dataclass
class DensifyConfig:
    grad_threshold: float = 2e-4      # SPEC.md:425 (3DGS)
    prune_opacity: float = 0.005
    split_scale_frac: float = 0.01    # of the scene extent
    clone_step: float = 0.0           # clone offset in max-scale units along -Adam moment (0 = copy)

    def c_struct(self, extent):
        if not 0.0 <= self.prune_opacity < 1.0 or self.grad_threshold < 0 or self.split_scale_frac <= 0:
            raise ConfigError("bad densify config %r" % (self,))
        return _lib.DensifyCfg(float(self.grad_threshold), float(self.prune_opacity),
                               float(self.split_scale_frac * extent), float(self.clone_step))


@dataclass
class DensifyReport:
    n_before: int
    n_after: int
    kept: int
    pruned: int
    cloned: int
    split: int


class DensifyStats:
    """Per-Gaussian accumulators on the device (types.py:48-49)."""

    def __init__(self, scene):
        import torch
        self.grad_accum = torch.zeros(scene.count, dtype=torch.float32, device=scene.device)
        self.obs_count = torch.zeros(scene.count, dtype=torch.int32, device=scene.device)

    def reset(self):
        self.grad_accum.zero_()
        self.obs_count.zero_()

    @property
    def count(self):
        return int(self.grad_accum.shape[0])


def accumulate(frame, stats, bwd_scratch, kg, touched):
    """Add one view's statistics (call right after grad.backward_device on
    ``frame`` with the same scratch; kg <= 4)."""
    scene = frame.scene
    if stats.count != scene.count:
        raise ConfigError("densify statistics do not match the scene")
    _lib.check(_lib.lib().hgs_densify_stats(
        _lib.scene_struct(scene), _lib.camera_struct(frame.camera), _lib.ptr(frame.buf), frame.info,
        _lib.ptr(bwd_scratch), int(kg), _lib.ptr(touched), _lib.ptr(stats.grad_accum),
        _lib.ptr(stats.obs_count), _lib.current_stream_handle(scene.device)), "hgs_densify_stats")


def densify(scene, stats, config=None, optimizer=None):
    """Returns (new DeviceGaussians, DensifyReport).  ``optimizer`` (optim.Adam)
    is re-targeted in place to the new scene with compacted moments; ``stats``
    is resized and reset."""
    import ctypes

    import torch
    cfg = config or DensifyConfig()
    if stats.count != scene.count:
        raise ConfigError("densify statistics do not match the scene")
    L = _lib.lib()
    dev = scene.device
    n = scene.count
    c = cfg.c_struct(scene.extent)
    nscr = L.hgs_densify_scratch_bytes(n)
    scratch = torch.empty(max(nscr, 1), dtype=torch.uint8, device=dev)
    n_out = ctypes.c_int64(0)
    census = (ctypes.c_int64 * 4)()
    sc = _lib.scene_struct(scene)
    stream = _lib.current_stream_handle(dev)
    _lib.check(L.hgs_densify_plan(sc, _lib.ptr(stats.grad_accum), _lib.ptr(stats.obs_count), c,
                                  _lib.ptr(scratch), nscr, ctypes.byref(n_out), census, stream),
               "hgs_densify_plan")
    m = int(n_out.value)
    B = scene.sh_bases
    out = DeviceGaussians(torch.empty((m, 3), device=dev), torch.empty((m, 3), device=dev),
                          torch.empty((m, 4), device=dev), torch.empty((m,), device=dev),
                          torch.empty((m, 3, B), device=dev),
                          torch.empty((m,), dtype=torch.uint8, device=dev), extent=scene.extent,
                          validate=False)
    m_src = v_src = m_dst = v_dst = None
    if optimizer is not None:
        P = 11 + 3 * B
        m_src, v_src = optimizer.exp_avg, optimizer.exp_avg_sq
        m_dst = torch.empty(m * P, dtype=torch.float32, device=dev)
        v_dst = torch.empty_like(m_dst)
    _lib.check(L.hgs_densify_apply(sc, _lib.ptr(m_src), _lib.ptr(v_src), _lib.ptr(scratch), c,
                                   _lib.params_struct(out), _lib.ptr(out.type_spec), _lib.ptr(m_dst),
                                   _lib.ptr(v_dst), stream), "hgs_densify_apply")
    if optimizer is not None:
        optimizer.scene = out
        optimizer.exp_avg, optimizer.exp_avg_sq = m_dst, v_dst
        optimizer.n_params = m_dst.numel()
    stats.grad_accum = torch.zeros(m, dtype=torch.float32, device=dev)
    stats.obs_count = torch.zeros(m, dtype=torch.int32, device=dev)
    rep = DensifyReport(n, m, int(census[0]), int(census[1]), int(census[2]), int(census[3]))
    return out, rep
