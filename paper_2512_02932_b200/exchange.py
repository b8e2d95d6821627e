"""Adaptive Type Exchange on the GPU -- drop-in for the reference's
``hybridsplat.exchange.exchange_pass`` (exchange.py:137-155).

One pass computes every effective rank in float64, flips 2D->3D types and
reparameterises 3D->2D Gaussians (covariance preserving: permuted scale axes,
R P^T back to a w >= 0 quaternion), in place on the scene arrays.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import DeviceGaussians, GaussianSet
from .settings import ExchangeConfig

__all__ = ["ExchangeConfig", "ExchangeReport", "exchange_pass"]


@dataclass
class ExchangeReport:
    """exchange.py:47-55 (+ the per-Gaussian eranks, float32)."""
    n_3d_to_2d: int
    n_2d_to_3d: int
    n_2d: int
    n_3d: int
    erank_hist: np.ndarray = field(default_factory=lambda: np.zeros(0))
    erank_edges: np.ndarray = field(default_factory=lambda: np.zeros(0))
    eranks: object = None


def exchange_pass_device(ds: DeviceGaussians, config: ExchangeConfig, eranks_out=None):
    import torch
    L = _lib.lib()
    n = ds.count
    scratch = torch.empty(256, dtype=torch.uint8, device=ds.device)
    if eranks_out is None:
        eranks_out = torch.empty(max(n, 1), dtype=torch.float32, device=ds.device)
    rep = _lib.ExchangeReport()
    _lib.check(L.hgs_exchange(n, _lib.ptr(ds.log_scale), _lib.ptr(ds.rotation),
                              _lib.ptr(ds.type_spec), float(config.theta_e), _lib.ptr(eranks_out),
                              _lib.ptr(scratch), rep, _lib.current_stream_handle(ds.device)),
               "hgs_exchange")
    edges = np.linspace(1.0, 3.0, 21)
    return ExchangeReport(int(rep.n_3d_to_2d), int(rep.n_2d_to_3d), int(rep.n_2d), int(rep.n_3d),
                          np.array(rep.erank_hist[:], np.int64), edges, eranks_out[:n])


def exchange_pass(scene, config: ExchangeConfig = None) -> ExchangeReport:
    """Flip types in place wherever effective rank disagrees with the type."""
    if config is None:
        config = ExchangeConfig()
    if isinstance(scene, DeviceGaussians):
        return exchange_pass_device(scene, config)
    ds = DeviceGaussians.from_host(scene)
    rep = exchange_pass_device(ds, config)
    # write back in place like the reference (float64 arrays)
    scene.log_scale[:] = ds.log_scale.double().cpu().numpy()
    scene.rotation[:] = ds.rotation.double().cpu().numpy()
    scene.type_spec[:] = ds.type_spec.cpu().numpy()
    rep.eranks = rep.eranks.double().cpu().numpy()
    return rep
