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
    return _exchange_pass_host(scene, config)


def _exchange_pass_host(scene, config):
    """Host GaussianSet: the float64 kernels (hgs_exchange_f64) on a float64
    copy of log_scale / rotation / type_spec, then only the flipped rows are
    written back in place -- demoted rows get their float64
    reparameterisation, promoted rows only the type flip -- exactly the rows
    the reference touches (exchange.py:137-149).  A DegenerateScaleError
    leaves the scene untouched."""
    import torch

    from ._hostio import upload
    n = scene.count
    dev = torch.device("cuda", torch.cuda.current_device())
    ls, rot, ty = upload([(scene.log_scale, torch.float64), (scene.rotation, torch.float64),
                          (scene.type_spec, torch.uint8)], dev, tag="exchange")
    eranks = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    scratch = torch.empty(256, dtype=torch.uint8, device=dev)
    rep = _lib.ExchangeReport()
    _lib.check(_lib.lib().hgs_exchange_f64(n, _lib.ptr(ls), _lib.ptr(rot), _lib.ptr(ty),
                                           float(config.theta_e), _lib.ptr(eranks),
                                           _lib.ptr(scratch), rep, _lib.current_stream_handle(dev)),
               "hgs_exchange_f64")
    new_ty = ty.cpu().numpy()
    demoted = np.flatnonzero((scene.type_spec == 1) & (new_ty == 0))
    if demoted.size:
        idx = torch.from_numpy(demoted).to(dev)
        scene.log_scale[demoted] = ls[idx].cpu().numpy()
        scene.rotation[demoted] = rot[idx].cpu().numpy()
    scene.type_spec[:] = new_ty
    return ExchangeReport(int(rep.n_3d_to_2d), int(rep.n_2d_to_3d), int(rep.n_2d), int(rep.n_3d),
                          np.array(rep.erank_hist[:], np.int64), np.linspace(1.0, 3.0, 21),
                          eranks[:n].cpu().numpy())
