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

__all__ = ["ExchangeConfig", "ExchangeReport", "exchange_pass", "effective_rank",
           "choose_permutation", "reparameterize_3d_to_2d", "modulated_z", "modulated_opacity",
           "modulated_opacity_grads", "modulate_opacity", "P_IDENTITY", "P_X", "P_Y"]

# exchange.py:19-25 -- the three axis permutations of choose_permutation
P_IDENTITY = np.eye(3)
P_X = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
P_Y = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
_PERMS = (P_IDENTITY, P_X, P_Y)


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


# ------------------------------------------------------------------ helpers
# The reference's per-primitive helpers (exchange.py:58-134), evaluated on the
# GPU in float64 by the same formulas as the exchange / preprocess kernels
# (hgs_helpers.cu).  They accept a single row or a batch, like the reference.

def _dev():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a):
    import torch
    return torch.from_numpy(np.array(a, dtype=np.float64, order="C")).to(_dev())


def effective_rank(log_scale):
    """exp of the entropy of the normalised squared scales, in [1, 3]
    (exchange.py:58-73); (3,) -> float, (N, 3) -> (N,)."""
    import torch
    ls = np.asarray(log_scale, dtype=np.float64)
    rows = ls.reshape(-1, 3)
    d_ls = _to_dev(rows)
    out = torch.empty(max(rows.shape[0], 1), dtype=torch.float64, device=d_ls.device)
    scratch = torch.empty(256, dtype=torch.uint8, device=d_ls.device)
    _lib.check(_lib.lib().hgs_effective_rank_f64(rows.shape[0], _lib.ptr(d_ls), _lib.ptr(out),
                                                 _lib.ptr(scratch),
                                                 _lib.current_stream_handle(d_ls.device)),
               "effective_rank")
    er = out.cpu().numpy()[:rows.shape[0]]
    return float(er[0]) if ls.ndim == 1 else er.reshape(ls.shape[:-1])


def _reparam(log_scale, rotation=None):
    import torch
    ls = np.asarray(log_scale, dtype=np.float64).reshape(-1, 3)
    n = ls.shape[0]
    d_ls = _to_dev(ls)
    dev = d_ls.device
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    scratch = torch.empty(256, dtype=torch.uint8, device=dev)
    o_ls = o_rot = d_rot = None
    if rotation is not None:
        d_rot = _to_dev(np.asarray(rotation, dtype=np.float64).reshape(-1, 4))
        o_ls = torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev)
        o_rot = torch.empty((max(n, 1), 4), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().hgs_reparameterize_f64(n, _lib.ptr(d_ls), _lib.ptr(d_rot), _lib.ptr(o_ls),
                                                 _lib.ptr(o_rot), _lib.ptr(perm), _lib.ptr(scratch),
                                                 _lib.current_stream_handle(dev)),
               "reparameterize_3d_to_2d")
    p = perm.cpu().numpy()[:n]
    if rotation is None:
        return p
    return p, o_ls.cpu().numpy()[:n], o_rot.cpu().numpy()[:n]


def choose_permutation(scale):
    """Permutation placing the smallest scale on z; ties prefer the identity,
    then P_x (exchange.py:76-88)."""
    # three comparisons, the rule k_exchange_apply / k_reparam apply per row
    sx, sy, sz = np.asarray(scale, dtype=np.float64)
    if sz <= sx and sz <= sy:
        return P_IDENTITY
    if sx <= sy:
        return P_X
    return P_Y


def reparameterize_3d_to_2d(g):
    """Convert a volumetric primitive to flat, preserving its covariance
    (exchange.py:91-99)."""
    from .core import Gaussian
    _, ls, rot = _reparam(np.asarray(g.log_scale)[None], np.asarray(g.rotation)[None])
    return Gaussian(np.array(g.center, dtype=np.float64, copy=True), ls[0], rot[0],
                    g.opacity_logit, np.array(g.sh_coeffs, dtype=np.float64, copy=True), 0)


def _modulation(opacity, log_scale_z, config, want):
    import torch
    lz = np.asarray(log_scale_z, dtype=np.float64)
    shape = np.broadcast_shapes(lz.shape, np.shape(opacity)) if opacity is not None else lz.shape
    lzb = np.broadcast_to(lz, shape).reshape(-1)
    n = lzb.shape[0]
    d_lz = _to_dev(lzb)
    dev = d_lz.device
    d_op = _to_dev(np.broadcast_to(np.asarray(opacity, np.float64), shape).reshape(-1)) \
        if opacity is not None else None
    outs = {k: torch.empty(max(n, 1), dtype=torch.float64, device=dev) for k in want}
    _lib.check(_lib.lib().hgs_modulation_f64(
        n, _lib.ptr(d_op), _lib.ptr(d_lz), float(config.theta_z), float(config.t_z),
        float(config.lambda_z), *(_lib.ptr(outs.get(k)) for k in
                                  ("sz_star", "alpha_eff", "d_alpha", "d_logz")),
        _lib.current_stream_handle(dev)), "modulation")
    res = [outs[k].cpu().numpy()[:n].reshape(shape) for k in want]
    return [float(r) if r.ndim == 0 else r for r in res]


def modulated_z(log_scale_z, config: ExchangeConfig):
    """Gated z scale s_z* = sigmoid((s_z - theta_z) / T_z) s_z (exchange.py:102-105)."""
    return _modulation(None, log_scale_z, config, ("sz_star",))[0]


def modulated_opacity(opacity, log_scale_z, config: ExchangeConfig):
    """alpha exp(-lambda_z s_z*) of a flat primitive (exchange.py:108-111)."""
    return _modulation(opacity, log_scale_z, config, ("alpha_eff",))[0]


def modulated_opacity_grads(opacity, log_scale_z, config: ExchangeConfig):
    """(d alpha_eff / d alpha, d alpha_eff / d log_scale_z) (exchange.py:114-129)."""
    a, b = _modulation(opacity, log_scale_z, config, ("d_alpha", "d_logz"))
    return a, b


def modulate_opacity(g, config: ExchangeConfig) -> float:
    """Scalar form for one primitive (exchange.py:132-134)."""
    return float(modulated_opacity(g.opacity, g.log_scale[2], config))
