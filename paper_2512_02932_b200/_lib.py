"""ctypes binding of libhgs.so (include/hgs.h).

The extension is mandatory: if libhgs.so is missing or fails to load, every
entry point raises ExtensionError.  There is no CPU fallback.
"""

import ctypes
import os

from .errors import (ConfigError, DegenerateScaleError, ExtensionError, IntegrityError,
                     InvalidParameterError, SplatError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGS_LIB", os.path.join(_HERE, "libhgs.so"))

ABI_VERSION = 3  # include/hgs.h HGS_ABI_VERSION

HGS_OK = 0
HGS_ERR_CONFIG = 1
HGS_ERR_INVALID_PARAMETER = 2
HGS_ERR_INTEGRITY = 3
HGS_ERR_DEGENERATE_SCALE = 4
HGS_ERR_PAIR_CAPACITY = 5
HGS_ERR_CUDA = 6

HGS_FLAG_NAIVE = 0x1
HGS_FLAG_FAST = 0x2
HGS_FLAG_COUNT = 0x4
HGS_FLAG_DETERMINISTIC = 0x8
HGS_FLAG_DEFER_ALL = 0x10  # tests: with HGS_FLAG_COUNT, every pixel goes through the float64 resume kernel
HGS_FLAG_REPLAY_ONLY = 0x20  # hgs_backward: replay only, the chain rule follows via hgs_backward_chain
HGS_FLAG_ACCUMULATE = 0x40   # grads += (multi-view batches)
HGS_FLAG_FRAME_ONLY = 0x80   # build_frame: no compositing
HGS_FLAG_ASYNC = 0x100       # hgs_forward without a host round trip (hgs_frame_sync_info later)
COMPOSITOR_TILE = 16         # the compositor's tile; other tile sizes are re-binned on export

# hgs_train.h constants
HGS_LOSS_L1, HGS_LOSS_SSIM, HGS_LOSS_LOW, HGS_LOSS_HIGH, HGS_LOSS_COLOR = range(5)
HGS_LOSS_COUNT = 5
COMBINE_MODES = {"projection": 0, "naive": 1, "mask": 2}

# Every symbol include/hgs.h and include/hgs_train.h declare.
EXPORTS = ("hgs_abi_version", "hgs_status_string", "hgs_frame_bytes", "hgs_forward",
           "hgs_backward_scratch_bytes", "hgs_backward_det_scratch_bytes", "hgs_backward",
           "hgs_backward_chain", "hgs_exchange",
           "hgs_exchange_f64",
           "hgs_frame_export_arrays", "hgs_blend_log", "hgs_frame_stats",
           "hgs_loss_scratch_bytes", "hgs_image_losses", "hgs_dwt_level1", "hgs_dwt_inverse",
           "hgs_combine_gradients", "hgs_adam_step", "hgs_combine_adam_step",
           "hgs_densify_stats", "hgs_densify_scratch_bytes", "hgs_densify_plan", "hgs_densify_apply",
           "hgs_tile_bins_scratch_bytes", "hgs_frame_tile_bins", "hgs_eval_contributions",
           "hgs_frame_sync_info", "hgs_host_register", "hgs_host_unregister", "hgs_widen_d2h",
           "hgs_host_widen", "hgs_host_narrow", "hgs_host_copy", "hgs_host_narrow_count",
           "hgs_host_sum_block", "hgs_host_block_sums", "hgs_host_copy_block_sums",
           "hgs_effective_rank_f64", "hgs_reparameterize_f64", "hgs_modulation_f64")

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class Scene(ctypes.Structure):
    _fields_ = [("n", _i64), ("sh_bases", _i32), ("reserved", _i32),
                ("center", _vp), ("log_scale", _vp), ("rotation", _vp),
                ("opacity_logit", _vp), ("sh", _vp), ("type_spec", _vp),
                ("center64", _vp), ("log_scale64", _vp), ("rotation64", _vp),
                ("opacity_logit64", _vp)]


class Camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", _i32), ("height", _i32),
                ("world_to_camera", ctypes.c_double * 16), ("near_plane", ctypes.c_double),
                ("far_plane", ctypes.c_double)]


class Settings(ctypes.Structure):
    _fields_ = [("background", ctypes.c_float * 3), ("tile_size", _i32),
                ("theta_z", ctypes.c_double), ("t_z", ctypes.c_double),
                ("lambda_z", ctypes.c_double), ("flags", ctypes.c_uint32),
                ("n_timing_events", _i32), ("timing_events", ctypes.POINTER(_vp)),
                ("aux_stream", _vp), ("aux_events", _vp * 2)]


class Images(ctypes.Structure):
    _fields_ = [("color", _vp), ("depth", _vp), ("transmittance", _vp), ("alpha", _vp),
                ("normal", _vp)]


class FrameInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("m", _i64), ("k", _i64), ("n_tiles", _i64),
                ("width", _i32), ("height", _i32), ("tiles_x", _i32), ("tiles_y", _i32),
                ("pair_capacity", _i64), ("sh_bases", _i32), ("flags", ctypes.c_uint32),
                ("internal", ctypes.c_uint32 * 4)]


class ExchangeReport(ctypes.Structure):
    _fields_ = [("n_3d_to_2d", _i64), ("n_2d_to_3d", _i64), ("n_2d", _i64), ("n_3d", _i64),
                ("erank_hist", _i64 * 20)]


class LossWeights(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("lambda_low", ctypes.c_double),
                ("lambda_high", ctypes.c_double)]


class Params(ctypes.Structure):
    _fields_ = [("n", _i64), ("sh_bases", _i32), ("reserved", _i32),
                ("center", _vp), ("log_scale", _vp), ("rotation", _vp),
                ("opacity_logit", _vp), ("sh", _vp)]


class AdamCfg(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float * 5), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("step", _i64)]


class DensifyCfg(ctypes.Structure):
    _fields_ = [("grad_threshold", ctypes.c_double), ("prune_opacity", ctypes.c_double),
                ("split_scale", ctypes.c_double), ("clone_step", ctypes.c_double)]


class FrameExport(ctypes.Structure):
    _fields_ = [("idx", _vp), ("typ", _vp), ("depth", _vp), ("center2d", _vp), ("cov2d", _vp),
                ("conic", _vp), ("mrow", _vp), ("alpha_eff", _vp), ("color", _vp),
                ("radius", _vp), ("normal", _vp), ("bbox", _vp), ("tile_offsets", _vp),
                ("tile_ids", _vp), ("pixel_count", _vp),
                ("t_cam", _vp), ("alpha", _vp), ("view_dir", _vp), ("cam_dist", _vp)]


_lib = None
_load_error = None


def lib():
    """The loaded libhgs.so; raises ExtensionError if it is unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise ExtensionError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = ("libhgs.so not built (%s); run __graft_entry__.build() or "
                       "make -C paper_2512_02932_b200/csrc" % LIB_PATH)
        raise ExtensionError(_load_error)
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the machine
        _load_error = "failed to load libhgs.so: %s" % e
        raise ExtensionError(_load_error)
    P = ctypes.POINTER
    L.hgs_abi_version.restype = ctypes.c_int
    L.hgs_status_string.restype = ctypes.c_char_p
    L.hgs_status_string.argtypes = [ctypes.c_int]
    L.hgs_frame_bytes.restype = ctypes.c_size_t
    L.hgs_frame_bytes.argtypes = [_i64, _i32, _i32, _i32, _i64]
    L.hgs_forward.argtypes = [P(Scene), P(Camera), P(Settings), _vp, ctypes.c_size_t, P(Images),
                              P(FrameInfo), _vp]
    L.hgs_backward_scratch_bytes.restype = ctypes.c_size_t
    L.hgs_backward_scratch_bytes.argtypes = [_i64, _i32]
    L.hgs_backward_det_scratch_bytes.restype = ctypes.c_size_t
    L.hgs_backward_det_scratch_bytes.argtypes = [_i64, _i32, _i64]
    L.hgs_backward.argtypes = [P(Scene), P(Camera), P(Settings), _vp, P(FrameInfo), _i32, _vp, _vp,
                               _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp, _vp]
    L.hgs_backward_chain.argtypes = [P(Scene), P(Camera), P(Settings), _vp, P(FrameInfo), _i32, _vp,
                                     _vp, _vp, _vp, ctypes.c_size_t, _i64, _i64, _vp, _vp]
    L.hgs_exchange.argtypes = [_i64, _vp, _vp, _vp, ctypes.c_double, _vp, _vp, P(ExchangeReport),
                               _vp]
    L.hgs_exchange_f64.argtypes = L.hgs_exchange.argtypes
    L.hgs_frame_export_arrays.argtypes = [P(Scene), P(Camera), P(Settings), _vp, P(FrameInfo),
                                          P(FrameExport), _vp]
    L.hgs_blend_log.argtypes = [P(Scene), P(Camera), P(Settings), _vp, P(FrameInfo), _vp, _vp,
                                _vp, _vp, _vp, _vp]
    L.hgs_frame_stats.argtypes = [_vp, P(FrameInfo), _vp, _vp]
    L.hgs_frame_sync_info.argtypes = [_vp, P(FrameInfo), _vp]
    L.hgs_host_register.argtypes = [_vp, ctypes.c_size_t]
    L.hgs_host_unregister.argtypes = [_vp]
    L.hgs_widen_d2h.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.hgs_host_widen.argtypes = [_vp, _vp, _i64, _i32]
    L.hgs_host_narrow.argtypes = [_vp, _vp, _i64, _i32]
    L.hgs_host_copy.argtypes = [_vp, _vp, _i64, _i32]
    L.hgs_host_narrow_count.argtypes = [_vp, _vp, _i64, _i32, _vp]
    L.hgs_host_sum_block.restype = _i64
    L.hgs_host_sum_block.argtypes = []
    L.hgs_host_block_sums.argtypes = [_vp, _i64, _vp, _i32]
    L.hgs_host_copy_block_sums.argtypes = [_vp, _vp, _i64, _vp, _i32]
    L.hgs_tile_bins_scratch_bytes.restype = ctypes.c_size_t
    L.hgs_tile_bins_scratch_bytes.argtypes = [_i64, _i32, _i32, _i32, _i64]
    L.hgs_frame_tile_bins.argtypes = [_vp, P(FrameInfo), _i32, _vp, _vp, _i64, _vp, ctypes.c_size_t,
                                      P(_i64), _vp]
    L.hgs_eval_contributions.argtypes = [_i64] + [_vp] * 11
    L.hgs_effective_rank_f64.argtypes = [_i64, _vp, _vp, _vp, _vp]
    L.hgs_reparameterize_f64.argtypes = [_i64] + [_vp] * 7
    L.hgs_modulation_f64.argtypes = [_i64, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, _vp, _vp, _vp, _vp, _vp]
    L.hgs_loss_scratch_bytes.restype = ctypes.c_size_t
    L.hgs_loss_scratch_bytes.argtypes = [_i32, _i32, _i32]
    L.hgs_image_losses.argtypes = [_i32, _i32, _i32, _vp, _vp, P(LossWeights), _vp, _vp, _vp,
                                   ctypes.c_size_t, _vp]
    L.hgs_dwt_level1.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
    L.hgs_dwt_inverse.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp]
    L.hgs_combine_gradients.argtypes = [_i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp]
    L.hgs_adam_step.argtypes = [P(Params), _vp, _vp, _vp, P(AdamCfg), _vp]
    L.hgs_combine_adam_step.argtypes = [P(Params), _vp, _vp, _vp, _vp, _i32, _vp, _vp, P(AdamCfg),
                                        _vp, _vp]
    L.hgs_densify_stats.argtypes = [P(Scene), P(Camera), _vp, P(FrameInfo), _vp, _i32, _vp, _vp, _vp,
                                    _vp]
    L.hgs_densify_scratch_bytes.restype = ctypes.c_size_t
    L.hgs_densify_scratch_bytes.argtypes = [_i64]
    L.hgs_densify_plan.argtypes = [P(Scene), _vp, _vp, P(DensifyCfg), _vp, ctypes.c_size_t,
                                   P(_i64), P(_i64), _vp]
    L.hgs_densify_apply.argtypes = [P(Scene), _vp, _vp, _vp, P(DensifyCfg), P(Params), _vp, _vp, _vp,
                                    _vp]
    if L.hgs_abi_version() != ABI_VERSION:
        _load_error = "libhgs.so ABI version mismatch"
        raise ExtensionError(_load_error)
    _lib = L
    return _lib


def available():
    try:
        lib()
        return True
    except ExtensionError:
        return False


_STATUS_EXC = {
    HGS_ERR_CONFIG: ConfigError,
    HGS_ERR_INVALID_PARAMETER: InvalidParameterError,
    HGS_ERR_INTEGRITY: IntegrityError,
    HGS_ERR_DEGENERATE_SCALE: DegenerateScaleError,
    HGS_ERR_CUDA: ExtensionError,
}


def check(status, what):
    if status == HGS_OK:
        return
    msg = "%s: %s" % (what, lib().hgs_status_string(status).decode())
    raise _STATUS_EXC.get(status, SplatError)(msg)


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def current_stream_handle(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def scene_struct(ds):
    """hgs_scene of a DeviceGaussians; carries the float64 geometry when the
    scene has a current one (DeviceGaussians.geom64)."""
    g = ds.geom64_current()
    g64 = [t.data_ptr() for t in g] if g is not None else [None] * 4
    return Scene(ds.count, ds.sh_bases, 0, ds.center.data_ptr(), ds.log_scale.data_ptr(),
                 ds.rotation.data_ptr(), ds.opacity_logit.data_ptr(), ds.sh_coeffs.data_ptr(),
                 ds.type_spec.data_ptr(), *g64)


def camera_struct(cam):
    w2c = [float(v) for v in cam.world_to_camera.reshape(16)]
    return Camera(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), int(cam.width),
                  int(cam.height), (ctypes.c_double * 16)(*w2c), float(cam.near), float(cam.far))


_aux = {}  # device index -> (side stream, fork event, join event)


def aux_handles(device):
    """(cudaStream_t, (fork, join) cudaEvent_t) of this process's side stream
    on ``device``: hgs_forward runs the float64 preprocess on it beside the
    depth sort (HGS_SORT_ON_AUX builds: the other way round)."""
    import torch
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _aux:
        # HGS_AUX_PRIORITY < 0: a higher-priority side stream (for builds with
        # HGS_SORT_ON_AUX, where the depth sort runs on it)
        stream = torch.cuda.Stream(device=idx, priority=int(os.environ.get("HGS_AUX_PRIORITY", "0")))
        evs = (torch.cuda.Event(), torch.cuda.Event())
        with torch.cuda.device(idx):
            for e in evs:
                e.record()  # creates the CUDA event
        _aux[idx] = (stream, evs)
    stream, evs = _aux[idx]
    return stream.cuda_stream, tuple(e.cuda_event for e in evs)


def settings_struct(st, flags=0, events=None, aux=None):
    """hgs_settings; ``events`` = list of torch.cuda.Event(enable_timing=True)
    recorded by the library at its stage boundaries (include/hgs.h); ``aux``
    = (side stream, (fork, join) events) from aux_handles()."""
    bg = [float(b) for b in st.background]
    if len(bg) != 3:
        raise ConfigError("background must have 3 channels")
    # the compositor always bins at 16 x 16; RenderSettings.tile_size only
    # selects the tile lists SplatFrame exports (hgs_frame_tile_bins)
    s = Settings((ctypes.c_float * 3)(*bg), COMPOSITOR_TILE, float(st.theta_z),
                 float(st.t_z), float(st.lambda_z), int(flags), 0, None)
    if events:
        arr = (_vp * len(events))(*[event_handle(e) for e in events])
        s.n_timing_events = len(events)
        s.timing_events = ctypes.cast(arr, ctypes.POINTER(_vp))
        s._keep = arr
    if aux is not None:
        s.aux_stream = aux[0]
        s.aux_events[0], s.aux_events[1] = aux[1]
    return s


def event_handle(ev):
    """Raw cudaEvent_t of a torch.cuda.Event (created on first record)."""
    if not ev.cuda_event:
        ev.record()
    return ev.cuda_event


def frame_stats(frame):
    import numpy as np
    out = np.zeros(16, np.uint64)
    check(lib().hgs_frame_stats(ptr(frame.buf), frame.info, out.ctypes.data_as(ctypes.c_void_p),
                                current_stream_handle(frame.buf.device)), "hgs_frame_stats")
    return out


def params_struct(ds):
    """hgs_params (mutable scene) of a DeviceGaussians."""
    return Params(ds.count, ds.sh_bases, 0, ds.center.data_ptr(), ds.log_scale.data_ptr(),
                  ds.rotation.data_ptr(), ds.opacity_logit.data_ptr(), ds.sh_coeffs.data_ptr())
