"""paper_2512_02932_b200 -- B200-native hybrid 2D/3D Gaussian rasterizer.

A from-scratch sm_100a implementation of the hot path of EGGS (arXiv
2512.02932): the hybrid Gaussian rasterizer forward and backward and the
Adaptive Type Exchange kernel, behind the Python call signatures of the
reference package ``hybridsplat`` (render / backward / exchange_pass).

Layout:
  core.py      GaussianSet / CameraView (reference types) + DeviceGaussians
  raster.py    render, render_naive, RenderOutput, SplatFrame, BlendLog
  grad.py      backward, ParamGrads
  exchange.py  exchange_pass
  parallel.py  camera-sharded multi-view step with an NCCL gradient all-reduce
  _lib.py      ctypes binding of libhgs.so (include/hgs.h)
  csrc/        the CUDA kernels and the C ABI
"""

from . import errors
from .core import CameraView, DeviceGaussians, Gaussian, GaussianSet, n_bases
from .errors import (CheckpointError, ConfigError, DegenerateIntersection, DegenerateScaleError,
                     ExtensionError,
                     IntegrityError, InvalidParameterError, ManifestError, NumericError,
                     SplatError)
from .settings import (ALPHA_CLAMP, EARLY_STOP_T, LOWPASS_SIGMA, MIN_ALPHA, SCREEN_DILATION,
                       ExchangeConfig, RenderSettings)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-facing modules import lazily so `import paper_2512_02932_b200` works
    # on machines without the extension (the entry points then raise
    # ExtensionError -- there is no CPU fallback).
    import importlib
    if name in ("raster", "grad", "exchange", "parallel", "synthetic"):
        return importlib.import_module("." + name, __name__)
    if name in ("render", "render_naive", "RenderOutput", "BlendLog", "SplatFrame", "build_frame",
                "evaluate_contribution", "ray_splat_intersect", "project_gaussian_3d",
                "ProjectedSplat"):
        return getattr(importlib.import_module(".raster", __name__), name)
    if name in ("backward", "ParamGrads", "GradientBundle", "param_labels", "finite_diff_check",
                "FiniteDiffReport"):
        return getattr(importlib.import_module(".grad", __name__), name)
    if name in ("exchange_pass", "ExchangeReport", "effective_rank", "choose_permutation",
                "reparameterize_3d_to_2d", "modulated_z", "modulated_opacity",
                "modulated_opacity_grads", "modulate_opacity"):
        return getattr(importlib.import_module(".exchange", __name__), name)
    raise AttributeError(name)
