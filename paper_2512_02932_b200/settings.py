"""Settings dataclasses and the rasterizer constants (reference
raster/project.py:20-45 and exchange.py:28-44), passed by value into the
C-ABI settings struct."""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

ALPHA_CLAMP = 0.99          # keeps 1/(1 - alpha) finite in the backward pass
MIN_ALPHA = 1.0 / 255.0     # contributions below this are dropped
EARLY_STOP_T = 1e-4         # stop blending once transmittance falls below
SCREEN_DILATION = 0.3       # px^2 added to the projected covariance diagonal
LOWPASS_SIGMA = 0.5         # px; screen-space low-pass for flat primitives
SUPPORT_C = 2.0 * np.log(255.0)
DEGENERATE_DEN = 1e-9
BBOX_PAD = 1.0
TILE_SIZE = 16              # the CUDA compositor is built for 16x16 tiles


@dataclass
class ExchangeConfig:
    """exchange.py:28-44"""
    theta_e: float = 2.05
    theta_z: float = 1.05
    t_z: float = 1e-3
    lambda_z: float = 1.0
    interval: int = 500
    start_iter: int = 500
    end_iter: int = 30_000

    def __post_init__(self):
        if not 1.0 < self.theta_e < 3.0:
            raise ConfigError("theta_e must be in (1, 3), got %r" % self.theta_e)
        if self.t_z <= 0:
            raise ConfigError("modulation temperature must be positive")
        if self.interval < 1:
            raise ConfigError("exchange interval must be >= 1")


@dataclass
class RenderSettings:
    """raster/project.py:34-45.  ``backend`` keeps the reference's values;
    "auto" and "cuda" select the sm_100a kernels, "cython"/"python" name the
    reference's CPU backends and are rejected (no CPU fallback here)."""
    background: tuple = (0.0, 0.0, 0.0)
    tile_size: int = TILE_SIZE
    theta_z: float = 1.05
    t_z: float = 1e-3
    lambda_z: float = 1.0
    backend: str = "auto"

    def modulation(self):
        return ExchangeConfig(theta_z=self.theta_z, t_z=self.t_z, lambda_z=self.lambda_z)
