"""Scene and camera types: the drop-in input layout of the hot path.

``GaussianSet`` and ``CameraView`` keep the reference's field names, shapes,
dtypes and validation errors (hybridsplat/core/types.py:32-197) so that code
written against the reference constructs them unchanged.  ``DeviceGaussians``
is the B200-resident form: the same six fields as float32 (uint8 for the type
mask) CUDA tensors in structure-of-arrays layout, which is what the C-ABI
kernels read.
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigError, InvalidParameterError

SH_MAX_DEGREE = 3


def n_bases(degree):
    """(degree+1)^2 SH coefficients per channel (core/sh.py:23-24)."""
    return (degree + 1) ** 2


@dataclass
class Gaussian:
    """One primitive (core/types.py:13-29); type_spec 0 = flat (2D), 1 =
    volumetric (3D)."""
    center: np.ndarray          # (3,)
    log_scale: np.ndarray       # (3,)
    rotation: np.ndarray        # (4,) w-first
    opacity_logit: float
    sh_coeffs: np.ndarray       # (3, B)
    type_spec: int

    @property
    def scale(self):
        return np.exp(self.log_scale)

    @property
    def opacity(self):
        return float(1.0 / (1.0 + np.exp(-self.opacity_logit)))


class GaussianSet:
    """Host structure-of-arrays scene, float64 like the reference
    (core/types.py:32-142).  ``sh_coeffs`` is (N, 3, B) channel-major;
    ``type_spec`` is uint8 with 0 = flat (2D surfel), 1 = volumetric (3D)."""

    FIELDS = ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs", "type_spec")

    def __init__(self, center, log_scale, rotation, opacity_logit, sh_coeffs, type_spec,
                 extent=1.0):
        self.center = np.ascontiguousarray(center, dtype=np.float64)
        self.log_scale = np.ascontiguousarray(log_scale, dtype=np.float64)
        self.rotation = np.ascontiguousarray(rotation, dtype=np.float64)
        self.opacity_logit = np.ascontiguousarray(opacity_logit, dtype=np.float64)
        self.sh_coeffs = np.ascontiguousarray(sh_coeffs, dtype=np.float64)
        self.type_spec = np.ascontiguousarray(type_spec, dtype=np.uint8)
        self.extent = float(extent)
        self.grad_accum = np.zeros(self.count, dtype=np.float64)
        self.obs_count = np.zeros(self.count, dtype=np.int64)
        self.validate()

    @classmethod
    def empty(cls, sh_degree=2, extent=1.0):
        b = n_bases(sh_degree)
        return cls(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                   np.zeros((0, 3, b)), np.zeros(0, np.uint8), extent=extent)

    @property
    def count(self):
        return self.center.shape[0]

    @property
    def sh_degree(self):
        return int(round(np.sqrt(self.sh_coeffs.shape[2]))) - 1

    @property
    def scales(self):
        return np.exp(self.log_scale)

    @property
    def opacities(self):
        return 1.0 / (1.0 + np.exp(-self.opacity_logit))

    def validate(self):
        """Shape / basis / type / finiteness checks (core/types.py:75-96)."""
        n = self.count
        want = {"center": (n, 3), "log_scale": (n, 3), "rotation": (n, 4),
                "opacity_logit": (n,), "type_spec": (n,)}
        for name, shape in want.items():
            got = getattr(self, name).shape
            if got != shape:
                raise InvalidParameterError(
                    "field %s has shape %s, expected %s" % (name, got, shape))
        if self.sh_coeffs.ndim != 3 or self.sh_coeffs.shape[:2] != (n, 3):
            raise InvalidParameterError("sh_coeffs has shape %s" % (self.sh_coeffs.shape,))
        b = self.sh_coeffs.shape[2]
        if n_bases(self.sh_degree) != b or self.sh_degree > SH_MAX_DEGREE:
            raise InvalidParameterError("sh basis count %d is not (l+1)^2, l <= 3" % b)
        if not np.all((self.type_spec == 0) | (self.type_spec == 1)):
            raise InvalidParameterError("type_spec must be 0 or 1")
        for name in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs"):
            if not np.all(np.isfinite(getattr(self, name))):
                raise InvalidParameterError("non-finite values in %s" % name)

    def get(self, i):
        """core/types.py:98-101"""
        return Gaussian(self.center[i].copy(), self.log_scale[i].copy(), self.rotation[i].copy(),
                        float(self.opacity_logit[i]), self.sh_coeffs[i].copy(),
                        int(self.type_spec[i]))

    def copy(self):
        out = GaussianSet(*(getattr(self, f).copy() for f in self.FIELDS), extent=self.extent)
        out.grad_accum = self.grad_accum.copy()
        out.obs_count = self.obs_count.copy()
        return out

    def keep(self, mask):
        mask = np.asarray(mask, dtype=bool)
        out = GaussianSet(*(getattr(self, f)[mask] for f in self.FIELDS), extent=self.extent)
        out.grad_accum = self.grad_accum[mask].copy()
        out.obs_count = self.obs_count[mask].copy()
        return out

    def type_census(self):
        n3 = int(np.count_nonzero(self.type_spec))
        return self.count - n3, n3

    def renormalize_rotations(self):
        norm = np.linalg.norm(self.rotation, axis=1, keepdims=True)
        bad = norm[:, 0] <= 1e-8
        if np.any(bad):
            self.rotation[bad] = (1.0, 0.0, 0.0, 0.0)
            norm[bad] = 1.0
        self.rotation /= norm

    def to_device(self, device="cuda"):
        return DeviceGaussians.from_host(self, device)


class DeviceGaussians:
    """B200-resident scene: float32 SoA CUDA tensors (uint8 type mask).

    Layout in HBM (N Gaussians, B SH bases): center (N,3), log_scale (N,3),
    rotation (N,4) w-first, opacity_logit (N,), sh_coeffs (N,3,B), type_spec
    (N,) -- 4(11+3B)+1 bytes per Gaussian (237 B at SH degree 3).  Tensors are
    used in place; the optimizer may update them between calls.

    ``geom64`` optionally holds the float64 geometry (center, log_scale,
    rotation, opacity_logit) a host ``GaussianSet`` was uploaded from: while
    it is current (no in-place update of the float32 fields since), the
    forward takes every discrete decision -- depth order, culls, bounding
    boxes, tile lists, the float64 re-checks -- on those exact values, as the
    reference does on its float64 inputs (core/types.py:40-45; hgs.h).
    """

    FIELDS = GaussianSet.FIELDS

    def __init__(self, center, log_scale, rotation, opacity_logit, sh_coeffs, type_spec,
                 extent=1.0, validate=True):
        import torch
        dev = center.device
        self.center = center.to(dev, torch.float32).contiguous()
        self.log_scale = log_scale.to(dev, torch.float32).contiguous()
        self.rotation = rotation.to(dev, torch.float32).contiguous()
        self.opacity_logit = opacity_logit.to(dev, torch.float32).contiguous()
        self.sh_coeffs = sh_coeffs.to(dev, torch.float32).contiguous()
        self.type_spec = type_spec.to(dev, torch.uint8).contiguous()
        self.extent = float(extent)
        self.geom64 = None
        self._geom64_versions = None
        self.host_fingerprint = None  # from_host(fingerprint=True): raster.scene_fingerprint of the source
        if validate:
            self.validate()

    GEOM_FIELDS = ("center", "log_scale", "rotation", "opacity_logit")

    @classmethod
    def from_host(cls, scene, device="cuda", validate=False, geom64=True, fingerprint=False):
        """Upload a host scene through pinned staging, pipelined with the DMA
        (_hostio.upload).  The geometry crosses as float64 (kept as ``geom64``
        for the exact decisions, its float32 rounding made on the device);
        SH coefficients are converted to float32 on the host cores.
        ``geom64=False`` uploads float32 geometry only.  ``fingerprint``:
        also set ``host_fingerprint`` -- raster.scene_fingerprint of the host
        scene, its sums taken by the staging pass itself (no extra read)."""
        import torch

        from ._hostio import upload
        if isinstance(device, str):
            device = torch.device(device)
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        gdt = torch.float64 if geom64 else torch.float32
        sums = {0: None, 1: None, 3: None} if fingerprint else None
        t = upload([(scene.center, gdt), (scene.log_scale, gdt), (scene.rotation, gdt),
                    (scene.opacity_logit, gdt), (scene.sh_coeffs, torch.float32),
                    (scene.type_spec, torch.uint8)], device, tag="scene", sums_out=sums)
        out = cls(*t, extent=scene.extent, validate=validate)
        if fingerprint:
            from .raster import scene_fingerprint
            if all(sums[k] is not None for k in (0, 1, 3)):
                out.host_fingerprint = (scene.count, sums[0], sums[3], sums[1])
            else:  # not staged as float64: the plain fingerprint
                out.host_fingerprint = scene_fingerprint(scene)
        if geom64:
            out.geom64 = tuple(t[:4])
            out._geom64_versions = out.versions()
        return out

    def geom64_current(self):
        """The float64 geometry if it still describes the float32 fields."""
        if self.geom64 is None or self.versions() != self._geom64_versions:
            return None
        return self.geom64

    def to_host(self):
        return GaussianSet(*(getattr(self, f).detach().cpu().numpy() for f in self.FIELDS),
                           extent=self.extent)

    @property
    def device(self):
        return self.center.device

    @property
    def count(self):
        return self.center.shape[0]

    @property
    def sh_bases(self):
        return self.sh_coeffs.shape[2]

    @property
    def sh_degree(self):
        return int(round(np.sqrt(self.sh_bases))) - 1

    def validate(self):
        import torch
        n = self.count
        want = {"center": (n, 3), "log_scale": (n, 3), "rotation": (n, 4),
                "opacity_logit": (n,), "type_spec": (n,)}
        for name, shape in want.items():
            got = tuple(getattr(self, name).shape)
            if got != shape:
                raise InvalidParameterError(
                    "field %s has shape %s, expected %s" % (name, got, shape))
        if self.sh_coeffs.dim() != 3 or tuple(self.sh_coeffs.shape[:2]) != (n, 3):
            raise InvalidParameterError("sh_coeffs has shape %s" % (tuple(self.sh_coeffs.shape),))
        if n_bases(self.sh_degree) != self.sh_bases or self.sh_degree > SH_MAX_DEGREE:
            raise InvalidParameterError("sh basis count %d is not (l+1)^2" % self.sh_bases)
        if n == 0:
            return
        checks = [((self.type_spec > 1).any(), "type_spec must be 0 or 1")]
        for name in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs"):
            checks.append(((~torch.isfinite(getattr(self, name))).any(),
                           "non-finite values in %s" % name))
        flags = torch.stack([c for c, _ in checks]).cpu().tolist()
        for bad, (_, msg) in zip(flags, checks):
            if bad:
                raise InvalidParameterError(msg)

    def versions(self):
        """Cheap, sync-free identity of the parameter state (tensor version
        counters bump on every in-place update)."""
        return tuple((getattr(self, f).data_ptr(), getattr(self, f)._version)
                     for f in self.FIELDS)


@dataclass
class CameraView:
    """Pinhole camera with a rigid world-to-camera pose (core/types.py:145-197).
    Pixel (ix, iy) is sampled at (ix + 0.5, iy + 0.5)."""
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray
    near: float = 0.01
    far: float = 100.0
    gt_image: Optional[np.ndarray] = None
    gt_depth: Optional[np.ndarray] = None
    cam_id: str = ""

    def __post_init__(self):
        self.world_to_camera = np.asarray(self.world_to_camera, dtype=np.float64)
        if self.fx <= 0 or self.fy <= 0:
            raise ConfigError("focal lengths must be positive")
        if not (0 < self.near < self.far):
            raise ConfigError("need 0 < near < far")
        if self.world_to_camera.shape != (4, 4):
            raise ConfigError("world_to_camera must be 4x4")
        R = self.world_to_camera[:3, :3]
        if not np.allclose(R @ R.T, np.eye(3), atol=1e-6):
            raise ConfigError("world_to_camera rotation block is not orthonormal")
        if int(self.width) <= 0 or int(self.height) <= 0:
            raise ConfigError("image dimensions must be positive")
        if self.gt_image is not None:
            self.gt_image = np.asarray(self.gt_image, dtype=np.float64)
            if self.gt_image.shape != (self.height, self.width, 3):
                raise ConfigError("gt_image shape does not match camera dims")

    @property
    def camera_center(self):
        R = self.world_to_camera[:3, :3]
        return -R.T @ self.world_to_camera[:3, 3]

    def projection_matrix(self):
        K = np.array([[self.fx, 0.0, self.cx, 0.0], [0.0, self.fy, self.cy, 0.0],
                      [0.0, 0.0, 1.0, 0.0], [0.0, 0.0, 1.0, 0.0]])
        return K @ self.world_to_camera
