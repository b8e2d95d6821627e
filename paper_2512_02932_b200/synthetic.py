"""Seeded synthetic workloads.

The generator draws, with ``numpy.random.default_rng(seed)`` in the order
centre, scale, rotation, opacity, SH, type:

* camera: fx = fy = 0.8 W, principal point at the image centre, W2C = I;
* depth z ~ U[2, 8]; pixel ~ U[0, W) x U[0, H) un-projected at z;
* per-axis screen sigma ~ log-U[0.5, 6] px, ``log_scale = ln(sigma z / fx)``;
* quaternion ~ normalised N(0, I4); opacity logit ~ N(0, 1); SH ~ N(0, 0.3);
* type ~ Bernoulli(frac_3d) (1 = volumetric / 3D, 0 = flat / 2D surfel).

Every value is rounded to float32 and stored back as float64, so the float32
device scene and the float64 CPU reference / oracle see bit-identical inputs.
"""

import numpy as np

from .core import CameraView, GaussianSet


def f32_exact(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def synthetic_camera(width, height, world_to_camera=None):
    w2c = np.eye(4) if world_to_camera is None else np.asarray(world_to_camera, np.float64)
    return CameraView(fx=0.8 * width, fy=0.8 * width, cx=width / 2.0, cy=height / 2.0,
                      width=width, height=height, world_to_camera=w2c)


def synthetic_scene(n, width, height, sh_degree, seed=0, frac_3d=0.5, sigma_px=(0.5, 6.0),
                    z_range=(2.0, 8.0), f32=True):
    """(GaussianSet, CameraView) for an n-Gaussian mixed scene at W x H.
    ``f32=False`` keeps the raw float64 draws (not float32-representable)."""
    rng = np.random.default_rng(seed)
    fx = 0.8 * width
    cx, cy = width / 2.0, height / 2.0
    z = rng.uniform(z_range[0], z_range[1], n)
    px = rng.uniform(0.0, width, n)
    py = rng.uniform(0.0, height, n)
    center = np.stack([(px - cx) * z / fx, (py - cy) * z / fx, z], axis=1)
    sigma = np.exp(rng.uniform(np.log(sigma_px[0]), np.log(sigma_px[1]), (n, 3)))
    log_scale = np.log(sigma * z[:, None] / fx)
    rot = rng.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    opacity_logit = rng.normal(size=n)
    b = (sh_degree + 1) ** 2
    sh = rng.normal(0.0, 0.3, size=(n, 3, b))
    type_spec = (rng.random(n) < frac_3d).astype(np.uint8)
    r = f32_exact if f32 else (lambda a: a)
    scene = GaussianSet(r(center), r(log_scale), r(rot), r(opacity_logit), r(sh), type_spec)
    return scene, synthetic_camera(width, height)


def orbit_cameras(scene, n_views, width, height, radius=5.0, seed=0):
    """C5: n_views cameras on a circle of ``radius`` around the scene centroid,
    looking at it.  Returns a list of CameraView."""
    centroid = scene.center.mean(axis=0)
    cams = []
    for v in range(n_views):
        ang = 2.0 * np.pi * v / n_views
        eye = centroid + radius * np.array([np.sin(ang), 0.0, -np.cos(ang)])
        fwd = centroid - eye
        fwd /= np.linalg.norm(fwd)
        up = np.array([0.0, 1.0, 0.0])
        right = np.cross(up, fwd)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd])          # rows: camera x, y, z in world
        w2c = np.eye(4)
        w2c[:3, :3] = R
        w2c[:3, 3] = -R @ eye
        cams.append(synthetic_camera(width, height, w2c))
    return cams
