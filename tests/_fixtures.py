"""Helpers shared by the tests: golden fixture loading and comparators."""

import os

import numpy as np

from paper_2512_02932_b200.core import CameraView, GaussianSet
from paper_2512_02932_b200.settings import RenderSettings

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
# raw_f64: float64 inputs that are not float32-representable (its float32
# rounding changes the depth order and tile lists); grazing: edge-on 2D surfels
# (near-degenerate ray/plane solves)
SCENES = ("tiny_sh3", "stress2d", "rotcam_sh2", "c1", "raw_f64", "grazing")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    scene = GaussianSet(d["in_center"], d["in_log_scale"], d["in_rotation"],
                        d["in_opacity_logit"], d["in_sh"], d["in_type"])
    fx, fy, cx, cy, near, far = d["cam_intr"]
    w, h = (int(v) for v in d["cam_size"])
    cam = CameraView(fx, fy, cx, cy, w, h, d["cam_w2c"], near=near, far=far)
    th, tz, lz = d["modulation"]
    st = RenderSettings(background=tuple(float(b) for b in d["background"]), theta_z=th,
                        t_z=tz, lambda_z=lz)
    return scene, cam, st, d


def grad_rel_err(a, b, B):
    """Per-field norm-wise relative error of flat (N, P) gradients."""
    fields = dict(center=slice(0, 3), log_scale=slice(3, 6), rotation=slice(6, 10),
                  opacity_logit=slice(10, 11), sh=slice(11, 11 + 3 * B))
    out = {}
    for k, s in fields.items():
        den = np.linalg.norm(b[:, s])
        out[k] = np.linalg.norm(a[:, s] - b[:, s]) / max(den, 1e-30)
    return out
