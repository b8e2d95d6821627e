"""cProfile of the reference-facing host API step at config 2 (render +
backward through float64 numpy): where the host time goes beyond the
conversions.  Run on the GPU box:  python tools/e2e_cprofile.py"""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import grad, raster  # noqa: E402
from paper_2512_02932_b200.core import GaussianSet  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                 scene.sh_coeffs, scene.type_spec)
st = RenderSettings()
pg = np.random.default_rng(0).normal(size=(1080, 1920, 3))


def step():
    out = raster.render(hs, cam, st)
    g, touched = grad.backward(hs, cam, out, pg)
    torch.cuda.synchronize()


for _ in range(4):
    step()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
