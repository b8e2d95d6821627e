"""Same-process A/B of the host I/O modes of the reference-facing API at
config 2 (alternating rounds; the median of each mode's per-step times).
Run on the GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio, grad, raster  # noqa: E402
from paper_2512_02932_b200.core import GaussianSet  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                 scene.sh_coeffs, scene.type_spec)
st = RenderSettings()
pg = np.random.default_rng(0).normal(size=(1080, 1920, 3))
MODES = {
    "torch copy, gpu widen 0.4": dict(widen=0.4, nt=False),
    "nt, gpu widen 0.25": dict(widen=0.25, nt=True),
    "nt, host only": dict(widen=0.0, nt=True),
}
res = {m: [] for m in MODES}
for rnd in range(4):
    for m, cfg in MODES.items():
        _hostio._GPU_WIDEN = cfg["widen"]
        _hostio._NT = cfg["nt"]
        for it in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = raster.render(hs, cam, st)
            gr, touched = grad.backward(hs, cam, out, pg)
            torch.cuda.synchronize()
            if it >= 2:
                res[m].append((time.perf_counter() - t0) * 1e3)
for m, v in res.items():
    print("%-26s median %.2f ms  min %.2f ms  (%d steps)" % (m, np.median(v), np.min(v), len(v)))
