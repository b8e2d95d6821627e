"""Fraction of Gaussians with a contribution (the backward's touched mask) at
config 2 -- how much of the chain rule's per-Gaussian input the touched-row
skip can leave unread.  Run on the GPU box."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

for cfg, (n, w, h) in {"c2": (1_000_000, 1920, 1080), "c3": (300_000, 800, 600)}.items():
    scene, cam = synthetic_scene(n, w, h, 3, seed=0)
    ds = DeviceGaussians.from_host(scene, torch.device("cuda", 0))
    imgs, frame = raster.rasterize(ds, cam, RenderSettings(), 0)
    pg = torch.randn((1, h, w, 3), device="cuda")
    touched = torch.empty(n, dtype=torch.uint8, device="cuda")
    grad.backward_device(frame, pg, touched_out=touched)
    torch.cuda.synchronize()
    t = touched.bool()
    warps = t.view(-1, 32).any(1) if n % 32 == 0 else t[: n - n % 32].view(-1, 32).any(1)
    print(cfg, "touched %.3f of Gaussians, %.3f of 32-Gaussian warp steps" % (t.float().mean(), warps.float().mean()))
