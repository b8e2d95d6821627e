"""Deferred-pixel counts of one config-2 frame (diag 10/11 = fixup pixels of
the forward / backward, 0/1 = float64 pair re-checks / transmittance replays).
Run on the GPU box."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _lib, grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
ds = DeviceGaussians.from_host(scene, "cuda:0")
_, fr = raster.rasterize(ds, cam, RenderSettings(), _lib.HGS_FLAG_COUNT)
pg = torch.randn((1, 1080, 1920, 3), device="cuda:0")
grad.backward_device(fr, pg, flags=_lib.HGS_FLAG_COUNT)
s = _lib.frame_stats(fr)
print({i: int(v) for i, v in enumerate(s)})
