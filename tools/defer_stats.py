"""Deferral statistics of one config-2 frame (HGS_FLAG_COUNT): why pixels go
to the float64 fixup kernels."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2512_02932_b200 import _lib, grad, raster
from paper_2512_02932_b200.core import DeviceGaussians
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_scene
scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
ds = DeviceGaussians.from_host(scene, "cuda:0")
imgs, fr = raster.rasterize(ds, cam, RenderSettings(), _lib.HGS_FLAG_COUNT)
pg = torch.randn((1, 1080, 1920, 3), device="cuda")
grad.backward_device(fr, pg, flags=_lib.HGS_FLAG_COUNT)
st = _lib.frame_stats(fr)
names = ["f64 re-evals", "T replays", "ev3", "ev2", "c3", "c2", "b3", "b2ray", "b2lp", "bev",
         "fixup fwd px", "fixup bwd px", "defer 3D pair", "defer 2D pair", "defer early-stop", "-"]
for n, v in zip(names, st):
    print("%-18s %d" % (n, v))
