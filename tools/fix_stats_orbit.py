"""Deferred-pixel counts and stage times of one config-5 orbit view (the
centred 1M scene, camera 0 and 16 of the 64).  Run on the GPU box:
HGS_LIB=... python tools/fix_stats_orbit.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _lib, grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import f32_exact, orbit_cameras, synthetic_scene  # noqa: E402

scene, _ = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
scene.center[:] = f32_exact(scene.center - scene.center.mean(axis=0))
cams = orbit_cameras(scene, 64, 1920, 1080, radius=5.0)
ds = DeviceGaussians.from_host(scene, "cuda:0")
pg = torch.randn((1, 1080, 1920, 3), device="cuda:0")
for v in (0, 16):
    _, fr = raster.rasterize(ds, cams[v], RenderSettings(), _lib.HGS_FLAG_COUNT)
    grad.backward_device(fr, pg, flags=_lib.HGS_FLAG_COUNT)
    s = _lib.frame_stats(fr)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    bv = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(3):
        _, fr = raster.rasterize(ds, cams[v], RenderSettings(), 0, events=ev)
        grad.backward_device(fr, pg, events=bv)
    torch.cuda.synchronize()
    st = [round(ev[j].elapsed_time(ev[j + 1]), 3) for j in range(4)] + \
         [round(bv[j].elapsed_time(bv[j + 1]), 3) for j in range(2)]
    print("view", v, "M", fr.count, "K", fr.pair_count, "stages", st,
          "f64 rechecks", int(s[0]), "T replays", int(s[1]), "fix fwd/bwd", int(s[10]), int(s[11]),
          "defer 3D/2D/T", int(s[12]), int(s[13]), int(s[14]), "longest", int(s[15]))
