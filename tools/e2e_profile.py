"""Phase breakdown of the reference-facing host path (float64 numpy in/out)
at config 2 -- where the e2e time goes.  Run on the GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio, grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians, GaussianSet  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

print("torch threads", torch.get_num_threads())
scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                 scene.sh_coeffs, scene.type_spec)
st = RenderSettings()
pg = np.random.default_rng(0).normal(size=(1080, 1920, 3))


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(4):
    T = {}
    t0 = t()
    ds = DeviceGaussians.from_host(hs)
    t1 = t(); T["upload scene"] = t1 - t0
    imgs, frame = raster.rasterize(ds, cam, st, 0)
    t2 = t(); T["rasterize"] = t2 - t1
    keys = ("color", "depth", "transmittance", "alpha", "normal")
    host = _hostio.download([imgs[k] for k in keys], tag="images")
    t3 = t(); T["download images"] = t3 - t2
    fp = raster.scene_fingerprint(hs)
    t4 = t(); T["fingerprint"] = t4 - t3
    pgd = grad._as_device(pg, ds.device, "pixel_grad", (0, 1080, 1920, 3))
    t5 = t(); T["upload pixel_grad"] = t5 - t4
    ok = bool(torch.isfinite(pgd).all())
    t6 = t(); T["validate pixel_grad"] = t6 - t5
    g, touched = grad.backward_device(frame, pgd)
    t7 = t(); T["backward"] = t7 - t6
    gh = _hostio.download([g], tag="grads")[0]
    t8 = t(); T["download grads"] = t8 - t7
    tb = touched.cpu().numpy().astype(bool)
    t9 = t(); T["touched"] = t9 - t8
    T["total"] = t9 - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()})
# the public API end to end
for it in range(8):
    t0 = t()
    out = raster.render(hs, cam, st)
    gr, touched = grad.backward(hs, cam, out, pg)
    print("public API ms", round((t() - t0) * 1e3, 2))
