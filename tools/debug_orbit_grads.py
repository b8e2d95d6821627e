"""Where do GPU and oracle gradients disagree on config-5 orbit view 16?
Run on the GPU box: python tools/debug_orbit_grads.py [view]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2512_02932_b200 import grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import f32_exact, orbit_cameras, synthetic_scene  # noqa: E402

view = int(sys.argv[1]) if len(sys.argv) > 1 else 16
scene, _ = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
if "sh0" in sys.argv:  # no view-dependent colour: isolates the projection chain
    scene.sh_coeffs[:, :, 1:] = 0.0
scene.center[:] = f32_exact(scene.center - scene.center.mean(axis=0))
cam = orbit_cameras(scene, 64, 1920, 1080, radius=5.0)[view]
st = RenderSettings()
ds = DeviceGaussians.from_host(scene, "cuda")
out = raster.render(ds, cam, st)
rng = np.random.default_rng(3)
pg = rng.normal(size=(1, 1080, 1920, 3)).astype(np.float32)
g, touched = grad.backward(ds, cam, out, torch.from_numpy(pg).cuda())
got = g[0].flat().double().cpu().numpy()
ofr = oracle.build_frame(scene, cam, st)
og, ot, acc = oracle.backward(scene, cam, st, pg.astype(np.float64), frame=ofr)
ref = og[0]
fields = dict(center=slice(0, 3), log_scale=slice(3, 6), rotation=slice(6, 10))
R = cam.world_to_camera[:3, :3]
t = cam.world_to_camera[:3, 3]
zc = (scene.center @ R.T + t)[:, 2]
pos = {int(i): k for k, i in enumerate(ofr.idx)}
for name, sl in fields.items():
    d = np.linalg.norm(got[:, sl] - ref[:, sl], axis=1)
    tot = np.linalg.norm(ref[:, sl])
    order = np.argsort(-d)
    share = np.cumsum(d[order] ** 2) / max((d ** 2).sum(), 1e-300)
    print("== %s rel %.3e; top-1/10/100 share of err^2: %.3f %.3f %.3f" %
          (name, np.linalg.norm(d) / tot, share[0], share[9], share[99]))
    for i in order[:12]:
        k = pos.get(int(i))
        info = ""
        if k is not None:
            bb = ofr.bbox[k]
            info = "typ %d z %.4f ctr (%.1f, %.1f) bbox %s rad %.1f a_eff %.3f" % (
                ofr.typ[k], ofr.depth[k], ofr.center2d[k][0], ofr.center2d[k][1], bb.tolist(),
                ofr.radius[k], ofr.alpha_eff[k])
        print("  g %7d err %.3e |ref| %.3e got %s ref %s %s" % (
            i, d[i], np.linalg.norm(ref[i, sl]), np.round(got[i, sl], 4).tolist(),
            np.round(ref[i, sl], 4).tolist(), info))
    # error split by type
    for ty in (0, 1):
        msk = scene.type_spec == ty
        print("   type %d rel-share %.3f" % (ty, (d[msk] ** 2).sum() / max((d ** 2).sum(), 1e-300)))

# screen-space accumulators: GPU (float64 scratch, (n, KG, 16)) vs oracle
scratch = torch.empty(int(__import__("paper_2512_02932_b200")._lib.lib().hgs_backward_scratch_bytes(
    ds.count, 1)), dtype=torch.uint8, device="cuda")
grad.backward_device(out.frame, torch.from_numpy(pg).cuda(), scratch=scratch)
gacc = scratch[: ds.count * 16 * 8].view(torch.float64).view(ds.count, 16).cpu().numpy()
d = np.linalg.norm(got[:, 0:3] - ref[:, 0:3], axis=1)
for i in np.argsort(-d)[:4]:
    k = pos[int(i)]
    print("acc g %d typ %d" % (i, ofr.typ[k]))
    print("  gpu   ", np.array2string(gacc[i, :9], precision=6))
    print("  oracle", np.array2string(acc[k, 0, :9], precision=6))
    print("  rel   ", np.array2string((gacc[i, :9] - acc[k, 0, :9]) / np.maximum(np.abs(acc[k, 0, :9]), 1e-30), precision=2))
