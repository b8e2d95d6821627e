"""Exercise every libhgs.so kernel on small inputs, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) runs:

    compute-sanitizer --tool racecheck --kernel-name kns=hgs \
        python tools/sanitize_drive.py

Covers: the tiled and naive forward (exact, fast, DEFER_ALL counting), the
async forward, the backward (atomic, deterministic, extension gradients,
KG = 3, replay-only + ranged chain rule), the fixup kernels, the exports /
blend log / re-binning, the exchange (float32 and float64), the helper
kernels, the loss stack, surgery + Adam and densification.  Run on the GPU
box (tools/gpu/sanitize.sh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from paper_2512_02932_b200 import _lib, densify, exchange, freq, grad, optim, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import ExchangeConfig, RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402
from _fixtures import load  # noqa: E402


def frame_suite(scene, cam, st, kg=1):
    ds = DeviceGaussians.from_host(scene, "cuda:0")
    H, W = cam.height, cam.width
    pg = torch.randn((kg, H, W, 3), device="cuda")
    for flags in (0, _lib.HGS_FLAG_FAST, _lib.HGS_FLAG_COUNT | _lib.HGS_FLAG_DEFER_ALL, _lib.HGS_FLAG_NAIVE):
        imgs, fr = raster.rasterize(ds, cam, st, flags)
        grad.backward_device(fr, pg)
    imgs, fr = raster.rasterize(ds, cam, st)
    dg = torch.randn((kg, H, W), device="cuda")
    ng = torch.randn((kg, H, W, 3), device="cuda")
    ag = torch.randn((kg, H, W), device="cuda")
    grad.backward_device(fr, pg, dg, ng, ag)
    grad.backward_device(fr, pg, deterministic=True)
    g, _ = grad.backward_device(fr, pg[:1], replay_only=True)
    grad.chain_range(fr, 0, ds.count // 2, g)
    grad.chain_range(fr, ds.count // 2, ds.count, g, accumulate=True)
    out = raster.RenderOutput(imgs["color"], imgs["depth"], imgs["transmittance"], imgs["alpha"],
                              imgs["normal"], fr, None)
    _ = out.blend_log
    fr.export()
    _, fa = raster.rasterize(ds, cam, st, async_=True)
    grad.backward_device(fa, pg)
    fa.sync()
    raster.build_frame(ds, cam, RenderSettings(tile_size=8)).export()
    torch.cuda.synchronize()
    return ds


def main():
    for name in ("tiny_sh3", "stress2d", "rotcam_sh2", "grazing"):
        scene, cam, st, _ = load(name)
        frame_suite(scene, cam, st, kg=3 if name == "rotcam_sh2" else 1)
        print("frame suite", name, flush=True)
    scene, cam = synthetic_scene(3000, 96, 64, 3, seed=2)
    ds = frame_suite(scene, cam, RenderSettings())
    # exchange (float32 device, float64 host) and the helper kernels
    exchange.exchange_pass(ds, ExchangeConfig())
    exchange.exchange_pass(scene.copy(), ExchangeConfig())
    exchange.effective_rank(scene.log_scale[:50])
    exchange.reparameterize_3d_to_2d(scene.get(0))
    exchange.modulated_opacity_grads(np.full(10, 0.5), np.log(np.linspace(0.9, 1.2, 10)), ExchangeConfig())
    f = raster.build_frame(scene, cam)
    raster.evaluate_contribution(f.splat(0), (10.5, 10.5), 0.7)
    # training step: losses, surgery + Adam, densification
    gt = torch.rand((cam.height, cam.width, 3), device="cuda")
    opt = optim.Adam(ds)
    stats = densify.DensifyStats(ds)
    for mode in ("projection", "mask", "naive"):
        optim.train_step(ds, cam, gt, opt, freq.LossWeights(mode=mode), stats=stats)
    freq.image_losses(gt, gt.flip(0))
    densify.densify(ds, stats, optimizer=opt)
    torch.cuda.synchronize()
    print("sanitize drive done", flush=True)


if __name__ == "__main__":
    main()
