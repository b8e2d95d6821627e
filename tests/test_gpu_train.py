"""GPU parity of the training-step kernels (include/hgs_train.h) against the
reference's own outputs (tests/golden/freq.npz) and the pinned oracle
(oracle/freq.py): loss stack, Haar transform, gradient surgery, Adam, and
the fused single-view training step.

Float tolerances (float32 kernels vs float64 reference): loss values
relative 1e-5; gradient images norm-wise relative 1e-4 (SSIM parts 1e-3,
its moments cancel in float32); surgery totals 1e-5 with conflict counts
exact; Adam relative 1e-5."""

import os

import numpy as np
import pytest

from oracle import freq as of

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "freq.npz")
TAGS = ("even", "odd", "mixed", "gray")


@pytest.fixture(scope="module")
def gold():
    z = np.load(GOLD)
    return {k: z[k] for k in z.files}


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("tag", TAGS)
def test_dwt_kernels_match_reference(gold, tag):
    from paper_2512_02932_b200 import freq
    r = gold[tag + "_r"].astype(np.float64)
    b = freq.dwt_level1(r)
    for nm in ("LL", "LH", "HL", "HH"):
        np.testing.assert_allclose(getattr(b, nm), gold["%s_%s" % (tag, nm)], atol=2e-6)
    np.testing.assert_allclose(freq.idwt_level1(b), gold[tag + "_idwt"], atol=2e-6)
    adj = freq.DwtBands(*(gold["%s_adjin_%s" % (tag, nm)] for nm in ("LL", "LH", "HL", "HH")),
                        r.shape)
    np.testing.assert_allclose(freq.dwt_adjoint(adj), gold[tag + "_adjoint"], atol=1e-5)


@pytest.mark.parametrize("tag", TAGS)
def test_loss_kernels_match_reference(gold, tag):
    from paper_2512_02932_b200 import freq
    r, g = gold[tag + "_r"], gold[tag + "_g"]
    lo, hi = freq.frequency_losses(r, g)
    ref = gold[tag + "_freq_losses"]
    assert abs(lo - ref[0]) <= 1e-5 * ref[0] and abs(hi - ref[1]) <= 1e-5 * ref[1]
    gl, gh = freq.frequency_loss_grads(r, g)
    assert nrel(gl, gold[tag + "_g_low"]) < 1e-5
    assert nrel(gh, gold[tag + "_g_high"]) < 1e-5
    assert abs(freq.ssim(r, g) - float(gold[tag + "_ssim"])) < 1e-5
    assert nrel(freq.ssim_grad(r, g), gold[tag + "_ssim_grad"]) < 1e-3
    for lam in (0.0, 0.2, 1.0):
        k = "%s_color_%g" % (tag, lam)
        assert abs(freq.color_loss(r, g, lam) - float(gold[k + "_loss"])) < 1e-5
        assert nrel(freq.color_loss_grad(r, g, lam), gold[k + "_grad"]) < 1e-3


def test_loss_stack_1080p_matches_oracle():
    """Full-size (1920 x 1080 x 3) loss stack against the oracle."""
    import torch
    from paper_2512_02932_b200 import freq
    rng = np.random.default_rng(7)
    r = rng.uniform(0, 1, size=(1080, 1920, 3)).astype(np.float32)
    g = np.clip(r + rng.normal(0, 0.1, size=r.shape), 0, 1).astype(np.float32)
    w = freq.LossWeights(lam=0.2, lambda_low=0.2, lambda_high=0.4)
    losses, stack = freq.image_losses(torch.from_numpy(r).cuda(), torch.from_numpy(g).cuda(), w)
    ref_stack, ref_l = of.loss_stack(r.astype(np.float64), g.astype(np.float64), 0.2, 0.2, 0.4)
    np.testing.assert_allclose(losses.cpu().numpy(), ref_l, rtol=1e-5)
    st = stack.cpu().numpy()
    for k, tol in ((0, 1e-3), (1, 1e-5), (2, 1e-5)):
        assert nrel(st[k], ref_stack[k]) < tol, k
    # deterministic: a second call is bitwise identical
    losses2, stack2 = freq.image_losses(torch.from_numpy(r).cuda(), torch.from_numpy(g).cuda(), w)
    assert torch.equal(losses, losses2) and torch.equal(stack, stack2)


@pytest.mark.parametrize("mode", ("projection", "naive", "mask"))
def test_surgery_kernel_matches_reference(gold, mode):
    from paper_2512_02932_b200 import freq
    tot, n = freq.combine_gradients(gold["surg_gc"], gold["surg_gl"], gold["surg_gh"],
                                    gold["surg_type"], mode)
    assert n == int(gold["surg_%s_n" % mode])
    np.testing.assert_allclose(tot, gold["surg_" + mode], rtol=1e-5, atol=1e-5)


def test_project_conflicting_gradients_spec_examples():
    from paper_2512_02932_b200 import freq
    l, h = freq.project_conflicting_gradients(np.array([1.0, 0.0]), np.array([1.0, 1.0]), 0)
    assert np.allclose(l, [1, 0]) and np.allclose(h, [1, 1])          # no conflict
    l, h = freq.project_conflicting_gradients(np.array([1.0, 0.0]), np.array([-1.0, 1.0]), 0)
    assert np.allclose(l, [1, 0]) and np.allclose(h, [0, 1])          # Eq. 9
    l, h = freq.project_conflicting_gradients(np.array([-1.0, 1.0]), np.array([1.0, 0.0]), 1)
    assert np.allclose(l, [0, 1]) and np.allclose(h, [1, 0])          # Eq. 10


def _scene(n=3000, W=96, H=72, deg=1, seed=5):
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(n, W, H, deg, seed=seed)
    return scene, cam, DeviceGaussians.from_host(scene, "cuda:0")


def _fields(ds):
    return [getattr(ds, f).detach().double().cpu().numpy().reshape(ds.count, -1)
            for f in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs")]


def test_adam_kernel_matches_oracle():
    import torch
    from paper_2512_02932_b200 import optim
    scene, cam, ds = _scene(500)
    n, B = ds.count, ds.sh_bases
    P = 11 + 3 * B
    cfg = optim.AdamConfig(decay_steps=10)
    opt = optim.Adam(ds, cfg)
    p = _fields(ds)
    m = [np.zeros_like(x) for x in p]
    v = [np.zeros_like(x) for x in p]
    rng = np.random.default_rng(3)
    widths = (3, 3, 4, 1, 3 * B)
    for step in range(1, 4):
        g = rng.normal(size=n * P).astype(np.float32)
        opt.step(torch.from_numpy(g).cuda())
        lrs = cfg.lrs(step, ds.extent)
        o = 0
        for f, wdt in enumerate(widths):
            gf = g[o:o + n * wdt].astype(np.float64).reshape(n, wdt)
            o += n * wdt
            p[f], m[f], v[f] = of.adam_step(p[f], gf, m[f], v[f], lrs[f], step, eps=1e-15)
            if f == 2:
                p[f] = of.renormalize_rotations(p[f])
    for got, want in zip(_fields(ds), p):
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)
    assert opt.exp_avg.abs().sum() > 0


def test_fused_combine_adam_equals_two_pass():
    import torch
    from paper_2512_02932_b200 import freq, optim
    _, _, ds1 = _scene(700, seed=8)
    _, _, ds2 = _scene(700, seed=8)
    n, P = ds1.count, 11 + 3 * ds1.sh_bases
    gen = torch.Generator(device="cuda").manual_seed(0)
    gc, gl, gh = (torch.randn(n * P, device="cuda", generator=gen) for _ in range(3))
    o1, o2 = optim.Adam(ds1), optim.Adam(ds2)
    nc1 = o1.step_combined(gc, gl, gh, "projection")
    comb, nc2 = freq.combine_gradients_device(gc, gl, gh, ds2.type_spec, "projection")
    o2.step(comb)
    assert int(nc1.item()) == int(nc2.item()) > 0
    for f in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs"):
        assert torch.equal(getattr(ds1, f), getattr(ds2, f)), f


def test_train_step_fixed_point_and_descent():
    import torch
    from paper_2512_02932_b200 import freq, optim, raster
    from paper_2512_02932_b200.settings import RenderSettings
    scene, cam, ds = _scene(2000, seed=11)
    st = RenderSettings()
    imgs, _ = raster.rasterize(ds, cam, st)
    gt = imgs["color"].clone()
    before = [getattr(ds, f).clone() for f in ("center", "log_scale", "opacity_logit", "sh_coeffs")]
    # gt == render -> all losses 0.  The D-SSIM gradient at the
    # optimum is 0 only up to rounding (2 d_sig_x + d_sig_xy cancels), so the
    # exact fixed point is checked with lam = 0 (L1 + frequency terms).
    losses, stack = freq.image_losses(imgs["color"], gt, freq.LossWeights())
    l = losses.cpu().numpy()
    assert l[0] == 0.0 and abs(l[1] - 1.0) < 1e-6 and l[2] == 0.0 and l[3] == 0.0 and l[4] < 1e-6
    assert float(stack.abs().max()) < 1e-9
    opt = optim.Adam(ds)
    res = optim.train_step(ds, cam, gt, opt, freq.LossWeights(lam=0.0), st)
    rl = res.losses.cpu().numpy()
    assert rl[0] == rl[2] == rl[3] == rl[4] == 0.0
    for b, f in zip(before, ("center", "log_scale", "opacity_logit", "sh_coeffs")):
        assert torch.equal(b, getattr(ds, f)), f  # zero gradient -> Adam update is exactly 0
    # descent: fit a perturbed copy back to the original render
    _, _, ds2 = _scene(2000, seed=11)
    with torch.no_grad():
        ds2.sh_coeffs.add_(0.05 * torch.randn_like(ds2.sh_coeffs))
    opt2 = optim.Adam(ds2, optim.AdamConfig(lr={"center": 1e-4, "log_scale": 1e-3,
                                                "rotation": 1e-3, "opacity_logit": 1e-2,
                                                "sh": 5e-3}))
    w = freq.LossWeights()
    hist = [optim.train_step(ds2, cam, gt, opt2, w, st).total_loss(w) for _ in range(40)]
    assert hist[-1] < 0.5 * hist[0], hist[::8]


def test_device_checkpoint_round_trip(tmp_path):
    import torch
    from paper_2512_02932_b200 import io as hio
    _, _, ds = _scene(1234, seed=2)
    hio.save_checkpoint(ds, tmp_path / "d.ckpt")
    back = hio.load_checkpoint(tmp_path / "d.ckpt", device="cuda:0")
    for f in ("center", "log_scale", "rotation", "opacity_logit", "sh_coeffs", "type_spec"):
        assert torch.equal(getattr(ds, f), getattr(back, f)), f
