"""GPU parity of the extension outputs' upstream gradients (depth / normal /
alpha images -> every Gaussian parameter) and of the two full-size configs the
round-1 suite did not cover at size: a config-5 orbit view and config 4's
3M-Gaussian KG=3 backward.

The extension has no reference counterpart (the reference backward takes
colour gradients only, grad/backward.py:37-50).  Its semantics (DESIGN.md
section 5) are pinned on the oracle by central differences
(tests/test_oracle_ext_fd.py); here the GPU is compared with that oracle at
full size and, on small scenes, directly with FD of the float64 oracle.

Tolerances (SURVEY.md 8c parity protocol): tile lists / sort order bit-exact;
images max-abs <= 1e-4, depth relative <= 5e-4; gradients norm-wise relative
<= 1e-3 per field and >= 99.5% of elements within 1e-3 of the field scale.
"""

import numpy as np
import pytest

from _fixtures import grad_rel_err

pytestmark = pytest.mark.gpu


def _frame_and_images(ds, scene, cam, st):
    import oracle
    from paper_2512_02932_b200 import raster
    out = raster.render(ds, cam, st)
    f = out.frame.export()
    ofr = oracle.build_frame(scene, cam, st)
    assert out.frame.count == ofr.count
    assert np.array_equal(f["idx"], ofr.idx), "depth sort order"
    assert np.array_equal(f["bbox"], ofr.bbox), "bboxes"
    assert np.array_equal(f["tile_offsets"], ofr.tile_offsets), "tile offsets"
    assert np.array_equal(f["tile_ids"], ofr.tile_ids), "tile lists"
    ref = oracle.render(scene, cam, st, frame=ofr)
    img = lambda t: t.double().cpu().numpy()  # noqa: E731
    errs = dict(color=np.abs(img(out.color) - ref["color"]).max(),
                T=np.abs(img(out.transmittance) - ref["transmittance"]).max(),
                alpha=np.abs(img(out.alpha) - ref["alpha"]).max(),
                normal=np.abs(img(out.normal) - ref["normal"]).max(),
                depth=(np.abs(img(out.depth) - ref["depth"])
                       / np.maximum(np.abs(ref["depth"]), 1.0)).max())
    for k in ("color", "T", "alpha", "normal"):
        assert errs[k] <= 1e-4, errs
    assert errs["depth"] <= 5e-4, errs
    assert np.array_equal(f["pixel_count"].reshape(-1), ref["counts"].reshape(-1)), "log lengths"
    return out, ofr, errs


def _check_grads(got_list, og, B, errs):
    for k, got in enumerate(got_list):
        e = grad_rel_err(got, og[k], B)
        assert max(e.values()) <= 1e-3, (k, e)
        scale = np.maximum(np.abs(og[k]).max(axis=0, keepdims=True), 1e-12)
        frac = np.mean(np.abs(got - og[k]) <= 1e-3 * scale)
        assert frac >= 0.995, (k, frac)
        errs["grad_%d" % k] = max(e.values())


def _compare_ext(scene, cam, st, kg, seed, ext=("depth", "normal", "alpha")):
    import torch

    import oracle
    from paper_2512_02932_b200 import grad
    from paper_2512_02932_b200.core import DeviceGaussians
    ds = DeviceGaussians.from_host(scene, "cuda")
    out, ofr, errs = _frame_and_images(ds, scene, cam, st)
    H, W = cam.height, cam.width
    rng = np.random.default_rng(seed)
    pg = rng.normal(size=(kg, H, W, 3)).astype(np.float32)
    dg = rng.normal(0, 0.2, size=(kg, H, W)).astype(np.float32) if "depth" in ext else None
    ng = rng.normal(size=(kg, H, W, 3)).astype(np.float32) if "normal" in ext else None
    ag = rng.normal(size=(kg, H, W)).astype(np.float32) if "alpha" in ext else None
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    g, touched = grad.backward(ds, cam, out, dev(pg), depth_grad=dev(dg), normal_grad=dev(ng),
                               alpha_grad=dev(ag))
    f64 = lambda a: None if a is None else a.astype(np.float64)  # noqa: E731
    og, otouched, _ = oracle.backward(scene, cam, st, f64(pg), depth_grad=f64(dg),
                                      normal_grad=f64(ng), alpha_grad=f64(ag), frame=ofr)
    assert np.array_equal(touched.cpu().numpy(), otouched)
    _check_grads([g[k].flat().double().cpu().numpy() for k in range(kg)], og,
                 scene.sh_coeffs.shape[2], errs)
    return errs


def _config3_scene():
    from paper_2512_02932_b200.synthetic import f32_exact, synthetic_camera, synthetic_scene
    scene, cam = synthetic_scene(300_000, 800, 600, 3, seed=2)
    a = 0.25
    R = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
    w2c = np.eye(4)
    w2c[:3, :3] = R
    w2c[:3, 3] = [0.1, -0.05, 0.3]
    scene.center[:] = f32_exact((scene.center - w2c[:3, 3]) @ R)
    return scene, synthetic_camera(800, 600, w2c)


def test_config3_extension_gradients_kg3():
    """Config 3 at full size (300k, 800x600, rotated camera), KG = 3, with
    colour, depth, normal and alpha upstream gradients all set -- the path
    bench.py --config 3 times."""
    from paper_2512_02932_b200.settings import RenderSettings
    scene, cam = _config3_scene()
    errs = _compare_ext(scene, cam, RenderSettings(background=(0.2, 0.3, 0.4)), kg=3, seed=21)
    print("config3 extension errors", errs)


@pytest.mark.parametrize("which", ["depth", "normal", "alpha"])
def test_single_extension_gradient(which):
    """Each extension gradient alone (no cancellation between terms can hide
    an error in one of them), 100k Gaussians at 640x480."""
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(100_000, 640, 480, 2, seed=31)
    errs = _compare_ext(scene, cam, RenderSettings(), kg=1, seed=32, ext=(which,))
    print(which, errs)


def test_extension_fd_gradcheck_gpu():
    """GPU analytic gradients of depth / normal / alpha / colour losses against
    central differences of the float64 oracle (>= 99% within 1e-3)."""
    import torch

    import oracle
    from paper_2512_02932_b200 import grad, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import f32_exact, synthetic_camera
    from test_oracle_ext_fd import _fields, _small_scene
    rng = np.random.default_rng(8)
    cam = synthetic_camera(16, 16)
    st = RenderSettings(background=(0.1, 0.2, 0.3))
    ok = total = 0
    for _ in range(8):
        sc = _small_scene(rng, cam, int(rng.integers(2, 7)))
        for a in _fields(sc):
            a[:] = f32_exact(a)
        w = [f32_exact(rng.normal(size=s)) for s in ((16, 16, 3), (16, 16), (16, 16, 3), (16, 16))]
        ds = DeviceGaussians.from_host(sc, "cuda")
        out = raster.render(ds, cam, st)
        t = [torch.from_numpy(x.astype(np.float32)).cuda() for x in w]
        g, _ = grad.backward(ds, cam, out, t[0], depth_grad=t[1], normal_grad=t[2], alpha_grad=t[3])
        an = g.flat().double().cpu().numpy()

        def loss(s_):
            r = oracle.render(s_, cam, st)
            return float((w[0] * r["color"]).sum() + (w[1] * r["depth"]).sum()
                         + (w[2] * r["normal"]).sum() + (w[3] * r["alpha"]).sum())
        base_idx = oracle.build_frame(sc, cam, st).idx
        offs = [0, 3, 6, 10, 11]
        n, P = an.shape
        eps = 1e-4
        for gi in range(n):
            for slot in range(P):
                fi = max(i for i, o in enumerate(offs) if o <= slot)

                def perturbed(d):
                    s2 = sc.copy()
                    _fields(s2)[fi][gi, slot - offs[fi]] += d
                    return s2
                sp, sm = perturbed(eps), perturbed(-eps)
                if not (np.array_equal(oracle.build_frame(sp, cam, st).idx, base_idx)
                        and np.array_equal(oracle.build_frame(sm, cam, st).idx, base_idx)):
                    continue
                fd = (loss(sp) - loss(sm)) / (2 * eps)
                total += 1
                if abs(an[gi, slot] - fd) <= 1e-3 * max(abs(fd), 1e-2):
                    ok += 1
    assert total > 200
    assert ok / total >= 0.99, (ok, total)


def test_config5_orbit_view16_full_size():
    """Config 5 (the centred 1M / SH3 scene, 64 orbit cameras at 1080p): view
    16, the rotated off-centre view that deferred 152k pixels before the
    eigenbasis records, against the oracle in full."""
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import f32_exact, orbit_cameras, synthetic_scene
    scene, _ = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
    scene.center[:] = f32_exact(scene.center - scene.center.mean(axis=0))
    cam = orbit_cameras(scene, 64, 1920, 1080, radius=5.0)[16]
    errs = _compare_ext(scene, cam, RenderSettings(), kg=1, seed=3, ext=())
    print("config5 view16 errors", errs)


def test_config4_size_kg3():
    """Config 4's size: 3M Gaussians at 1080p (SH3), backward with KG = 3
    stacked upstream gradients (the frequency-decoupled loss stack)."""
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(3_000_000, 1920, 1080, 3, seed=4)
    errs = _compare_ext(scene, cam, RenderSettings(), kg=3, seed=5, ext=())
    print("config4-size errors", errs)
