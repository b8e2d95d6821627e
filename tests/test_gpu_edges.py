"""GPU edge cases of the tiling / contribution-mask machinery against the CPU
oracle: ragged image sizes (partial tiles), a 1x1 image, and very long tile
lists (hundreds of 32-entry chunks per tile, every pixel deferred-heavy)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _check(scene, cam, st, img_tol=1e-4, grad_tol=1e-3):
    import torch
    from paper_2512_02932_b200 import grad, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    ds = DeviceGaussians.from_host(scene, "cuda:0")
    out = raster.render(ds, cam, st)
    ref = oracle.render(scene, cam, st)
    f = out.frame.export()
    assert np.array_equal(f["tile_ids"], ref["frame"].tile_ids)
    assert np.array_equal(f["idx"], ref["frame"].idx)
    assert np.abs(out.color.double().cpu().numpy() - ref["color"]).max() <= img_tol
    assert np.abs(out.transmittance.double().cpu().numpy() - ref["transmittance"]).max() <= img_tol
    rng = np.random.default_rng(3)
    pg = rng.normal(size=(cam.height, cam.width, 3)).astype(np.float32)
    g, touched = grad.backward(ds, cam, out, torch.from_numpy(pg).cuda())
    og, ot, _ = oracle.backward(scene, cam, st, pg.astype(np.float64))
    got = g.flat().double().cpu().numpy()
    den = np.linalg.norm(og[0])
    if den > 0:
        assert np.linalg.norm(got - og[0]) / den <= grad_tol
    assert np.array_equal(touched.cpu().numpy(), ot)
    return out


@pytest.mark.parametrize("wh", [(37, 23), (17, 50), (1, 1), (16, 17)])
def test_ragged_sizes(wh):
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    w, h = wh
    scene, cam = synthetic_scene(1500 if w * h > 1 else 50, w, h, 2, seed=w * 31 + h)
    _check(scene, cam, RenderSettings(background=(0.3, 0.2, 0.1)))


def test_long_tile_lists():
    """Large, low-opacity splats over a small image: thousands of entries per
    tile list (many mask chunks per pixel), late early stops."""
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(6000, 48, 40, 1, seed=7, sigma_px=(4.0, 30.0))
    scene.opacity_logit[:] = np.float32(-3.0)
    out = _check(scene, cam, RenderSettings())
    lists = np.diff(out.frame.export()["tile_offsets"])
    assert lists.max() > 2000  # > 60 chunks in the longest list


@pytest.mark.parametrize("case", range(8))
def test_randomised_scenes(case):
    """Seeded sweep over density, opacity, splat size, SH degree, type mix
    and image shape: images, tile lists and gradients against the oracle."""
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    rng = np.random.default_rng(1000 + case)
    w, h = int(rng.integers(8, 70)), int(rng.integers(8, 70))
    n = int(rng.integers(50, 4000))
    deg = int(rng.integers(0, 4))
    lo_s = float(rng.uniform(0.3, 2.0))
    scene, cam = synthetic_scene(n, w, h, deg, seed=case, frac_3d=float(rng.uniform(0, 1)),
                                 sigma_px=(lo_s, lo_s * float(rng.uniform(1.5, 10.0))))
    scene.opacity_logit[:] = (scene.opacity_logit + np.float32(rng.uniform(-2, 3))).astype(np.float32)
    bg = tuple(float(x) for x in rng.uniform(0, 1, 3))
    _check(scene, cam, RenderSettings(background=bg))


@pytest.mark.gpu
def test_host_fingerprint_fused_with_upload():
    """render's scene fingerprint comes from the upload's staging pass; it must
    equal raster.scene_fingerprint of the same host scene (what backward
    checks), or backward would raise IntegrityError on an unchanged scene."""
    from paper_2512_02932_b200 import raster
    from paper_2512_02932_b200.core import DeviceGaussians, GaussianSet
    from paper_2512_02932_b200.synthetic import synthetic_scene
    for n in (1000, 70_000, 300_000):
        scene, _ = synthetic_scene(n, 64, 48, 3, seed=1)
        hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                         scene.sh_coeffs, scene.type_spec)
        ds = DeviceGaussians.from_host(hs, fingerprint=True)
        assert ds.host_fingerprint == raster.scene_fingerprint(hs)
        hs.center[0, 0] += 1.0  # a changed scene no longer matches
        assert ds.host_fingerprint != raster.scene_fingerprint(hs)


@pytest.mark.gpu
def test_nonfinite_upstream_gradients_rejected():
    """grad.backward raises IntegrityError for inf / NaN upstream gradients,
    checked on the float64 host values while they are narrowed for upload
    and on the device for CUDA tensors (grad/backward.py's validation)."""
    import torch
    from paper_2512_02932_b200 import grad, raster
    from paper_2512_02932_b200.core import GaussianSet
    from paper_2512_02932_b200.errors import IntegrityError
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(2000, 64, 48, 3, seed=4)
    hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                     scene.sh_coeffs, scene.type_spec)
    out = raster.render(hs, cam)
    pg = np.random.default_rng(0).normal(size=(48, 64, 3))
    grad.backward(hs, cam, out, pg)  # finite: fine
    for bad in (np.nan, np.inf, -np.inf):
        p = pg.copy()
        p[7, 9, 1] = bad
        with pytest.raises(IntegrityError):
            grad.backward(hs, cam, out, p)
        with pytest.raises(IntegrityError):
            grad.backward(hs, cam, out, torch.from_numpy(p).float().cuda())
    d = np.zeros((48, 64))
    d[3, 3] = np.nan
    with pytest.raises(IntegrityError):
        grad.backward(hs, cam, out, pg, depth_grad=d)
