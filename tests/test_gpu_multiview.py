"""GPU tests of the multi-view gradient path: the chain rule's
accumulate mode (HGS_FLAG_ACCUMULATE), the replay-only backward + ranged
chain rule (hgs_backward_chain) the bucketed all-reduce overlaps with, and
parallel.view_batch_grads on one rank."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(n=20000, w=320, h=240, deg=3, views=3):
    import torch

    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import f32_exact, orbit_cameras, synthetic_scene
    scene, _ = synthetic_scene(n, w, h, deg, seed=5)
    scene.center[:] = f32_exact(scene.center - scene.center.mean(axis=0))
    cams = orbit_cameras(scene, 16, w, h, radius=5.0)[:views]
    ds = DeviceGaussians.from_host(scene, "cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    pgs = [torch.randn((1, h, w, 3), device="cuda", generator=g) for _ in cams]
    return ds, cams, pgs, RenderSettings()


def _single(ds, cam, st, pg, **kw):
    from paper_2512_02932_b200 import grad, raster
    _, frame = raster.rasterize(ds, cam, st)
    g, t = grad.backward_device(frame, pg, **kw)
    return g.clone(), t.clone()


def test_accumulate_equals_sum_of_views():
    import torch

    from paper_2512_02932_b200 import grad, raster
    ds, cams, pgs, st = _setup()
    ref = sum(_single(ds, c, st, p)[0] for c, p in zip(cams, pgs))
    out = torch.full_like(ref, float("nan"))
    for j, (c, p) in enumerate(zip(cams, pgs)):
        _, frame = raster.rasterize(ds, c, st)
        grad.backward_device(frame, p, grads_out=out, accumulate=j > 0)
    err = (out - ref).abs().max() / ref.abs().max()
    assert float(err) < 1e-6


def test_replay_only_then_ranged_chain_rule_equals_full_backward():
    import torch

    from paper_2512_02932_b200 import grad, raster
    from paper_2512_02932_b200.parallel import bucket_bounds
    ds, cams, pgs, st = _setup(views=1)
    ref, tref = _single(ds, cams[0], st, pgs[0])
    _, frame = raster.rasterize(ds, cams[0], st)
    out = torch.full_like(ref, float("nan"))
    _, touched = grad.backward_device(frame, pgs[0], grads_out=out, replay_only=True)
    assert bool(torch.isnan(out).all())  # the replay alone writes no gradient
    for g0, g1 in bucket_bounds(ds.count, 5):
        grad.chain_range(frame, g0, g1, out)
    assert torch.equal(out, ref)
    assert torch.equal(touched, tref)
    # a ranged chain rule is idempotent (the accumulators are read-only)
    grad.chain_range(frame, 0, ds.count, out)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("pipeline", [0, 1, 2])
@pytest.mark.parametrize("views", [2, 3, 4])
def test_view_batch_grads_one_rank(pipeline, views):
    """Sequential and two-stream pipelined view loops both sum every view's
    gradient; the caller's image buffers end up holding the last view."""
    import torch

    from paper_2512_02932_b200 import parallel, raster
    ds, cams, pgs, st = _setup(views=views)
    ref = sum(_single(ds, c, st, p)[0] for c, p in zip(cams, pgs))[0]
    out = torch.empty_like(ref)
    h, w = pgs[0].shape[1:3]
    outputs = dict(color=torch.empty((h, w, 3), device="cuda"), depth=torch.empty((h, w), device="cuda"),
                   transmittance=torch.empty((h, w), device="cuda"), alpha=torch.empty((h, w), device="cuda"),
                   normal=torch.empty((h, w, 3), device="cuda"))
    parallel.view_batch_grads(ds, cams, st, lambda j, im: pgs[j], out, outputs=outputs, pipeline=pipeline)
    err = (out - ref).abs().max() / ref.abs().max()
    assert float(err) < 1e-6
    last, _ = raster.rasterize(ds, cams[-1], st)
    for k in ("color", "depth", "transmittance", "normal"):
        assert torch.equal(outputs[k], last[k]), k


def test_densify_statistics_use_pixel_axis_centre_gradient():
    """hgs_densify_stats rotates the 3D eigenbasis centre sums back to pixel
    axes: its statistic equals |NDC centre gradient| from the oracle's
    screen-space accumulators."""
    import torch

    import oracle
    from paper_2512_02932_b200 import densify, grad, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(3000, 160, 120, 1, seed=8)
    st = RenderSettings()
    ds = DeviceGaussians.from_host(scene, "cuda")
    _, frame = raster.rasterize(ds, cam, st)
    rng = np.random.default_rng(2)
    pg = rng.normal(size=(1, 120, 160, 3)).astype(np.float32)
    from paper_2512_02932_b200 import _lib
    scratch = torch.empty(_lib.lib().hgs_backward_scratch_bytes(ds.count, 1), dtype=torch.uint8,
                          device="cuda")
    _, touched = grad.backward_device(frame, torch.from_numpy(pg).cuda(), scratch=scratch)
    stats = densify.DensifyStats(ds)
    densify.accumulate(frame, stats, scratch, 1, touched)
    got = stats.grad_accum.double().cpu().numpy()
    ofr = oracle.build_frame(scene, cam, st)
    _, ot, acc = oracle.backward(scene, cam, st, pg.astype(np.float64), frame=ofr)
    want = np.zeros(scene.count)
    k3 = ofr.typ == 1
    gx = acc[:, 0, oracle.ACC_CTR] * 80.0
    gy = acc[:, 0, oracle.ACC_CTR + 1] * 60.0
    want[ofr.idx[k3]] = np.hypot(gx, gy)[k3]
    sel = np.zeros(scene.count, bool)
    sel[ofr.idx[k3]] = True
    sel &= ot
    np.testing.assert_allclose(got[sel], want[sel], rtol=2e-3, atol=1e-6 * want.max())


@pytest.mark.parametrize("pipeline", [0, 1, 2])
def test_view_batch_grads_redoes_views_that_outgrew_the_pair_capacity(pipeline):
    """Asynchronous views that overflow the frame's pair capacity composite
    nothing and back-propagate zeros; the batch redoes them synchronously
    (the frame buffer grows), so the summed gradient is unchanged."""
    import torch

    from paper_2512_02932_b200 import parallel, raster
    ds, cams, pgs, st = _setup()
    ref = sum(_single(ds, c, st, p)[0] for c, p in zip(cams, pgs))[0]
    key = (ds.count, int(cams[0].width), int(cams[0].height))
    for first_bad in (True, False):
        raster._pair_hint[key] = 1000  # far below K: every asynchronous view overflows
        out = torch.empty_like(ref)
        views = cams if first_bad else cams[::-1]
        grads = pgs if first_bad else pgs[::-1]
        parallel.view_batch_grads(ds, views, st, lambda j, im: grads[j], out, pipeline=pipeline)
        err = (out - ref).abs().max() / ref.abs().max()
        assert float(err) < 1e-6
        assert raster._pair_hint[key] > 1000  # the synchronous redo grew the hint
