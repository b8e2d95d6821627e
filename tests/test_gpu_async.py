"""The sync-free forward (HGS_FLAG_ASYNC): every launch sized from host-known
bounds, the data-dependent counts read on the device.  The same frame as the
synchronous call, capturable in a CUDA graph (forward + backward replayed
with no host round trip), and the failure statuses reported after the fact."""

import numpy as np
import pytest
import torch

from paper_2512_02932_b200 import errors, grad, raster
from paper_2512_02932_b200.core import DeviceGaussians
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    scene, cam = synthetic_scene(20000, 320, 240, 3, seed=4)
    ds = DeviceGaussians.from_host(scene, "cuda:0")
    return scene, cam, ds


def _imgs(cam):
    H, W = cam.height, cam.width
    return dict(color=torch.empty((H, W, 3), device="cuda"), depth=torch.empty((H, W), device="cuda"),
                transmittance=torch.empty((H, W), device="cuda"), alpha=torch.empty((H, W), device="cuda"),
                normal=torch.empty((H, W, 3), device="cuda"))


def test_async_matches_sync(case):
    scene, cam, ds = case
    st = RenderSettings()
    ref, fr_ref = raster.rasterize(ds, cam, st)
    out, fr = raster.rasterize(ds, cam, st, async_=True)
    assert fr.pending
    pg = torch.randn((1, cam.height, cam.width, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    g, t = grad.backward_device(fr, pg)          # backward before the counts are read
    g_ref, t_ref = grad.backward_device(fr_ref, pg)
    for k in ref:
        assert torch.equal(out[k], ref[k]), k
    fr.sync()
    assert not fr.pending
    assert fr.count == fr_ref.count and fr.pair_count == fr_ref.pair_count
    assert np.array_equal(fr.tile_ids, fr_ref.tile_ids)
    assert torch.equal(t, t_ref)
    rel = float((g - g_ref).norm() / g_ref.norm())
    assert rel < 1e-5, rel  # float atomics: summation order only


def test_cuda_graph_replay(case):
    scene, cam, ds = case
    st = RenderSettings()
    ref, fr_ref = raster.rasterize(ds, cam, st)
    n, P = ds.count, 11 + 3 * ds.sh_bases
    imgs = _imgs(cam)
    buf = torch.empty(raster.frame_bytes(n, cam.width, cam.height), dtype=torch.uint8, device="cuda")
    pg = torch.randn((1, cam.height, cam.width, 3), device="cuda")
    grads = torch.empty((1, n * P), device="cuda")
    touched = torch.empty(n, dtype=torch.uint8, device="cuda")
    from paper_2512_02932_b200 import _lib
    scratch = torch.empty(_lib.lib().hgs_backward_scratch_bytes(n, 1), dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside the capture
        _, fr = raster.rasterize(ds, cam, st, outputs=imgs, async_=True, frame_buf=buf)
        grad.backward_device(fr, pg, grads_out=grads, touched_out=touched, scratch=scratch)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        _, fr = raster.rasterize(ds, cam, st, outputs=imgs, async_=True, frame_buf=buf)
        grad.backward_device(fr, pg, grads_out=grads, touched_out=touched, scratch=scratch)
    for k in imgs:
        imgs[k].zero_()
    grads.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(imgs[k], ref[k]), k
    g_ref, _ = grad.backward_device(fr_ref, pg)
    assert float((grads - g_ref).norm() / g_ref.norm()) < 1e-5
    fr.sync()
    assert fr.pair_count == fr_ref.pair_count


def test_async_capacity_and_parameter_errors(case):
    scene, cam, ds = case
    st = RenderSettings()
    small = torch.empty(raster.frame_bytes(ds.count, cam.width, cam.height, pairs=1000), dtype=torch.uint8,
                        device="cuda")
    _, fr = raster.rasterize(ds, cam, st, async_=True, frame_buf=small)
    with pytest.raises(errors.ConfigError):
        fr.sync()
    # the synchronous call grows the buffer and succeeds
    out, fr2 = raster.rasterize(ds, cam, st)
    assert fr2.pair_count > 1000
    bad = DeviceGaussians.from_host(scene, "cuda:0")
    bad.rotation[5] = 0.0
    bad.geom64 = None
    _, fr3 = raster.rasterize(bad, cam, st, async_=True)
    with pytest.raises(errors.InvalidParameterError):
        fr3.sync()
