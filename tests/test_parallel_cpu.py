"""Multi-process (gloo, world size 2) tests of the camera-sharded step's
sharding and reduction logic, on CPU.  The per-view gradients come from the
oracle (test infrastructure) so no GPU is needed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2512_02932_b200.parallel import (MultiViewStep, bucket_bounds, bucketed_allreduce,
                                            field_slices, shard_views)


def test_shard_views_partition():
    for n in range(0, 20):
        for w in range(1, 6):
            got = [v for r in range(w) for v in shard_views(n, r, w)]
            assert got == list(range(n))
            sizes = [len(shard_views(n, r, w)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene_and_views(n_views):
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import orbit_cameras, synthetic_scene
    scene, _ = synthetic_scene(300, 40, 32, 1, seed=11)
    cams = orbit_cameras(scene, n_views, 40, 32, radius=6.0)
    return scene, cams, RenderSettings()


def _oracle_view_grad(scene, camera, settings, loss_grad, out_buf):
    import oracle
    out = oracle.render(scene, camera, settings)
    pg = loss_grad(torch.from_numpy(out["color"]))
    grads, _, _ = oracle.backward(scene, camera, settings, pg.numpy())
    n, B = scene.count, scene.sh_coeffs.shape[2]
    flat = grads[0]  # (N, P) row-major -> field-major like the C ABI
    fm = np.concatenate([flat[:, 0:3].ravel(), flat[:, 3:6].ravel(), flat[:, 6:10].ravel(),
                         flat[:, 10].ravel(), flat[:, 11:].ravel()])
    assert fm.size == n * (11 + 3 * B)
    out_buf += torch.from_numpy(fm).float()


def _loss_grad(v, color):
    rng = np.random.default_rng(100 + v)
    target = torch.from_numpy(rng.uniform(0, 1, tuple(color.shape)))
    return 2.0 * (color.double() - target)


def _worker(rank, world, port, n_views, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams, st = _scene_and_views(n_views)
    P = 11 + 3 * scene.sh_coeffs.shape[2]
    step = MultiViewStep(scene, cams, st, scene.count * P, view_grad=_oracle_view_grad)
    buf = step.step(_loss_grad)
    out_q.put((rank, step.views, buf.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.slow
def test_two_rank_allreduce_equals_single_process_sum():
    n_views = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_views, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    views = res[0][1] + res[1][1]
    assert sorted(views) == list(range(n_views))
    # every rank ends with the same summed buffer
    assert np.array_equal(res[0][2], res[1][2])
    # = the single-process sum over all views
    scene, cams, st = _scene_and_views(n_views)
    P = 11 + 3 * scene.sh_coeffs.shape[2]
    single = MultiViewStep(scene, cams, st, scene.count * P, view_grad=_oracle_view_grad)
    ref = single.step(_loss_grad).numpy()
    np.testing.assert_allclose(res[0][2], ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())


def test_bucket_slices_partition_the_field_major_buffer():
    """Every element of the (n*P) field-major buffer is in exactly one
    bucket's slices, and the slices of Gaussians [g0, g1) hold exactly their
    rows of each field."""
    for n, B, nb in ((1000, 16, 4), (37, 1, 3), (64, 4, 8), (5, 9, 1)):
        P = 11 + 3 * B
        buf = torch.arange(n * P, dtype=torch.float64)
        seen = torch.zeros(n * P, dtype=torch.int64)
        bounds = bucket_bounds(n, nb)
        assert bounds[0][0] == 0 and bounds[-1][1] == n
        assert all(b[1] == c[0] for b, c in zip(bounds, bounds[1:]))
        for g0, g1 in bounds:
            for sl, width, off in zip(field_slices(buf, n, B, g0, g1), (3, 3, 4, 1, 3 * B),
                                      (0, 3 * n, 6 * n, 10 * n, 11 * n)):
                idx = sl.long()
                assert torch.equal(idx, torch.arange(off + width * g0, off + width * g1))
                seen[idx] += 1
        assert bool((seen == 1).all())


def _bucket_worker(rank, world, port, n, B, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = 11 + 3 * B
    full = torch.from_numpy(np.random.default_rng(rank).normal(size=n * P)).float()
    out = torch.full((n * P,), float("nan"))
    order = []

    def write(g0, g1):  # what the chain rule does for a range: write its rows of each field
        order.append((g0, g1))
        for dst, src in zip(field_slices(out, n, B, g0, g1), field_slices(full, n, B, g0, g1)):
            dst.copy_(src)
    bucketed_allreduce(out, n, B, 4, write)
    ref = full.clone()
    dist.all_reduce(ref)
    out_q.put((rank, order, out.numpy().copy(), ref.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_bucketed_allreduce_equals_one_allreduce():
    """The overlapped, bucketed reduction of the multi-view step
    (parallel.view_batch_grads) gives the same buffer as one all-reduce."""
    n, B = 1000, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, n, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, order, out, ref in res:
        assert len(order) == 4
        np.testing.assert_allclose(out, ref, rtol=1e-6, atol=1e-6)
    assert np.array_equal(res[0][2], res[1][2])
