"""Multi-process (gloo, world size 2) tests of the camera-sharded step's
sharding and reduction logic, on CPU.  The per-view gradients come from the
oracle (test infrastructure) so no GPU is needed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2512_02932_b200.parallel import MultiViewStep, shard_views


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
