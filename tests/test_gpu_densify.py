"""GPU adaptive density control (csrc/hgs_densify.cu) against the oracle
restatement (oracle/densify.py) and the SPEC's examples;
the count invariant SPEC.md:433."""

import numpy as np
import pytest

from oracle import densify as od

pytestmark = pytest.mark.gpu


def _scene(n=2000, deg=1, seed=4):
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(n, 96, 72, deg, seed=seed)
    return scene, cam, DeviceGaussians.from_host(scene, "cuda:0")


def _host(ds):
    return {f: getattr(ds, f).detach().double().cpu().numpy() if f != "type_spec"
            else ds.type_spec.cpu().numpy() for f in ds.FIELDS}


def test_densify_matches_oracle():
    import torch
    from paper_2512_02932_b200 import densify, optim
    _, _, ds = _scene(3000, seed=9)
    n = ds.count
    rng = np.random.default_rng(1)
    st = densify.DensifyStats(ds)
    obs = rng.integers(0, 5, size=n).astype(np.int32)
    acc = (rng.uniform(0, 2e-3, size=n) * obs).astype(np.float32)
    st.grad_accum.copy_(torch.from_numpy(acc))
    st.obs_count.copy_(torch.from_numpy(obs))
    with torch.no_grad():  # some Gaussians below the prune opacity
        ds.opacity_logit[::17] = -7.0
    opt = optim.Adam(ds)
    opt.exp_avg.normal_()
    opt.exp_avg_sq.uniform_()
    m_before, v_before = opt.exp_avg.clone(), opt.exp_avg_sq.clone()
    src = _host(ds)
    cfg = densify.DensifyConfig(grad_threshold=5e-4, split_scale_frac=0.05)
    out, rep = densify.densify(ds, st, cfg, optimizer=opt)
    ref, census, parent, new = od.densify(src, acc, obs, 5e-4, 0.005, 0.05 * ds.extent)
    assert (rep.kept, rep.pruned, rep.cloned, rep.split) == census
    assert rep.cloned > 0 and rep.split > 0 and rep.pruned > 0
    assert rep.n_after == n + rep.cloned + 2 * rep.split - rep.split - rep.pruned
    got = _host(out)
    for f in ds.FIELDS:
        np.testing.assert_allclose(got[f], ref[f].astype(got[f].dtype), rtol=2e-6, atol=2e-6,
                                   err_msg=f)
    # Adam moments: rows that continue a parent carry its moments, new rows are zero
    P = 11 + 3 * ds.sh_bases
    B = ds.sh_bases
    widths, offs_in, offs_out = (3, 3, 4, 1, 3 * B), [], []
    o_in = o_out = 0
    for w in widths:
        offs_in.append(o_in)
        offs_out.append(o_out)
        o_in += n * w
        o_out += rep.n_after * w
    mb, ma = m_before.cpu().numpy(), opt.exp_avg.cpu().numpy()
    for f, w in enumerate(widths):
        src_m = mb[offs_in[f]:offs_in[f] + n * w].reshape(n, w)
        dst_m = ma[offs_out[f]:offs_out[f] + rep.n_after * w].reshape(rep.n_after, w)
        np.testing.assert_array_equal(dst_m[~new], src_m[parent[~new]])
        assert np.all(dst_m[new] == 0)
    assert opt.exp_avg.numel() == rep.n_after * P and opt.scene is out
    assert st.count == rep.n_after and int(st.obs_count.sum()) == 0


def test_densify_spec_examples():
    import torch
    from paper_2512_02932_b200 import densify
    _, _, ds = _scene(64, seed=3)
    n = ds.count
    with torch.no_grad():
        ds.opacity_logit.fill_(0.0)
        ds.log_scale.fill_(-6.0)  # small
    st = densify.DensifyStats(ds)
    # no accumulator above threshold -> unchanged except pruning
    with torch.no_grad():
        ds.opacity_logit[5] = float(np.log(0.001 / 0.999))  # alpha = 0.001 < 0.005 -> pruned
    out, rep = densify.densify(ds, st)
    assert rep.n_after == n - 1 and rep.pruned == 1 and rep.cloned == rep.split == 0
    keep = np.ones(n, bool)
    keep[5] = False
    assert torch.equal(out.center, ds.center[torch.from_numpy(keep).cuda()])
    # one over-threshold large Gaussian -> count + 1, parent removed, two children
    _, _, ds = _scene(64, seed=3)
    with torch.no_grad():
        ds.opacity_logit.fill_(0.0)
        ds.log_scale.fill_(-6.0)
        ds.log_scale[7] = torch.tensor([0.0, -1.0, -2.0])
    st = densify.DensifyStats(ds)
    st.grad_accum[7] = 1.0
    st.obs_count[7] = 1
    out, rep = densify.densify(ds, st)
    assert rep.n_after == n + 1 and rep.split == 1
    c = ds.center[7].double().cpu().numpy()
    kids = out.center[7:9].double().cpu().numpy()
    assert not np.any(np.all(np.isclose(out.center.double().cpu().numpy(), c), axis=1))
    np.testing.assert_allclose(kids.mean(axis=0), c, atol=1e-6)
    np.testing.assert_allclose(np.linalg.norm(kids[0] - kids[1]), 1.0, rtol=1e-5)  # 2 x 0.5 sigma
    np.testing.assert_allclose(out.log_scale[7].cpu().numpy(), [-np.log(1.6), -1 - np.log(1.6),
                                                               -2 - np.log(1.6)], rtol=1e-6)


def test_train_step_accumulates_stats():
    import torch
    from paper_2512_02932_b200 import densify, freq, optim, raster
    from paper_2512_02932_b200.settings import RenderSettings
    _, cam, ds = _scene(2000, seed=11)
    imgs, _ = raster.rasterize(ds, cam, RenderSettings())
    gt = (imgs["color"] * 0.9).contiguous()
    st = densify.DensifyStats(ds)
    opt = optim.Adam(ds)
    for _ in range(3):
        optim.train_step(ds, cam, gt, opt, freq.LossWeights(), stats=st)
    obs = st.obs_count.cpu().numpy()
    acc = st.grad_accum.cpu().numpy()
    assert obs.max() == 3 and (obs > 0).sum() > 100
    assert np.all(acc[obs == 0] == 0) and np.all(acc >= 0) and acc[obs > 0].mean() > 0
    out, rep = densify.densify(ds, st, densify.DensifyConfig(grad_threshold=float(np.median(
        acc[obs > 0] / obs[obs > 0]))), optimizer=opt)
    assert rep.cloned + rep.split > 0
    res = optim.train_step(out, cam, gt, opt, freq.LossWeights(), stats=st)  # keeps training
    assert np.isfinite(res.losses.cpu().numpy()).all()
