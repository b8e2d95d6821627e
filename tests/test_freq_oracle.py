"""CPU: the loss-stack / surgery / optimizer oracle (oracle/freq.py) against
fixtures produced by the reference itself (tests/golden/make_freq_golden.py),
plus the SPEC's known-answer examples."""

import os

import numpy as np
import pytest

from oracle import freq as of

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "freq.npz")
TAGS = ("even", "odd", "mixed", "gray")


@pytest.fixture(scope="module")
def gold():
    z = np.load(GOLD)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("tag", TAGS)
def test_dwt_matches_reference(gold, tag):
    r = gold[tag + "_r"].astype(np.float64)
    bands = of.dwt_level1(r)
    for nm, b in zip(("LL", "LH", "HL", "HH"), bands):
        np.testing.assert_allclose(b, gold["%s_%s" % (tag, nm)], rtol=0, atol=1e-14)
    np.testing.assert_allclose(of.idwt_level1(bands, r.shape), gold[tag + "_idwt"], atol=1e-14)
    np.testing.assert_allclose(of.idwt_level1(bands, r.shape), r, atol=1e-14)  # perfect reconstruction
    adj_in = [gold["%s_adjin_%s" % (tag, nm)].astype(np.float64) for nm in ("LL", "LH", "HL", "HH")]
    np.testing.assert_allclose(of.dwt_adjoint(adj_in, r.shape), gold[tag + "_adjoint"], atol=1e-14)


@pytest.mark.parametrize("tag", TAGS)
def test_losses_and_grads_match_reference(gold, tag):
    r, g = gold[tag + "_r"].astype(np.float64), gold[tag + "_g"].astype(np.float64)
    np.testing.assert_allclose(of.frequency_losses(r, g), gold[tag + "_freq_losses"], rtol=1e-12)
    gl, gh = of.frequency_loss_grads(r, g)
    np.testing.assert_allclose(gl, gold[tag + "_g_low"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(gh, gold[tag + "_g_high"], rtol=0, atol=1e-15)
    assert abs(of.ssim(r, g) - float(gold[tag + "_ssim"])) < 1e-12
    np.testing.assert_allclose(of.ssim_grad(r, g), gold[tag + "_ssim_grad"], rtol=1e-9, atol=1e-15)
    for lam in (0.0, 0.2, 1.0):
        k = "%s_color_%g" % (tag, lam)
        assert abs(of.color_loss(r, g, lam) - float(gold[k + "_loss"])) < 1e-12
        np.testing.assert_allclose(of.color_loss_grad(r, g, lam), gold[k + "_grad"], rtol=1e-9,
                                   atol=1e-15)


@pytest.mark.parametrize("mode", ("projection", "naive", "mask"))
def test_surgery_matches_reference(gold, mode):
    args = [gold[k].astype(np.float64) for k in ("surg_gc", "surg_gl", "surg_gh")]
    tot, n = of.combine_gradients(*args, gold["surg_type"], mode)
    assert n == int(gold["surg_%s_n" % mode]) and n > 0
    np.testing.assert_allclose(tot, gold["surg_" + mode], rtol=1e-12, atol=1e-12)


def test_adam_matches_torch(gold):
    p = gold["adam_p0"].astype(np.float64)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for t, gr in enumerate(gold["adam_grads"].astype(np.float64), start=1):
        p, m, v = of.adam_step(p, gr, m, v, 1e-2, t)
    np.testing.assert_allclose(p, gold["adam_p5"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(m, gold["adam_m5"], rtol=1e-12)
    np.testing.assert_allclose(v, gold["adam_v5"], rtol=1e-12)


def test_spec_examples():
    # constant c -> LL = 2c, details 0; checkerboard -> HH = 2
    ll, lh, hl, hh = of.dwt_level1(np.full((4, 4), 0.25))
    assert np.allclose(ll, 0.5) and np.allclose(lh, 0) and np.allclose(hl, 0) and np.allclose(hh, 0)
    ll, lh, hl, hh = of.dwt_level1(np.array([[1.0, -1.0], [-1.0, 1.0]]))
    assert np.allclose([ll, lh, hl], 0) and np.allclose(hh, 2.0)
    # rendered = gt + 0.1 -> L_low = 0.04, L_high = 0
    g = np.random.default_rng(0).uniform(size=(8, 6, 3))
    lo, hi = of.frequency_losses(g + 0.1, g)
    assert abs(lo - 0.04) < 1e-12 and abs(hi) < 1e-20
    # identity -> 0; lam = 0, +0.1 -> 0.1
    assert abs(of.color_loss(g, g, 0.2)) < 1e-12
    assert abs(of.color_loss(g + 0.1, g, 0.0) - 0.1) < 1e-12
    # projection example -> (1, 1); mask -> (1, 0)
    gc, gl, gh = np.zeros((1, 2)), np.array([[1.0, 0.0]]), np.array([[-1.0, 1.0]])
    tot, n = of.combine_gradients(gc, gl, gh, np.array([0]), "projection")
    assert n == 1 and np.allclose(tot, [[1.0, 1.0]])
    tot, _ = of.combine_gradients(gc, gl, gh, np.array([0]), "mask")
    assert np.allclose(tot, [[1.0, 0.0]])
