"""Pin the CPU oracle (oracle/hgs_oracle.c) to golden vectors produced by the
reference itself (tests/golden/make_golden.py) and to the SPEC's known-answer
examples.  CPU only."""

import numpy as np
import pytest

import oracle
from _fixtures import SCENES, grad_rel_err, load
from paper_2512_02932_b200.core import GaussianSet
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_camera

FRAME_EXACT = ("idx", "typ", "bbox", "tile_offsets", "tile_ids")
FRAME_FLOAT = ("depth", "center2d", "cov2d", "conic", "mrow", "alpha", "alpha_eff", "color",
               "radius")


@pytest.mark.parametrize("name", SCENES)
def test_frame_matches_reference(name):
    scene, cam, st, d = load(name)
    f = oracle.build_frame(scene, cam, st)
    for k in FRAME_EXACT:
        assert np.array_equal(getattr(f, k), d["f_" + k]), k
    for k in FRAME_FLOAT:
        np.testing.assert_allclose(getattr(f, k), d["f_" + k], rtol=1e-9, atol=1e-11, err_msg=k)


@pytest.mark.parametrize("name", SCENES)
def test_render_matches_reference(name):
    scene, cam, st, d = load(name)
    out = oracle.render(scene, cam, st)
    for k in ("color", "depth", "transmittance"):
        np.testing.assert_allclose(out[k], d[k], rtol=0, atol=1e-12, err_msg=k)
    if "log_offsets" in d:
        off, pos, al, u, v = oracle.blend_log(out)
        assert np.array_equal(off, d["log_offsets"])
        assert np.array_equal(pos, d["log_pos"])
        np.testing.assert_allclose(al, d["log_alpha"], atol=1e-13)
        np.testing.assert_allclose(u, d["log_u"], atol=1e-9, rtol=1e-12)
        np.testing.assert_allclose(v, d["log_v"], atol=1e-9, rtol=1e-12)
    else:
        assert np.array_equal(out["counts"].reshape(-1), d["log_counts"])
    if "naive_color" in d:
        nv = oracle.render(scene, cam, st, naive=True)
        np.testing.assert_allclose(nv["color"], d["naive_color"], atol=1e-12)
        np.testing.assert_allclose(nv["transmittance"], d["naive_transmittance"], atol=1e-12)


def test_raw_f64_fixture_discriminates_float32_rounding():
    """The raw_f64 fixture is only passed by a float64-faithful path: the
    float32 rounding of its inputs changes the depth order and tile lists."""
    from paper_2512_02932_b200.synthetic import f32_exact
    scene, cam, st, d = load("raw_f64")
    s2 = scene.copy()
    for a in (s2.center, s2.log_scale, s2.rotation, s2.opacity_logit):
        a[:] = f32_exact(a)
    f = oracle.build_frame(s2, cam, st)
    assert not np.array_equal(f.idx, d["f_idx"])
    assert not np.array_equal(f.tile_ids, d["f_tile_ids"])


@pytest.mark.parametrize("name", SCENES)
def test_backward_matches_reference(name):
    scene, cam, st, d = load(name)
    pg = d["pixel_grad"].astype(np.float64)
    grads, touched, _ = oracle.backward(scene, cam, st, pg)
    assert np.array_equal(touched, d["touched"])
    B = scene.sh_coeffs.shape[2]
    for kg in range(pg.shape[0]):
        err = grad_rel_err(grads[kg], d["grads"][kg], B)
        assert max(err.values()) < 1e-10, err


@pytest.mark.parametrize("name", ["exchange", "exchange_f64"])
def test_exchange_matches_reference(name):
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz"))
    ls, rot, ty, rep = oracle.exchange_pass(z["in_log_scale"], z["in_rotation"], z["in_type"])
    assert np.array_equal(ty, z["out_type"])
    np.testing.assert_allclose(ls, z["out_log_scale"], atol=1e-14)
    np.testing.assert_allclose(rot, z["out_rotation"], atol=1e-14)
    np.testing.assert_allclose(rep["eranks"], z["eranks"], rtol=1e-14)
    assert [rep["n_3d_to_2d"], rep["n_2d_to_3d"], rep["n_2d"], rep["n_3d"]] == list(z["counts"])
    assert np.array_equal(rep["erank_hist"], z["hist"])


# ---- SPEC known-answer examples (SPEC.md; verified on the reference)

def _one(center, ls, q, logit, rgb_band0, typ, B=1):
    sh = np.zeros((len(center), 3, B))
    sh[:, :, 0] = (np.asarray(rgb_band0) - 0.5) / 0.28209479177387814
    return GaussianSet(np.asarray(center, float), np.asarray(ls, float), np.asarray(q, float),
                       np.asarray(logit, float), sh, np.asarray(typ, np.uint8))


def test_two_splat_blend_known_answer():
    """alpha 0.6 red in front of alpha 0.5 blue -> (0.6, 0, 0.2)."""
    cam = synthetic_camera(16, 16)
    big = np.log(50.0)  # huge 3D Gaussians: d ~ 0 at the centre pixel
    logit = lambda a: np.log(a / (1 - a))  # noqa: E731
    ctr = [[0.0, 0.0, 2.0], [0.0, 0.0, 3.0]]
    sc = _one(ctr, [[big] * 3] * 2, [[1, 0, 0, 0]] * 2, [logit(0.6), logit(0.5)],
              [[1, 0, 0], [0, 0, 1]], [1, 1])
    out = oracle.render(sc, cam, RenderSettings())
    np.testing.assert_allclose(out["color"][8, 8], [0.6, 0.0, 0.2], atol=2e-4)
    np.testing.assert_allclose(out["transmittance"][8, 8], 0.2, atol=2e-4)


def test_erank_and_reparam_known_answers():
    """erank(1,1,1)=3, erank(1,1,2.6)~2.005; reparam
    s=(3,.5,2) -> (2,3,.5), q = (.5,-.5,-.5,-.5)."""
    ls = np.log(np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 2.6], [3.0, 0.5, 2.0]]))
    rot = np.array([[1.0, 0, 0, 0]] * 3)
    ty = np.array([1, 1, 1], np.uint8)
    ls2, rot2, ty2, rep = oracle.exchange_pass(ls, rot, ty, theta_e=2.05)
    assert abs(rep["eranks"][0] - 3.0) < 1e-12
    assert 1.99 <= rep["eranks"][1] <= 2.02
    np.testing.assert_allclose(np.exp(ls2[2]), [2.0, 3.0, 0.5], rtol=1e-14)
    np.testing.assert_allclose(rot2[2], [0.5, -0.5, -0.5, -0.5], atol=1e-14)
    assert ty2[2] == 0


def test_modulation_known_answer():
    """s_z = 2.1: alpha* = alpha * e^{-2.1} ~ 0.1225 alpha."""
    cam = synthetic_camera(16, 16)
    sc = _one([[0.0, 0.0, 2.0]], [[np.log(50.0), np.log(50.0), np.log(2.1)]], [[1, 0, 0, 0]],
              [0.0], [[1, 1, 1]], [0])
    f = oracle.build_frame(sc, cam, RenderSettings())
    assert abs(f.alpha_eff[0] / f.alpha[0] - np.exp(-2.1)) < 1e-9
