"""CPU: the densify oracle (oracle/densify.py) on the SPEC's examples
 and the count invariant."""

import numpy as np

from oracle import densify as od


def _scene(n, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    return {"center": rng.normal(size=(n, 3)), "log_scale": np.full((n, 3), -6.0),
            "rotation": q / np.linalg.norm(q, axis=1, keepdims=True),
            "opacity_logit": np.zeros(n), "sh_coeffs": rng.normal(size=(n, 3, 4)),
            "type_spec": (rng.uniform(size=n) < 0.5).astype(np.uint8)}


def test_spec_examples():
    f = _scene(10)
    acc, obs = np.zeros(10), np.zeros(10, np.int32)
    out, census, parent, new = od.densify(f, acc, obs, 2e-4, 0.005, 0.01)
    assert census == (10, 0, 0, 0) and np.array_equal(out["center"], f["center"])  # unchanged
    f["opacity_logit"][3] = np.log(0.001 / 0.999)  # alpha 0.001 -> pruned
    out, census, parent, _ = od.densify(f, acc, obs, 2e-4, 0.005, 0.01)
    assert census[1] == 1 and out["center"].shape[0] == 9 and 3 not in parent
    f = _scene(10)
    f["log_scale"][4] = (0.0, -1.0, -2.0)
    f["type_spec"][4] = 1
    acc[4], obs[4] = 1.0, 1
    out, census, parent, new = od.densify(f, acc, obs, 2e-4, 0.005, 0.01)
    assert census[3] == 1 and out["center"].shape[0] == 11  # count + 1, two children
    kids = out["center"][parent == 4]
    assert kids.shape == (2, 3) and np.allclose(kids.mean(axis=0), f["center"][4])
    assert np.isclose(np.linalg.norm(kids[0] - kids[1]), 1.0)


def test_count_invariant_random():
    rng = np.random.default_rng(5)
    for seed in range(5):
        f = _scene(200, seed)
        f["log_scale"] = rng.uniform(-6, -1, size=(200, 3))
        f["opacity_logit"] = rng.normal(-3, 2, size=200)
        obs = rng.integers(0, 4, size=200).astype(np.int32)
        acc = rng.uniform(0, 1e-3, size=200) * obs
        out, (k, p, c, s), parent, new = od.densify(f, acc, obs, 2e-4, 0.005, 0.05)
        assert k + p + c + s == 200
        assert out["center"].shape[0] == 200 + c + 2 * s - s - p
        assert new.sum() == c + 2 * s
