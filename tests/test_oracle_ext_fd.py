"""FD pin of the oracle's extension semantics (CPU, no GPU).

The reference has no alpha / normal image and no depth / normal / alpha
upstream gradient (grad/backward.py:37-50 takes colour gradients only), so the
oracle's ``backward(..., depth_grad=, normal_grad=, alpha_grad=)`` is pinned
here the only way it can be: against central differences of the oracle's own
float64 forward images.  The GPU path is then compared
with this FD-pinned oracle (tests/test_gpu_ext_grads.py).

Protocol as the reference's own FD checker (grad/findiff.py:78-133): central
differences, parameters whose perturbation changes the depth order are
excluded, >= 99% within 1e-3 relative (floor 1e-2 absolute).
"""

import numpy as np
import pytest

from paper_2512_02932_b200.core import GaussianSet
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_camera


def _small_scene(rng, cam, n):
    z = rng.uniform(2, 4, n)
    px = rng.uniform(2, cam.width - 2, (n, 2))
    c = np.stack([(px[:, 0] - cam.cx) * z / cam.fx, (px[:, 1] - cam.cy) * z / cam.fy, z], 1)
    ls = np.log(rng.uniform(1.5, 4.0, (n, 3)) * z[:, None] / cam.fx)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return GaussianSet(c, ls, q, rng.normal(0, 1, n), rng.normal(0, .3, (n, 3, 4)),
                       (rng.random(n) < .5).astype(np.uint8))


def _fields(s):
    n = s.count
    return [s.center, s.log_scale, s.rotation, s.opacity_logit[:, None], s.sh_coeffs.reshape(n, -1)]


def ext_fd_check(oracle, scene, cam, st, weights, eps=1e-5, tol=1e-3):
    """(ok, total) of analytic oracle gradients of
    L = sum wc*color + sum wd*depth + sum wn*normal + sum wa*alpha
    against central differences of the oracle forward."""
    wc, wd, wn, wa = weights

    def loss(s_):
        r = oracle.render(s_, cam, st)
        return float((wc * r["color"]).sum() + (wd * r["depth"]).sum()
                     + (wn * r["normal"]).sum() + (wa * r["alpha"]).sum())

    g, _, _ = oracle.backward(scene, cam, st, wc, depth_grad=wd, normal_grad=wn, alpha_grad=wa)
    an = g[0]
    n, P = an.shape
    base_idx = oracle.build_frame(scene, cam, st).idx
    offs = [0, 3, 6, 10, 11]
    ok = total = 0
    for gi in range(n):
        for slot in range(P):
            fi = max(i for i, o in enumerate(offs) if o <= slot)
            col = slot - offs[fi]

            def perturbed(d):
                s2 = scene.copy()
                _fields(s2)[fi][gi, col] += d
                return s2
            sp, sm = perturbed(eps), perturbed(-eps)
            if not (np.array_equal(oracle.build_frame(sp, cam, st).idx, base_idx)
                    and np.array_equal(oracle.build_frame(sm, cam, st).idx, base_idx)):
                continue
            fd = (loss(sp) - loss(sm)) / (2 * eps)
            total += 1
            if abs(an[gi, slot] - fd) <= tol * max(abs(fd), 1e-2):
                ok += 1
    return ok, total


@pytest.mark.parametrize("which", ["depth", "normal", "alpha", "all"])
def test_oracle_extension_gradients_match_fd(which):
    import oracle
    rng = np.random.default_rng({"depth": 1, "normal": 2, "alpha": 3, "all": 4}[which])
    cam = synthetic_camera(16, 16)
    st = RenderSettings(background=(0.1, 0.2, 0.3))
    ok = total = 0
    for _ in range(6):
        sc = _small_scene(rng, cam, int(rng.integers(2, 7)))
        z = np.zeros
        w = [z((16, 16, 3)), z((16, 16)), z((16, 16, 3)), z((16, 16))]
        if which in ("depth", "all"):
            w[1] = rng.normal(size=(16, 16))
        if which in ("normal", "all"):
            w[2] = rng.normal(size=(16, 16, 3))
        if which in ("alpha", "all"):
            w[3] = rng.normal(size=(16, 16))
        if which == "all":
            w[0] = rng.normal(size=(16, 16, 3))
        a, t = ext_fd_check(oracle, sc, cam, st, w)
        ok += a
        total += t
    assert total > 150
    assert ok / total >= 0.99, (ok, total)
