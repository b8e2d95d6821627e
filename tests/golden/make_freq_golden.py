"""Generate tests/golden/freq.npz by running the REFERENCE loss stack and
gradient surgery (hybridsplat.freq) and torch.optim.Adam.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_freq_golden.py

Pins oracle/freq.py (tests/test_freq_oracle.py) and, on the GPU box where the
reference is absent, the CUDA loss / surgery / optimizer kernels
(tests/test_gpu_train.py).  Inputs are float32-representable and stored as
float32; reference outputs are float64.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import importlib  # noqa: E402

# the reference modules (hybridsplat.freq re-exports functions that shadow them)
rdwt = importlib.import_module("hybridsplat.freq.dwt")
rssim = importlib.import_module("hybridsplat.freq.ssim")
rsurg = importlib.import_module("hybridsplat.freq.surgery")


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(2512)
    out = {}
    # images: even, odd x odd, odd x even, grayscale
    shapes = {"even": (24, 40, 3), "odd": (19, 27, 3), "mixed": (17, 32, 3), "gray": (22, 15)}
    for tag, shp in shapes.items():
        r = f32(rng.uniform(0, 1, size=shp))
        g = f32(np.clip(r + rng.normal(0, 0.15, size=shp), 0, 1))
        out["%s_r" % tag] = r.astype(np.float32)
        out["%s_g" % tag] = g.astype(np.float32)
        b = rdwt.dwt_level1(r)
        for nm in ("LL", "LH", "HL", "HH"):
            out["%s_%s" % (tag, nm)] = getattr(b, nm)
        out["%s_idwt" % tag] = rdwt.idwt_level1(b)
        # adjoint applied to random bands
        rb = [f32(rng.normal(size=b.LL.shape)) for _ in range(4)]
        for nm, x in zip(("LL", "LH", "HL", "HH"), rb):
            out["%s_adjin_%s" % (tag, nm)] = x.astype(np.float32)
        out["%s_adjoint" % tag] = rdwt.dwt_adjoint(rdwt.DwtBands(*rb, r.shape))
        out["%s_freq_losses" % tag] = np.array(rdwt.frequency_losses(r, g))
        gl, gh = rdwt.frequency_loss_grads(r, g)
        out["%s_g_low" % tag] = gl
        out["%s_g_high" % tag] = gh
        out["%s_ssim" % tag] = np.array(rssim.ssim(r, g))
        out["%s_ssim_grad" % tag] = rssim.ssim_grad(r, g)
        for lam in (0.0, 0.2, 1.0):
            k = "%s_color_%g" % (tag, lam)
            out[k + "_loss"] = np.array(rssim.color_loss(r, g, lam))
            out[k + "_grad"] = rssim.color_loss_grad(r, g, lam)

    # gradient surgery: (N, P) rows, P = 59 (SH degree 3), mixed conflicts
    n, p = 500, 59
    gc = f32(rng.normal(size=(n, p)))
    gl = f32(rng.normal(size=(n, p)))
    gh = f32(rng.normal(size=(n, p)) * 0.5 - 0.3 * gl)
    gl[:7] = 0.0  # zero-norm preserved vectors skip the projection
    gh[7:14] = 0.0
    t = (rng.uniform(size=n) < 0.5).astype(np.uint8)
    out["surg_gc"], out["surg_gl"], out["surg_gh"] = (x.astype(np.float32) for x in (gc, gl, gh))
    out["surg_type"] = t
    for mode in rsurg.MODES:
        tot, nconf = rsurg.combine_gradients(gc, gl, gh, t, mode)
        out["surg_%s" % mode] = tot
        out["surg_%s_n" % mode] = np.array(nconf)

    # optimizer pin: torch.optim.Adam (the optimizer of 3DGS) over 5 steps
    import torch
    p0 = f32(rng.normal(size=(64, 7)))
    grads = [f32(rng.normal(size=(64, 7))) for _ in range(5)]
    w = torch.tensor(p0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([w], lr=1e-2, betas=(0.9, 0.999), eps=1e-15, foreach=False)
    for gr in grads:
        opt.zero_grad()
        w.grad = torch.tensor(gr, dtype=torch.float64)
        opt.step()
    out["adam_p0"] = p0.astype(np.float32)
    out["adam_grads"] = np.stack(grads).astype(np.float32)
    out["adam_p5"] = w.detach().numpy()
    st = opt.state[w]
    out["adam_m5"] = st["exp_avg"].numpy()
    out["adam_v5"] = st["exp_avg_sq"].numpy()
    np.savez_compressed(os.path.join(HERE, "freq.npz"), **out)
    print("wrote freq.npz with %d arrays" % len(out))


if __name__ == "__main__":
    main()
