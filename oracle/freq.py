"""CPU oracle for the training-step rows of SURVEY.md 8(f): the
frequency-decoupled loss stack, gradient surgery and the optimizer step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the parity checker for the
CUDA kernels in ``paper_2512_02932_b200/csrc/hgs_loss.cu`` and
``hgs_optim.cu``.  Only ``tests/`` and ``bench.py`` may import it.

A float64 numpy restatement -- not a copy -- of the reference algorithms
(paths relative to /root/reference/pkg/src/hybridsplat):

* ``dwt_level1`` / ``idwt_level1`` / ``dwt_adjoint`` -- freq/dwt.py:32-105,
  written in closed 2x2-block form (LL = (a+b+c+d)/2, ...);
* ``frequency_losses`` / ``frequency_loss_grads`` -- freq/dwt.py:108-137;
* ``ssim`` / ``ssim_grad`` -- freq/ssim.py:13-74, the zero-padded separable
  window as explicit shifted sums (no scipy);
* ``color_loss`` / ``color_loss_grad`` -- freq/ssim.py:77-94;
* ``combine_gradients`` -- freq/surgery.py:55-92;
* ``adam_step`` -- SPEC.md:424 ("first-order adaptive-moment method", 3DGS
  learning rates) in torch.optim.Adam's single-tensor arithmetic; the
  reference ships no optimizer code, so this row is pinned to torch's Adam
  (tests/golden/make_freq_golden.py) rather than to reference source.

Parity is pinned against ``tests/golden/freq.npz``, produced by running the
reference functions themselves (tests/golden/make_freq_golden.py).
"""

import numpy as np

WINDOW_SIZE = 11
WINDOW_SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def _edge_pad(img):
    """Replicate the last row / column when a size is odd (dwt.py:32-38)."""
    h, w = img.shape[:2]
    if h % 2:
        img = np.concatenate([img, img[-1:]], axis=0)
    if w % 2:
        img = np.concatenate([img, img[:, -1:]], axis=1)
    return img


def dwt_level1(image):
    """(LL, LH, HL, HH) of the orthonormal level-1 Haar transform.  With
    a = I[2i,2j], b = I[2i,2j+1], c = I[2i+1,2j], d = I[2i+1,2j+1]:
    LL = (a+b+c+d)/2, LH = (a+b-c-d)/2 (row high-pass), HL = (a-b+c-d)/2
    (column high-pass), HH = (a-b-c+d)/2 (dwt.py:55-74)."""
    p = _edge_pad(np.asarray(image, dtype=np.float64))
    a, b = p[0::2, 0::2], p[0::2, 1::2]
    c, d = p[1::2, 0::2], p[1::2, 1::2]
    return (0.5 * (a + b + c + d), 0.5 * (a + b - c - d), 0.5 * (a - b + c - d),
            0.5 * (a - b - c + d))


def _synth(LL, LH, HL, HH):
    """Padded-size synthesis: the transpose of the orthonormal analysis."""
    h2, w2 = LL.shape[:2]
    out = np.zeros((2 * h2, 2 * w2) + LL.shape[2:])
    out[0::2, 0::2] = 0.5 * (LL + LH + HL + HH)
    out[0::2, 1::2] = 0.5 * (LL + LH - HL - HH)
    out[1::2, 0::2] = 0.5 * (LL - LH + HL - HH)
    out[1::2, 1::2] = 0.5 * (LL - LH - HL + HH)
    return out


def idwt_level1(bands, shape):
    """Inverse, cropped to the original (H, W) (dwt.py:77-93)."""
    h, w = shape[:2]
    return _synth(*bands)[:h, :w]


def dwt_adjoint(bands, shape):
    """Adjoint on the original image space: synthesis, then the padded row /
    column folded back onto the edge (dwt.py:41-52, 96-105)."""
    h, w = shape[:2]
    g = _synth(*bands)
    if g.shape[0] != h:
        g[h - 1] += g[h]
        g = g[:h]
    if g.shape[1] != w:
        g[:, w - 1] += g[:, w]
        g = g[:, :w]
    return g


def frequency_losses(rendered, gt):
    """(L_low, L_high): MSE of the LL band, summed MSE of the detail bands."""
    br, bg = dwt_level1(rendered), dwt_level1(gt)
    l_low = float(np.mean((br[0] - bg[0]) ** 2))
    l_high = float(sum(np.mean((x - y) ** 2) for x, y in zip(br[1:], bg[1:])))
    return l_low, l_high


def frequency_loss_grads(rendered, gt):
    rendered = np.asarray(rendered, np.float64)
    br, bg = dwt_level1(rendered), dwt_level1(gt)
    size = br[0].size
    d = [2.0 * (x - y) / size for x, y in zip(br, bg)]
    z = np.zeros_like(d[0])
    g_low = dwt_adjoint((d[0], z, z, z), rendered.shape)
    g_high = dwt_adjoint((z, d[1], d[2], d[3]), rendered.shape)
    return g_low, g_high


def _window():
    x = np.arange(WINDOW_SIZE, dtype=np.float64) - WINDOW_SIZE // 2
    w = np.exp(-x * x / (2.0 * WINDOW_SIGMA ** 2))
    return w / w.sum()


def _blur(img):
    """Zero-padded 11-tap window along axis 0 then axis 1 (ssim.py:26-29)."""
    w = _window()
    r = WINDOW_SIZE // 2
    out = img
    for axis in (0, 1):
        n = out.shape[axis]
        pad = [(0, 0)] * out.ndim
        pad[axis] = (r, r)
        p = np.pad(out, pad)
        acc = np.zeros_like(out)
        for t in range(WINDOW_SIZE):
            acc += w[t] * np.take(p, np.arange(t, t + n), axis=axis)
        out = acc
    return out


def _moments(x, y):
    mx, my = _blur(x), _blur(y)
    return mx, my, _blur(x * x) - mx * mx, _blur(y * y) - my * my, _blur(x * y) - mx * my


def ssim(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    mx, my, sx, sy, sxy = _moments(x, y)
    return float(np.mean(((2 * mx * my + C1) * (2 * sxy + C2))
                         / ((mx * mx + my * my + C1) * (sx + sy + C2))))


def ssim_grad(x, y):
    """d mean(SSIM) / dx for fixed y (ssim.py:52-74)."""
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    mx, my, sx, sy, sxy = _moments(x, y)
    a1, a2 = 2 * mx * my + C1, 2 * sxy + C2
    b1, b2 = mx * mx + my * my + C1, sx + sy + C2
    d_mx = 2 * (my * a2 * b1 - mx * a1 * a2) / (b1 * b1 * b2)
    d_sx = -a1 * a2 / (b1 * b2 * b2)
    d_sxy = 2 * a1 / (b1 * b2)
    return (_blur(d_mx - 2 * mx * d_sx - my * d_sxy) + 2 * x * _blur(d_sx)
            + y * _blur(d_sxy)) / x.size


def color_loss(r, g, lam):
    r, g = np.asarray(r, np.float64), np.asarray(g, np.float64)
    l1 = float(np.mean(np.abs(r - g)))
    return l1 if lam == 0.0 else (1 - lam) * l1 + lam * (1 - ssim(r, g)) / 2


def color_loss_grad(r, g, lam):
    r, g = np.asarray(r, np.float64), np.asarray(g, np.float64)
    out = (1 - lam) * np.sign(r - g) / r.size
    if lam > 0.0:
        out = out - 0.5 * lam * ssim_grad(r, g)
    return out


def loss_stack(r, g, lam, lambda_low, lambda_high):
    """The (3, H, W, C) upstream gradient stack of one training view and the
    five loss values in hgs_image_losses order (include/hgs_train.h)."""
    gl, gh = frequency_loss_grads(r, g)
    stack = np.stack([color_loss_grad(r, g, lam), lambda_low * gl, lambda_high * gh])
    l_low, l_high = frequency_losses(r, g)
    l1 = float(np.mean(np.abs(np.asarray(r, np.float64) - g)))
    s = ssim(r, g)
    return stack, np.array([l1, s, l_low, l_high, color_loss(r, g, lam)])


def combine_gradients(g_color, g_low, g_high, type_spec, mode="projection"):
    """(N, P) rows -> (total, n_conflicts) (surgery.py:55-92)."""
    gc, gl, gh = (np.array(a, np.float64) for a in (g_color, g_low, g_high))
    t = np.asarray(type_spec)
    dot = (gl * gh).sum(axis=1)
    conf = dot < 0.0
    n = int(conf.sum())
    if mode == "naive" or n == 0:
        return gc + gl + gh, n
    flat, volu = conf & (t == 0), conf & (t == 1)
    if mode == "mask":
        gh[flat] = 0.0
        gl[volu] = 0.0
    else:
        nl, nh = (gl * gl).sum(axis=1), (gh * gh).sum(axis=1)
        f = flat & (nl > 0)
        v = volu & (nh > 0)
        gh[f] = gh[f] - (dot[f] / nl[f])[:, None] * gl[f]
        gl[v] = gl[v] - (dot[v] / nh[v])[:, None] * gh[v]
    return gc + gl + gh, n


def adam_step(param, grad, m, v, lr, step, beta1=0.9, beta2=0.999, eps=1e-15):
    """One Adam update (torch.optim.Adam, single-tensor path), float64."""
    m = m + (1 - beta1) * (grad - m)
    v = beta2 * v + (1 - beta2) * grad * grad
    bc1, bc2 = 1 - beta1 ** step, 1 - beta2 ** step
    denom = np.sqrt(v) / np.sqrt(bc2) + eps
    return param - (lr / bc1) * m / denom, m, v


def renormalize_rotations(q):
    """core/types.py:136-142: |q| <= 1e-8 -> identity, else q / |q|."""
    q = np.array(q, np.float64)
    nrm = np.linalg.norm(q, axis=1, keepdims=True)
    bad = nrm[:, 0] <= 1e-8
    q[bad] = (1.0, 0.0, 0.0, 0.0)
    nrm[bad] = 1.0
    return q / nrm
