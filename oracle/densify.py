"""CPU oracle for adaptive density control.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The reference ships no
densify code -- only the statistics fields and keep / append / reset_stats
helpers of GaussianSet (core/types.py:48-49, 110-130) -- so this restates the
SPEC's rules exactly as include/hgs_train.h defines
them ("parity unpinned": there are no reference outputs to pin against; the
SPEC examples SPEC.md:417-419 are checked in tests/test_gpu_densify.py):

  prune:  sigmoid(opacity_logit) < prune_opacity
  grow:   grad_accum / obs_count > grad_threshold (obs 0 -> 0)
  split:  grow and max scale > split_scale (in-plane axes for 2D surfels):
          two children at +-0.5 sigma along the major axis, log_scale - ln 1.6
  clone:  grow otherwise: parent + copy
  order:  survivors in index order, each followed by its second row.
"""

import numpy as np


def quat_to_matrix(q):
    q = np.asarray(q, np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
                    axis=1).reshape(-1, 3, 3)


def densify(f, grad_accum, obs_count, grad_threshold, prune_opacity, split_scale):
    """f: dict of float64 arrays center, log_scale, rotation, opacity_logit,
    sh_coeffs, type_spec.  Returns (new dict, census (kept, pruned, cloned,
    split), parent index of every output row, is_new flag per row)."""
    n = f["center"].shape[0]
    alpha = 1.0 / (1.0 + np.exp(-f["opacity_logit"]))
    prune = alpha < prune_opacity
    obs = np.asarray(obs_count)
    avg = np.where(obs > 0, np.asarray(grad_accum, np.float64) / np.maximum(obs, 1), 0.0)
    grow = ~prune & (avg > grad_threshold)
    ls = f["log_scale"]
    is3d = f["type_spec"] == 1
    lmax = np.where(is3d, ls.max(axis=1), ls[:, :2].max(axis=1))
    split = grow & (lmax > np.log(split_scale))
    clone = grow & ~split
    keep = ~prune & ~grow
    rows, parent, new = {k: [] for k in f}, [], []
    R = quat_to_matrix(f["rotation"])
    for i in range(n):
        if prune[i]:
            continue
        if keep[i] or clone[i]:
            reps = 1 if keep[i] else 2
            for r in range(reps):
                for k in f:
                    rows[k].append(f[k][i])
                parent.append(i)
                new.append(r == 1)
            continue
        ax = 1 if ls[i, 1] > ls[i, 0] else 0
        if is3d[i] and ls[i, 2] > ls[i, ax]:
            ax = 2
        d = 0.5 * np.exp(ls[i, ax]) * R[i, :, ax]
        for sg in (1.0, -1.0):
            for k in f:
                rows[k].append(f[k][i])
            rows["center"][-1] = f["center"][i] + sg * d
            rows["log_scale"][-1] = ls[i] - np.log(1.6)
            parent.append(i)
            new.append(True)
    out = {k: (np.array(v) if v else np.zeros((0,) + f[k].shape[1:], f[k].dtype)) for k, v in rows.items()}
    census = (int(keep.sum()), int(prune.sum()), int(clone.sum()), int(split.sum()))
    return out, census, np.array(parent, np.int64), np.array(new, bool)
