"""Distribution of the backward compositor's per-visit pixel counts at config 2:
for every (splat, 8 x 16 warp block) visit, n = the number of the block's
pixels the splat contributes to (from the blend log).  Also the fraction of
consecutive visits (in a warp's back-to-front order) that are pixel-disjoint
and both small -- the candidates for sharing one evaluation pass.  Run on the
GPU box:  python tools/visit_stats.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

W, H = 1920, 1080
scene, cam = synthetic_scene(1_000_000, W, H, 3, seed=0)
ds = DeviceGaussians.from_host(scene, "cuda:0")
imgs, fr = raster.rasterize(ds, cam, RenderSettings())
out = raster.RenderOutput(imgs["color"], imgs["depth"], imgs["transmittance"], imgs["alpha"],
                          imgs["normal"], fr, None)
lg = out.blend_log
off = torch.from_numpy(lg.offsets).cuda()
pos = torch.from_numpy(lg.position.astype(np.int64)).cuda()
cnt = off[1:] - off[:-1]
pix = torch.repeat_interleave(torch.arange(W * H, device="cuda"), cnt)
ix, iy = pix % W, pix // W
import os
if os.environ.get("BLOCK", "8x16") == "16x16":
    block = (iy // 16) * ((W + 15) // 16) + (ix // 16)
else:
    block = (iy // 16) * ((W + 15) // 16) * 2 + (ix // 16) * 2 + ((ix % 16) >= 8).long()
# (block, rank) visits; rank order within a block is the walk order reversed
key = block * (1 << 24) + pos
uk, n = torch.unique(key, return_counts=True)
h = torch.bincount(n, minlength=257).cpu().numpy()
tot = int(n.numel())
print("visits", tot, "pairs", int(n.sum()), "mean n", float(n.float().mean()))
for lo, hi in ((1, 4), (5, 8), (9, 16), (17, 32), (33, 64), (65, 128), (129, 256)):
    s = int(h[lo:hi + 1].sum())
    print("n in [%3d, %3d]: %6.2f%% of visits, %6.2f%% of pairs" % (lo, hi, 100.0 * s / tot,
          100.0 * float((np.arange(257)[lo:hi + 1] * h[lo:hi + 1]).sum()) / float(n.sum())))
passes = int(((n + 31) // 32).sum())
print("passes", passes, "lanes per pass", float(n.sum()) / passes)
# consecutive visits of one block, both n <= 16: pair candidates (ignoring disjointness)
ub = uk // (1 << 24)
same = ub[1:] == ub[:-1]
small = (n[1:] <= 16) & (n[:-1] <= 16)
print("consecutive same-block visits both n<=16: %.2f%%" % (100.0 * float((same & small).sum()) / tot))

# pairing candidates: consecutive visits of one block (walk order), both with
# <= 16 pixels, the same splat type and disjoint pixel sets
typ = torch.from_numpy(fr.typ.astype(np.int64)).cuda()  # by slot (rank)
lx = (ix % 8) if os.environ.get("BLOCK", "8x16") != "16x16" else (ix % 16)
ly = iy % 16
bit = (ly * 8 + lx) if os.environ.get("BLOCK", "8x16") != "16x16" else (ly * 16 + lx)
inv = torch.empty_like(key)
order = torch.argsort(key)
ks = key[order]
vid = torch.searchsorted(uk, ks)  # visit index of each (sorted) pair
b = bit[order]
lo_m = torch.zeros(uk.numel(), dtype=torch.int64, device="cuda")
hi_m = torch.zeros(uk.numel(), dtype=torch.int64, device="cuda")
one = torch.ones_like(b)
lo_m.index_put_((vid[b < 64],), torch.bitwise_left_shift(one[b < 64], b[b < 64]), accumulate=True)
hi_m.index_put_((vid[b >= 64],), torch.bitwise_left_shift(one[b >= 64], b[b >= 64] - 64), accumulate=True)
vt = typ[uk % (1 << 24)]
cand = same & small & (vt[1:] == vt[:-1]) & ((lo_m[1:] & lo_m[:-1]) == 0) & ((hi_m[1:] & hi_m[:-1]) == 0)
print("adjacent pairs: same block, both n<=16, same type, disjoint pixels: %.2f%% of visits"
      % (100.0 * float(cand.sum()) / tot))
