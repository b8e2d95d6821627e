"""How many tile-list entries (splat, 16x16 tile) at config 2 have no
contributing pixel in their tile (an upper bound on what an exact tile-level
cull could remove), split by splat type.  Run on the GPU box."""
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
tx = (W + 15) // 16
off = torch.from_numpy(lg.offsets).cuda()
pos = torch.from_numpy(lg.position.astype(np.int64)).cuda()
cnt = off[1:] - off[:-1]
pix = torch.repeat_interleave(torch.arange(W * H, device="cuda"), cnt)
tile = (pix // W // 16) * tx + (pix % W) // 16
contrib = torch.unique(tile * (1 << 24) + pos)
to = torch.from_numpy(fr.tile_offsets).cuda()
ids = torch.from_numpy(fr.tile_ids.astype(np.int64)).cuda()
tl = torch.repeat_interleave(torch.arange(to.numel() - 1, device="cuda"), to[1:] - to[:-1])
listed = tl * (1 << 24) + ids
hit = torch.isin(listed, contrib)
typ = torch.from_numpy(fr.typ.astype(np.int64)).cuda()[ids]
for t, name in ((1, "3D"), (0, "2D")):
    m = typ == t
    print("%s: %d tile-list entries, %.1f%% with no contributing pixel in the tile"
          % (name, int(m.sum()), 100.0 * float((~hit[m]).sum()) / float(m.sum())))
print("all: K = %d, %.1f%% empty" % (ids.numel(), 100.0 * float((~hit).sum()) / ids.numel()))
