"""Forward walk iterations at config 2 (a measurement build with
-DHGS_DIAG_ITER=1): diag[11] = (splat, 8x4 block) iterations, diag[15] = those
in which no pixel of the block contributed.  Run on the GPU box with
HGS_LIB=tools/var/diag/libhgs.so."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _lib, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
ds = DeviceGaussians.from_host(scene, "cuda:0")
_, fr = raster.rasterize(ds, cam, RenderSettings(), _lib.HGS_FLAG_COUNT)
s = _lib.frame_stats(fr)
print("iterations", int(s[11]), "empty", int(s[15]), "frac %.3f" % (s[15] / max(s[11], 1)),
      "evals 3D", int(s[2]), "2D", int(s[3]), "contrib 3D", int(s[4]), "2D", int(s[5]))
