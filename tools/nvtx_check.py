"""Two forward + backward calls on a small scene: the workload for checking
the library's NVTX ranges under `ncu --nvtx --nvtx-include ...` (only the
kernels enqueued inside the named range are profiled).  Run on the GPU box."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import grad, raster  # noqa: E402
from paper_2512_02932_b200.core import DeviceGaussians  # noqa: E402
from paper_2512_02932_b200.settings import RenderSettings  # noqa: E402
from paper_2512_02932_b200.synthetic import synthetic_scene  # noqa: E402

scene, cam = synthetic_scene(20000, 320, 240, 3, seed=1)
ds = DeviceGaussians.from_host(scene, torch.device("cuda", 0))
pg = torch.randn((1, 240, 320, 3), device="cuda")
for _ in range(2):
    imgs, frame = raster.rasterize(ds, cam, RenderSettings(), 0)
    grad.backward_device(frame, pg)
torch.cuda.synchronize()
print("ok")
