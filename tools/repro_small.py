import sys
sys.path.insert(0, ".")
import torch
from paper_2512_02932_b200 import raster
from paper_2512_02932_b200.core import DeviceGaussians
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_scene
scene, cam = synthetic_scene(2000, 64, 48, 3, seed=1)
ds = DeviceGaussians.from_host(scene, "cuda:0")
imgs, frame = raster.rasterize(ds, cam, RenderSettings())
torch.cuda.synchronize()
print("ok", frame.count, frame.pair_count, float(imgs["color"].sum()))
