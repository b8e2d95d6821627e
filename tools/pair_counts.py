"""Tile/splat pairs of the compositor (tile-level culled) vs the reference bbox lists.  GPU box."""
import sys
sys.path.insert(0, ".")
from paper_2512_02932_b200 import raster
from paper_2512_02932_b200.core import DeviceGaussians
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_scene
for n, w, h in ((1_000_000, 1920, 1080), (300_000, 800, 600)):
    scene, cam = synthetic_scene(n, w, h, 3, seed=0)
    ds = DeviceGaussians.from_host(scene, "cuda:0")
    _, fr = raster.rasterize(ds, cam, RenderSettings())
    print(n, "compositor pairs", fr.pair_count, "bbox pairs", fr.export()["tile_ids"].size)
