import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_02932_b200 import raster
from paper_2512_02932_b200.core import DeviceGaussians, GaussianSet
from paper_2512_02932_b200.synthetic import synthetic_scene
for n in (1000, 300_000, 1_000_000):
    scene, cam = synthetic_scene(n, 64, 48, 3, seed=0)
    hs = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit, scene.sh_coeffs, scene.type_spec)
    ds = DeviceGaussians.from_host(hs, fingerprint=True)
    a, b = ds.host_fingerprint, raster.scene_fingerprint(hs)
    print(n, a == b, a[:2])
    assert a == b
