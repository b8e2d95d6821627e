import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2512_02932_b200 import raster
from paper_2512_02932_b200.core import DeviceGaussians
from paper_2512_02932_b200.settings import RenderSettings
from paper_2512_02932_b200.synthetic import synthetic_scene
w, h = 37, 23
scene, cam = synthetic_scene(1500, w, h, 2, seed=w * 31 + h)
st = RenderSettings(background=(0.3, 0.2, 0.1))
ds = DeviceGaussians.from_host(scene, "cuda:0")
out = raster.render(ds, cam, st)
ref = oracle.render(scene, cam, st)
err = np.abs(out.color.double().cpu().numpy() - ref["color"]).max(axis=2)
off, pos, al, u, v = oracle.blend_log(ref)
gl = out.blend_log
fr = out.frame.export()
bad = np.argwhere(err > 2e-5)
print("pixels > 2e-5:", len(bad))
for iy, ix in bad[:6]:
    p = iy * w + ix
    ro = set(pos[off[p]:off[p + 1]].tolist())
    go = set(gl.position[gl.offsets[p]:gl.offsets[p + 1]].tolist())
    print("px", ix, iy, "err %.2e" % err[iy, ix], "only_oracle", sorted(ro - go)[:5], "only_gpu", sorted(go - ro)[:5])
    for k in sorted(ro ^ go)[:3]:
        print("   splat slot", k, "typ", int(fr["typ"][k]), "bbox", fr["bbox"][k], "ctr", fr["center2d"][k],
              "alpha_eff %.4f" % fr["alpha_eff"][k], "mrow", np.round(fr["mrow"][k], 3).tolist())
