import sys, time, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio, _lib
from paper_2512_02932_b200.core import DeviceGaussians, GaussianSet
from paper_2512_02932_b200.synthetic import synthetic_scene
scene, cam = synthetic_scene(1_000_000, 1920, 1080, 3, seed=0)
def t(f, reps=5):
    f(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 2)
c = torch.from_numpy(np.ascontiguousarray(scene.center)).reshape(-1)
pin = torch.empty(c.numel(), dtype=torch.float64, pin_memory=True)
print("center f64 copy_ into pinned", c.numel()*8/1e6, "MB", t(lambda: pin.copy_(c)))
sh = torch.from_numpy(np.ascontiguousarray(scene.sh_coeffs)).reshape(-1)
pin32 = torch.empty(sh.numel(), dtype=torch.float32, pin_memory=True)
print("sh narrow", t(lambda: _hostio._convert("hgs_host_narrow", sh, pin32)))
d32 = torch.empty(sh.numel(), dtype=torch.float32, device="cuda")
print("sh DMA 192MB", t(lambda: d32.copy_(pin32, non_blocking=True)))
print("upload()", t(lambda: _hostio.upload([(scene.center, torch.float64), (scene.log_scale, torch.float64), (scene.rotation, torch.float64), (scene.opacity_logit, torch.float64), (scene.sh_coeffs, torch.float32), (scene.type_spec, torch.uint8)], torch.device("cuda:0"), tag="x")))
print("from_host", t(lambda: DeviceGaussians.from_host(scene)))
print("upload sh only", t(lambda: _hostio.upload([(scene.sh_coeffs, torch.float32)], torch.device("cuda:0"), tag="y")))
print("upload geom only", t(lambda: _hostio.upload([(scene.center, torch.float64), (scene.log_scale, torch.float64), (scene.rotation, torch.float64), (scene.opacity_logit, torch.float64)], torch.device("cuda:0"), tag="z")))
print(type(scene.sh_coeffs), scene.sh_coeffs.dtype, scene.sh_coeffs.flags['C_CONTIGUOUS'], scene.center.flags['C_CONTIGUOUS'])
