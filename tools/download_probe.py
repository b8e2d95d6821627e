"""Where the image download of the host API goes (config 2, 1080p): the
three float32 images -> float64 numpy through _hostio.download, repeated
with the results dropped each time (pool recycled), against the raw DMA and
the raw host widening of the same bytes.  Run on the GPU box."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio, _lib  # noqa: E402

H, W = 1080, 1920
dev = torch.device("cuda", 0)
imgs = [torch.rand((H, W, 3), device=dev), torch.rand((H, W), device=dev), torch.rand((H, W), device=dev)]
grads = [torch.rand(1_000_000 * 59, device=dev)]


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for name, ts in (("images", imgs), ("grads", grads)):
    for it in range(6):
        t0 = t()
        out = _hostio.download(ts, tag=name)
        t1 = t()
        del out
        print(name, "download ms %.2f" % ((t1 - t0) * 1e3))
    nb = sum(x.numel() for x in ts) * 4
    pin = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
    flat = torch.cat([x.reshape(-1) for x in ts])
    for it in range(3):
        t0 = t()
        pin.copy_(flat, non_blocking=True)
        t1 = t()
        print(name, "raw DMA ms %.2f (%.1f GB/s)" % ((t1 - t0) * 1e3, nb / (t1 - t0) / 1e9))
    dst = _hostio.host_empty((nb // 4,), np.float64)
    dt = torch.from_numpy(dst)
    for it in range(3):
        t0 = time.perf_counter()
        _hostio._convert("hgs_host_widen", pin, dt)
        t1 = time.perf_counter()
        print(name, "host widen ms %.2f" % ((t1 - t0) * 1e3))
    for it in range(2):
        t0 = time.perf_counter()
        d2 = _hostio.host_empty((nb // 4,), np.float64)
        d2t = torch.from_numpy(d2)
        _hostio._convert("hgs_host_widen", pin, d2t)
        t1 = time.perf_counter()
        del d2, d2t
        print(name, "host_empty + widen ms %.2f" % ((t1 - t0) * 1e3))
