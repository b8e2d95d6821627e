"""Does DMA'd data land in the host's last-level cache (DDIO)?  Time a
single-threaded float32 -> float64 widening of a chunk (a) hot in cache, (b)
cold (after a 512 MB sweep), (c) right after a device -> pinned DMA of that
chunk; and the converse for uploads: a DMA from a pinned chunk (d) just
written by the CPU vs (e) cold.  Run on the GPU box."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _lib  # noqa: E402

L = _lib.lib()
V = ctypes.c_void_p
sweep = np.ones(64 << 20)  # 512 MB


def cold():
    sweep[::8] += 1.0  # touches every line


for mb in (1, 4, 16):
    n = (mb << 20) // 4
    pin = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dev = torch.randn(n, device="cuda")
    out = np.empty(n, np.float64)
    out[:] = 0
    widen = lambda: L.hgs_host_widen(V(pin.data_ptr()), V(out.ctypes.data), n, 1)  # noqa: E731
    res = {"hot": [], "cold": [], "post-dma": []}
    for _ in range(15):
        widen()
        t0 = time.perf_counter(); widen(); res["hot"].append(time.perf_counter() - t0)
        cold()
        t0 = time.perf_counter(); widen(); res["cold"].append(time.perf_counter() - t0)
        cold()
        pin.copy_(dev, non_blocking=True); torch.cuda.synchronize()
        t0 = time.perf_counter(); widen(); res["post-dma"].append(time.perf_counter() - t0)
    print("widen %2d MB, 1 thread: " % mb + "  ".join("%s %.1f GB/s" % (k, 4 * n / np.median(v) / 1e9)
                                                       for k, v in res.items()))
    # upload side: DMA time from a pinned chunk just written by the CPU vs cold
    src = np.random.default_rng(0).standard_normal(n)
    narrow = lambda: L.hgs_host_narrow(V(src.ctypes.data), V(pin.data_ptr()), n, 1)  # noqa: E731
    r2 = {"dma after cpu write": [], "dma cold": []}
    for _ in range(15):
        narrow()  # streaming stores: the lines go to DRAM
        cold()
        torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(pin, non_blocking=True); torch.cuda.synchronize()
        r2["dma cold"].append(time.perf_counter() - t0)
        pin.fill_(1.0)  # cached stores: the lines sit in the cache
        torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(pin, non_blocking=True); torch.cuda.synchronize()
        r2["dma after cpu write"].append(time.perf_counter() - t0)
    print("h2d %2d MB: " % mb + "  ".join("%s %.1f GB/s" % (k, 4 * n / np.median(v) / 1e9) for k, v in r2.items()))
