"""Host f32 <-> f64 conversion throughput on the box: torch copy_ (the
_hostio path so far) vs hgs_host_widen / hgs_host_narrow (streaming stores),
at the e2e step's sizes (59M-element ParamGrads, 48M-element SH).
Run on the GPU box:  python tools/hostconv_bench.py"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio, _lib  # noqa: E402

L = _lib.lib()
print("cores", os.cpu_count(), "torch threads", torch.get_num_threads())


def t(f, reps=5):
    f()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


for n in (59_000_000, 6_220_800):
    src = torch.empty(n, dtype=torch.float32, pin_memory=True).uniform_()
    dst = torch.from_numpy(_hostio.host_empty((n,), np.float64))
    ms = t(lambda: dst.copy_(src))
    print("widen n=%d torch copy_: %.2f ms (%.1f GB/s of 12 B/elem)" % (n, ms, 12 * n / ms / 1e6))
    for th in (0, 8, 16, 32):
        ms = t(lambda: L.hgs_host_widen(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), n, th))
        print("widen n=%d nt threads=%d: %.2f ms (%.1f GB/s)" % (n, th, ms, 12 * n / ms / 1e6))
    assert torch.equal(dst, src.double())
n = 48_000_000
src64 = torch.from_numpy(np.random.default_rng(0).standard_normal(n))
dst32 = torch.empty(n, dtype=torch.float32, pin_memory=True)
ms = t(lambda: dst32.copy_(src64))
print("narrow n=%d torch copy_: %.2f ms (%.1f GB/s)" % (n, ms, 12 * n / ms / 1e6))
for th in (0, 8, 16, 32):
    ms = t(lambda: L.hgs_host_narrow(ctypes.c_void_p(src64.data_ptr()), ctypes.c_void_p(dst32.data_ptr()), n, th))
    print("narrow n=%d nt threads=%d: %.2f ms (%.1f GB/s)" % (n, th, ms, 12 * n / ms / 1e6))
assert torch.equal(dst32, src64.float())
