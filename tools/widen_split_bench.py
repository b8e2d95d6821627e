"""_hostio.download of a ParamGrads-sized float32 device tensor (59M) into
float64 host memory at several GPU-widened shares (_GPU_WIDEN), medians of
alternating rounds.  Run on the GPU box:  python tools/widen_split_bench.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_02932_b200 import _hostio  # noqa: E402

g = torch.randn(59_000_000, device="cuda")
shares = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5]
res = {f: [] for f in shares}
for rnd in range(6):
    for f in shares:
        _hostio._GPU_WIDEN = f
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = _hostio.download([g], tag="g")[0]
        torch.cuda.synchronize()
        if rnd:
            res[f].append((time.perf_counter() - t0) * 1e3)
        del out
for f, v in res.items():
    print("gpu widen %.1f: median %.2f ms  min %.2f ms" % (f, np.median(v), np.min(v)))
