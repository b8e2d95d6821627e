"""Host <-> device staging for the reference-facing API (float64 numpy in/out).

The reference's ``render``/``backward`` take and return float64 numpy arrays
(core/types.py:40-45, raster/render.py:54-61, grad/bundle.py:11-63).  The
kernels read float32 SoA, so every host call converts.  Doing that naively
(``torch.from_numpy(f64).to(dev)`` then a device-side cast, or ``.double()``
on the device then a pageable ``.cpu()``) moves 2x the bytes through pageable
memory, single-threaded.  Here instead:

* upload: the float64 -> float32 conversion is written straight into a
  persistent pinned staging buffer on all host cores (hgs_host_narrow),
  chunk by chunk, and each chunk's DMA to the device is issued as soon as it
  is converted, so conversion of chunk i+1 overlaps the copy of chunk i;
* download: float32 results are DMA'd into pinned staging chunk by chunk and
  widened to float64 on all host cores as each chunk lands (hgs_host_widen).

Both directions are host-DRAM bound, not PCIe bound, so the conversions
(csrc/hgs_hostconv.cpp) write with streaming stores: no read-for-ownership
of the destination lines (widening 59M floats 8.5 -> 4.3 ms on the box).

Only float32 crosses PCIe in either direction.

Large host outputs come from a recycling pool of anonymous mappings
(``host_empty``): at 1M Gaussians the float64 ParamGrads is 472 MB, and
first-touch page faults of fresh memory -- not the copies -- dominated its
download (25-50 ms per call).  A mapping goes back to the pool only when the
last numpy view of it has been garbage collected (a finalizer on the buffer
owner, which every view's base chain keeps alive), the way a caching
allocator recycles device memory.
"""

import ctypes
import os
import mmap
import threading
import weakref

import numpy as np

_POOL_MIN = 4 << 20        # bytes; smaller outputs use the normal allocator
_POOL_CAP = 8 << 30        # bytes of idle mappings kept for reuse
_pool = {}                 # nbytes -> [mmap]
_pool_bytes = [0]
_pool_lock = threading.Lock()


_registered = {}  # id(mmap) -> host address of a page-locked (cudaHostRegister) pool mapping


def _recycle(mm, nbytes):
    with _pool_lock:
        if _pool_bytes[0] + nbytes <= _POOL_CAP:
            _pool.setdefault(nbytes, []).append(mm)
            _pool_bytes[0] += nbytes
            return
        addr = _registered.pop(id(mm), None)
    if addr is not None:
        from . import _lib
        _lib.lib().hgs_host_unregister(ctypes.c_void_p(addr))
    mm.close()


def _register(mm, size):
    """Page-lock a pool mapping once (it is recycled, so the registration is
    amortised): copies into it are DMAs."""
    addr = _registered.get(id(mm))
    if addr is None:
        from . import _lib
        tmp = (ctypes.c_char * size).from_buffer(mm)
        addr = ctypes.addressof(tmp)
        del tmp
        if _lib.lib().hgs_host_register(ctypes.c_void_p(addr), size) != 0:
            return None
        _registered[id(mm)] = addr
    return addr


def host_empty(shape, dtype=np.float64, register=False):
    """A new (uninitialised) numpy array; large ones reuse pooled, already
    faulted-in mappings (``register``: page-locked, so a device copy into it
    is a DMA)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) if len(shape) else 1
    nbytes = n * dtype.itemsize
    if nbytes < _POOL_MIN:
        return np.empty(shape, dtype)
    size = (nbytes + (2 << 20) - 1) & ~((2 << 20) - 1)
    with _pool_lock:
        lst = _pool.get(size)
        mm = lst.pop() if lst else None
        if mm is not None:
            _pool_bytes[0] -= size
    if mm is None:
        mm = mmap.mmap(-1, size)
    if register:
        _register(mm, size)
    # buffer owner of the mapping: a ctypes array exports the buffer protocol
    # on every supported Python (3.10+) and is weak-referenceable, so the
    # finalizer runs when the last numpy view of it is gone
    owner = (ctypes.c_char * size).from_buffer(mm)
    weakref.finalize(owner, _recycle, mm, size)
    return np.frombuffer(owner, dtype=dtype, count=n).reshape(shape)


_CHUNK = 16 << 20  # bytes of float32 per pipelined chunk
# float64 <-> float32 conversions through hgs_host_widen / hgs_host_narrow
# (all cores, streaming stores: widening 59M floats 8.5 -> 4.3 ms on the box,
# tools/hostconv_bench.py) instead of torch's converting copy
_NT = os.environ.get("HGS_HOST_NT", "1") != "0"


def _convert(fn, src, dst):
    from . import _lib
    rc = getattr(_lib.lib(), fn)(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), src.numel(), 0)
    if rc != 0:
        raise RuntimeError("%s failed (%d)" % (fn, rc))


def _copy(src, dst):
    from . import _lib
    nb = src.numel() * src.element_size()
    rc = _lib.lib().hgs_host_copy(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), nb, 0)
    if rc != 0:
        raise RuntimeError("hgs_host_copy failed (%d)" % rc)
_stages = {}       # tag -> [pinned uint8 tensor, cuda event guarding reuse]


def _stage(tag, nbytes):
    import torch
    ent = _stages.get(tag)
    if ent is not None and ent[1] is not None:
        ent[1].synchronize()  # the previous DMA out of / into this buffer is done
    if ent is None or ent[0].numel() < nbytes:
        ent = [torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True), None]
        _stages[tag] = ent
    return ent


def _align(n):
    return (n + 255) & ~255


def fingerprint_sum(a):
    """The scene fingerprint's sum of one float64 host array: deterministic
    block sums (hgs_host_block_sums, all cores) added in order -- the same
    value ``upload(..., sums_out=)`` produces while it stages the array."""
    import torch
    a = np.asarray(a)
    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        return float(torch.from_numpy(np.ascontiguousarray(a)).sum())
    from . import _lib
    L = _lib.lib()
    n = a.size
    sums = np.zeros(max(-(-n // L.hgs_host_sum_block()), 1))
    if L.hgs_host_block_sums(ctypes.c_void_p(a.ctypes.data), n, ctypes.c_void_p(sums.ctypes.data), 0) != 0:
        raise RuntimeError("hgs_host_block_sums failed")
    return _add_in_order(sums)


def _add_in_order(sums):
    t = 0.0
    for v in sums.tolist():
        t += v
    return t


def upload(arrays, device, tag="up", sums_out=None, nonfinite_out=None):
    """[(numpy array, torch dtype)] -> list of device tensors of those dtypes.

    One pinned staging buffer and one device allocation for the whole list.
    ``sums_out``: a dict whose keys are indices of float64 arrays staged as
    float64; their fingerprint sums (``fingerprint_sum``) are stored under
    the same keys, computed by the staging pass itself.  ``nonfinite_out``:
    likewise, for float64 arrays narrowed to float32, the number of inf /
    NaN float64 inputs (counted by the narrowing pass)."""
    import torch
    metas = []
    total = 0
    for i, (a, dt) in enumerate(arrays):
        a = np.ascontiguousarray(a)
        nb = a.size * torch.empty((), dtype=dt).element_size()
        metas.append((i, a, dt, total, nb))
        total += _align(nb)
    ent = _stage(tag, total)
    stage = ent[0]
    dev = torch.empty(max(total, 1), dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    outs = []
    for i, a, dt, off, nb in metas:
        src = torch.from_numpy(a).reshape(-1)
        hv = stage[off:off + nb].view(dt)
        dv = dev[off:off + nb].view(dt)
        esz = max(hv.element_size(), 1)
        step = max(_CHUNK // esz, 1)
        narrow = _NT and src.dtype == torch.float64 and dt == torch.float32
        count_bad = narrow and nonfinite_out is not None and i in nonfinite_out
        bad = 0
        want_sum = (sums_out is not None and i in sums_out and _NT
                    and src.dtype == torch.float64 and dt == torch.float64)
        if want_sum:
            from . import _lib
            B = _lib.lib().hgs_host_sum_block()
            assert step % B == 0, "staging chunks must hold whole fingerprint blocks"
            bsums = np.zeros(max(-(-src.numel() // B), 1))
        for s in range(0, src.numel(), step):
            e = min(s + step, src.numel())
            if count_bad:  # f64 -> f32 and the finiteness check in one pass
                from . import _lib
                c = ctypes.c_int64(0)
                if _lib.lib().hgs_host_narrow_count(ctypes.c_void_p(src[s:e].data_ptr()),
                                                    ctypes.c_void_p(hv[s:e].data_ptr()), e - s, 0,
                                                    ctypes.byref(c)) != 0:
                    raise RuntimeError("hgs_host_narrow_count failed")
                bad += c.value
            elif narrow:  # f64 -> f32 into pinned on all cores, streaming stores
                _convert("hgs_host_narrow", src[s:e], hv[s:e])
            elif want_sum:  # copy + the fingerprint's block sums in one pass (step is a multiple of B)
                rc = _lib.lib().hgs_host_copy_block_sums(ctypes.c_void_p(src[s:e].data_ptr()),
                                                         ctypes.c_void_p(hv[s:e].data_ptr()), e - s,
                                                         ctypes.c_void_p(bsums.ctypes.data + 8 * (s // B)), 0)
                if rc != 0:
                    raise RuntimeError("hgs_host_copy_block_sums failed (%d)" % rc)
            elif _NT and src.dtype == dt:
                _copy(src[s:e], hv[s:e])
            else:
                hv[s:e].copy_(src[s:e])
            dv[s:e].copy_(hv[s:e], non_blocking=True)    # async DMA while the next chunk converts
        if want_sum:
            sums_out[i] = _add_in_order(bsums)
        if count_bad:
            nonfinite_out[i] = bad
        outs.append(dv.view(a.shape))
    ev = torch.cuda.Event()
    ev.record(stream)
    ent[1] = ev
    return outs


# share of each large float64 output widened on the GPU and DMA'd as float64
# into the page-locked destination; the rest crosses as float32 and is
# widened on the host cores -- both at once.  Paid (0.4: 26.0 -> 25.0 ms per
# step) while host widening cost ~20 B of host DRAM traffic per element; with
# streaming-store widening (~16 B) the host-only split is as fast or faster
# (tools/e2e_ab.py: 20.9 vs 21.2 ms at 0.2), so the default is 0.
_GPU_WIDEN = float(os.environ.get("HGS_GPU_WIDEN", "0.0"))
_GPU_WIDEN_MIN = 1 << 21  # elements; smaller outputs are widened on the host


def download(tensors, dtype=np.float64, tag="down"):
    """Device float32 tensors -> list of new numpy arrays of ``dtype``.

    DMA into pinned staging in chunks (one event per chunk) and widen each
    chunk on the host while later chunks are still in flight; for large
    float64 outputs the leading ``_GPU_WIDEN`` share is widened on the GPU
    (hgs_widen_d2h) and DMA'd straight into the destination on a side
    stream, concurrently."""
    import torch
    tdt = {np.float64: torch.float64, np.float32: torch.float32}[dtype]
    metas = []
    total = 0
    for t in tensors:
        t = t.contiguous()
        nb = t.numel() * t.element_size()
        metas.append((t, total, nb))
        total += _align(nb)
    ent = _stage(tag, total)
    stage = ent[0]
    dev = tensors[0].device if tensors else None
    stream = torch.cuda.current_stream(dev)
    outs, pending, gpu_parts = [], [], []
    side = None
    for t, off, nb in metas:
        flat = t.reshape(-1)
        hv = stage[off:off + nb].view(t.dtype)
        step = max(_CHUNK // t.element_size(), 1)
        n = flat.numel()
        split = (int(n * _GPU_WIDEN) & ~1023) if (dtype is np.float64 and t.dtype == torch.float32
                                                  and n >= _GPU_WIDEN_MIN) else 0
        out = torch.from_numpy(host_empty(tuple(t.shape), dtype, register=split > 0))
        oflat = out.reshape(-1)
        if split:
            from . import _lib
            if side is None:
                side = _side_stream(dev)
                side.wait_stream(stream)
            scratch = torch.empty(split, dtype=torch.float64, device=dev)
            scratch.record_stream(side)
            flat.record_stream(side)
            rc = _lib.lib().hgs_widen_d2h(ctypes.c_void_p(flat.data_ptr()), ctypes.c_void_p(oflat.data_ptr()),
                                          split, ctypes.c_void_p(scratch.data_ptr()),
                                          ctypes.c_void_p(side.cuda_stream))
            if rc == 0:
                gpu_parts.append(scratch)
            else:
                split = 0
        else:
            split = 0
        for s in range(split, n, step):
            e = min(s + step, flat.numel())
            hv[s:e].copy_(flat[s:e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            pending.append((ev, oflat[s:e], hv[s:e]))
        outs.append(out)
    widen = _NT and dtype is np.float64
    for ev, o, h in pending:
        ev.synchronize()
        if widen and h.dtype == torch.float32:  # f32 -> f64 while later chunks are in flight
            _convert("hgs_host_widen", h, o)
        else:
            o.copy_(h)
    if side is not None:
        side.synchronize()  # the GPU-widened shares have landed
    ent[1] = None
    return [o.numpy() for o in outs]


_sides = {}


def _side_stream(dev):
    import torch
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _sides:
        _sides[idx] = torch.cuda.Stream(device=idx)
    return _sides[idx]
