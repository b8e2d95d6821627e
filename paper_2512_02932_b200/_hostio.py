"""Host <-> device staging for the reference-facing API (float64 numpy in/out).

The reference's ``render``/``backward`` take and return float64 numpy arrays
(core/types.py:40-45, raster/render.py:54-61, grad/bundle.py:11-63).  The
kernels read float32 SoA, so every host call converts.  Doing that naively
(``torch.from_numpy(f64).to(dev)`` then a device-side cast, or ``.double()``
on the device then a pageable ``.cpu()``) moves 2x the bytes through pageable
memory, single-threaded.  Here instead:

* upload: the float64 -> float32 conversion is written straight into a
  persistent pinned staging buffer by torch's multi-threaded CPU copy, chunk
  by chunk, and each chunk's DMA to the device is issued as soon as it is
  converted, so conversion of chunk i+1 overlaps the copy of chunk i;
* download: float32 results are DMA'd into pinned staging chunk by chunk and
  widened to float64 on all host cores as each chunk lands.

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
import mmap
import threading
import weakref

import numpy as np

_POOL_MIN = 4 << 20        # bytes; smaller outputs use the normal allocator
_POOL_CAP = 8 << 30        # bytes of idle mappings kept for reuse
_pool = {}                 # nbytes -> [mmap]
_pool_bytes = [0]
_pool_lock = threading.Lock()


def _recycle(mm, nbytes):
    with _pool_lock:
        if _pool_bytes[0] + nbytes <= _POOL_CAP:
            _pool.setdefault(nbytes, []).append(mm)
            _pool_bytes[0] += nbytes
            return
    mm.close()


def host_empty(shape, dtype=np.float64):
    """A new (uninitialised) numpy array; large ones reuse pooled, already
    faulted-in mappings."""
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
    # buffer owner of the mapping: a ctypes array exports the buffer protocol
    # on every supported Python (3.10+) and is weak-referenceable, so the
    # finalizer runs when the last numpy view of it is gone
    owner = (ctypes.c_char * size).from_buffer(mm)
    weakref.finalize(owner, _recycle, mm, size)
    return np.frombuffer(owner, dtype=dtype, count=n).reshape(shape)


_CHUNK = 16 << 20  # bytes of float32 per pipelined chunk
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


def upload(arrays, device, tag="up"):
    """[(numpy array, torch dtype)] -> list of device tensors of those dtypes.

    One pinned staging buffer and one device allocation for the whole list."""
    import torch
    metas = []
    total = 0
    for a, dt in arrays:
        a = np.ascontiguousarray(a)
        nb = a.size * torch.empty((), dtype=dt).element_size()
        metas.append((a, dt, total, nb))
        total += _align(nb)
    ent = _stage(tag, total)
    stage = ent[0]
    dev = torch.empty(max(total, 1), dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    outs = []
    for a, dt, off, nb in metas:
        src = torch.from_numpy(a).reshape(-1)
        hv = stage[off:off + nb].view(dt)
        dv = dev[off:off + nb].view(dt)
        esz = max(hv.element_size(), 1)
        step = max(_CHUNK // esz, 1)
        for s in range(0, src.numel(), step):
            e = min(s + step, src.numel())
            hv[s:e].copy_(src[s:e])                      # multi-threaded f64 -> f32 into pinned
            dv[s:e].copy_(hv[s:e], non_blocking=True)    # async DMA while the next chunk converts
        outs.append(dv.view(a.shape))
    ev = torch.cuda.Event()
    ev.record(stream)
    ent[1] = ev
    return outs


def download(tensors, dtype=np.float64, tag="down"):
    """Device float32 tensors -> list of new numpy arrays of ``dtype``.

    DMA into pinned staging in chunks (one event per chunk) and widen each
    chunk on the host while later chunks are still in flight."""
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
    outs, pending = [], []
    for t, off, nb in metas:
        flat = t.reshape(-1)
        hv = stage[off:off + nb].view(t.dtype)
        step = max(_CHUNK // t.element_size(), 1)
        out = torch.from_numpy(host_empty(tuple(t.shape), dtype))
        oflat = out.reshape(-1)
        for s in range(0, flat.numel(), step):
            e = min(s + step, flat.numel())
            hv[s:e].copy_(flat[s:e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            pending.append((ev, oflat[s:e], hv[s:e]))
        outs.append(out)
    for ev, o, h in pending:
        ev.synchronize()
        o.copy_(h)  # multi-threaded f32 -> f64 while later chunks are in flight
    ent[1] = None
    return [o.numpy() for o in outs]
