"""Checkpoint I/O and diagnostics output (SPEC.md
module ``io``, lines 460-500, and the CSV logs of lines 285 / 371 / 444).

The reference declares this module in its SPEC but ships no code for it, so
the byte layout below is this package's (documented byte-exact, as SPEC.md:503
asks).  All integers and floats are little-endian.

Checkpoint file::

    offset  size  field
    0       8     magic  b"HGSCKPT1"
    8       4     u32    format version (1)
    12      4     u32    SH degree l (0..3); B = (l + 1)^2
    16      8     u64    record count n
    24      4     u32    record size in bytes = 4 (11 + 3B) + 1
    28      4     u32    reserved (0)
    32      n x record, packed (no padding):
            center 3 x f32, log_scale 3 x f32, rotation 4 x f32 (w first),
            opacity_logit f32, sh 3B x f32 (channel-major, (3, B)), type_spec u8

``load_checkpoint(save_checkpoint(s))`` is bitwise identical for float32
scenes (device scenes, or host scenes of float32-representable values);
float64 host values are rounded to float32 on save.
"""

import csv
import os
import struct
import zlib

import numpy as np

from .core import DeviceGaussians, GaussianSet, n_bases
from .errors import CheckpointError, ConfigError, IntegrityError

__all__ = ["save_checkpoint", "load_checkpoint", "checkpoint_dtype", "write_image", "write_depth",
           "append_exchange_csv", "append_conflict_csv", "MAGIC", "VERSION"]

MAGIC = b"HGSCKPT1"
VERSION = 1
_HEADER = struct.Struct("<8sIIQII")  # 32 bytes


def checkpoint_dtype(sh_degree):
    """numpy structured dtype of one packed record."""
    b = n_bases(sh_degree)
    return np.dtype([("center", "<f4", (3,)), ("log_scale", "<f4", (3,)),
                     ("rotation", "<f4", (4,)), ("opacity_logit", "<f4"),
                     ("sh", "<f4", (3, b)), ("type_spec", "u1")], align=False)


def _host_fields(scene):
    if isinstance(scene, DeviceGaussians):
        return {f: getattr(scene, f).detach().cpu().numpy() for f in scene.FIELDS}, scene.sh_degree
    return {f: getattr(scene, f) for f in GaussianSet.FIELDS}, scene.sh_degree


def save_checkpoint(scene, path):
    """Write ``scene`` (GaussianSet or DeviceGaussians) to ``path``."""
    f, deg = _host_fields(scene)
    n = f["center"].shape[0]
    dt = checkpoint_dtype(deg)
    rec = np.empty(n, dtype=dt)
    rec["center"] = f["center"]
    rec["log_scale"] = f["log_scale"]
    rec["rotation"] = f["rotation"]
    rec["opacity_logit"] = f["opacity_logit"]
    rec["sh"] = f["sh_coeffs"]
    rec["type_spec"] = f["type_spec"]
    tmp = str(path) + ".tmp"
    try:
        with open(tmp, "wb") as fh:
            fh.write(_HEADER.pack(MAGIC, VERSION, deg, n, dt.itemsize, 0))
            fh.write(rec.tobytes())
        os.replace(tmp, path)
    except OSError as e:
        raise ConfigError("cannot write checkpoint %s: %s" % (path, e))


def load_checkpoint(path, device=None, extent=1.0):
    """Read a checkpoint; returns a GaussianSet (float64 fields holding the
    float32 values), or a DeviceGaussians on ``device`` if given."""
    try:
        with open(path, "rb") as fh:
            head = fh.read(_HEADER.size)
            if len(head) < _HEADER.size:
                raise CheckpointError("%s: truncated header" % path)
            magic, ver, deg, n, rsize, _ = _HEADER.unpack(head)
            if magic != MAGIC:
                raise CheckpointError("%s: bad magic %r" % (path, magic))
            if ver != VERSION:
                raise CheckpointError("%s: unknown checkpoint version %d" % (path, ver))
            if deg > 3:
                raise CheckpointError("%s: SH degree %d > 3" % (path, deg))
            dt = checkpoint_dtype(deg)
            if rsize != dt.itemsize:
                raise CheckpointError("%s: record size %d, expected %d" % (path, rsize, dt.itemsize))
            body = fh.read()
    except OSError as e:
        raise CheckpointError("cannot read checkpoint %s: %s" % (path, e))
    if len(body) != n * rsize:
        raise IntegrityError("%s: truncated or oversized body (%d bytes for %d records of %d)"
                             % (path, len(body), n, rsize))
    rec = np.frombuffer(body, dtype=dt, count=n)
    if n and not np.all(rec["type_spec"] <= 1):
        raise IntegrityError("%s: type_spec values other than 0/1" % path)
    if device is not None:
        import torch
        dev = torch.device(device)
        t = [torch.from_numpy(np.ascontiguousarray(rec[k])).to(dev)
             for k in ("center", "log_scale", "rotation", "opacity_logit", "sh", "type_spec")]
        return DeviceGaussians(*t, extent=extent)
    return GaussianSet(rec["center"], rec["log_scale"], rec["rotation"], rec["opacity_logit"],
                       rec["sh"], rec["type_spec"], extent=extent)


# ------------------------------------------------------------------ images
def _png(path, arr, bit_depth):
    """Minimal greyscale / RGB PNG writer (zlib, no filtering)."""
    h, w = arr.shape[:2]
    ch = 1 if arr.ndim == 2 else arr.shape[2]
    color_type = {1: 0, 3: 2, 4: 6}[ch]
    if bit_depth == 16:
        raw = arr.astype(">u2").reshape(h, w * ch)
    else:
        raw = arr.astype(np.uint8).reshape(h, w * ch)
    rows = b"".join(b"\x00" + raw[y].tobytes() for y in range(h))

    def chunk(tag, data):
        return (struct.pack(">I", len(data)) + tag + data
                + struct.pack(">I", zlib.crc32(tag + data) & 0xffffffff))
    ihdr = struct.pack(">IIBBBBB", w, h, bit_depth, color_type, 0, 0, 0)
    try:
        with open(path, "wb") as fh:
            fh.write(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", ihdr) + chunk(b"IDAT", zlib.compress(rows, 6))
                     + chunk(b"IEND", b""))
    except OSError as e:
        raise ConfigError("cannot write image %s: %s" % (path, e))


def _host(a):
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.asarray(a, dtype=np.float64)


def write_image(buffer, path):
    """8-bit PNG; values clamped to [0, 1] then rounded half-to-even to
    [0, 255] (constant 0.5 -> 128)."""
    a = _host(buffer)
    if not np.all(np.isfinite(a)):
        raise IntegrityError("image buffer is not finite")
    _png(path, np.rint(np.clip(a, 0.0, 1.0) * 255.0), 8)


def write_depth(depth, path, far):
    """16-bit greyscale PNG of depth / far, clamped and rounded half-to-even."""
    a = _host(depth)
    if not np.all(np.isfinite(a)) or not far > 0:
        raise IntegrityError("depth buffer is not finite or far <= 0")
    _png(path, np.rint(np.clip(a / far, 0.0, 1.0) * 65535.0), 16)


# -------------------------------------------------------------------- logs
def _append_csv(path, header, row):
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as fh:
        w = csv.writer(fh)
        if new:
            w.writerow(header)
        w.writerow(row)


def append_exchange_csv(path, iteration, report):
    """ExchangeReport row (iteration, n_2d, n_3d, conv_3to2, conv_2to3)."""
    _append_csv(path, ["iteration", "n_2d", "n_3d", "conv_3to2", "conv_2to3"],
                [int(iteration), int(report.n_2d), int(report.n_3d), int(report.n_3d_to_2d),
                 int(report.n_2d_to_3d)])


def append_conflict_csv(path, iteration, n_conflicted, n_total):
    """Gradient-conflict diagnostics (iteration, n_conflicted, n_total)."""
    _append_csv(path, ["iteration", "n_conflicted", "n_total"],
                [int(iteration), int(n_conflicted), int(n_total)])
