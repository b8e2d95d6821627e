"""CPU: checkpoint I/O, image export and CSV logs (SPEC.md io module,
lines 460-500; examples at 480-492)."""

import struct
import zlib

import numpy as np
import pytest

from paper_2512_02932_b200 import io as hio
from paper_2512_02932_b200.errors import CheckpointError, IntegrityError
from paper_2512_02932_b200.synthetic import synthetic_scene


def _read_png(path):
    data = open(path, "rb").read()
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat, ihdr = 8, b"", None
    while pos < len(data):
        (ln,) = struct.unpack(">I", data[pos:pos + 4])
        tag = data[pos + 4:pos + 8]
        body = data[pos + 8:pos + 8 + ln]
        (crc,) = struct.unpack(">I", data[pos + 8 + ln:pos + 12 + ln])
        assert crc == zlib.crc32(tag + body) & 0xffffffff
        if tag == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body)
        elif tag == b"IDAT":
            idat += body
        pos += 12 + ln
    w, h, depth, ctype = ihdr[:4]
    ch = {0: 1, 2: 3, 6: 4}[ctype]
    bpp = ch * depth // 8
    raw = zlib.decompress(idat)
    rows = []
    for y in range(h):
        line = raw[y * (1 + w * bpp):(y + 1) * (1 + w * bpp)]
        assert line[0] == 0
        rows.append(np.frombuffer(line[1:], dtype=">u2" if depth == 16 else np.uint8))
    return np.stack(rows).reshape(h, w, ch) if ch > 1 else np.stack(rows), depth


@pytest.mark.parametrize("deg", [0, 1, 3])
def test_checkpoint_round_trip_bitwise(tmp_path, deg):
    scene, _ = synthetic_scene(777, 64, 48, deg, seed=deg)
    p = tmp_path / "s.ckpt"
    hio.save_checkpoint(scene, p)
    back = hio.load_checkpoint(p)
    for f in scene.FIELDS:
        a, b = getattr(scene, f), getattr(back, f)
        assert a.shape == b.shape and np.array_equal(a, b), f
    assert back.type_census() == scene.type_census()  # mixed types reload identically
    size = 32 + 777 * (4 * (11 + 3 * (deg + 1) ** 2) + 1)
    assert p.stat().st_size == size


def test_checkpoint_errors(tmp_path):
    scene, _ = synthetic_scene(50, 32, 32, 1, seed=0)
    p = tmp_path / "s.ckpt"
    hio.save_checkpoint(scene, p)
    raw = p.read_bytes()
    (tmp_path / "trunc.ckpt").write_bytes(raw[:-7])  # truncated mid-record
    with pytest.raises(IntegrityError):
        hio.load_checkpoint(tmp_path / "trunc.ckpt")
    (tmp_path / "magic.ckpt").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(CheckpointError):
        hio.load_checkpoint(tmp_path / "magic.ckpt")
    (tmp_path / "ver.ckpt").write_bytes(raw[:8] + struct.pack("<I", 99) + raw[12:])
    with pytest.raises(CheckpointError):
        hio.load_checkpoint(tmp_path / "ver.ckpt")
    (tmp_path / "short.ckpt").write_bytes(raw[:20])
    with pytest.raises(CheckpointError):
        hio.load_checkpoint(tmp_path / "short.ckpt")


def test_empty_scene_round_trip(tmp_path):
    from paper_2512_02932_b200.core import GaussianSet
    e = GaussianSet.empty(sh_degree=2)
    hio.save_checkpoint(e, tmp_path / "e.ckpt")
    assert hio.load_checkpoint(tmp_path / "e.ckpt").count == 0


def test_write_image_and_depth(tmp_path):
    hio.write_image(np.full((4, 5, 3), 0.5), tmp_path / "c.png")
    img, depth = _read_png(tmp_path / "c.png")
    assert depth == 8 and img.shape == (4, 5, 3) and np.all(img == 128)
    hio.write_image(np.array([[-1.0, 2.0], [0.25, 1.0]]), tmp_path / "g.png")
    g, _ = _read_png(tmp_path / "g.png")
    assert g.tolist() == [[0, 255], [64, 255]]
    hio.write_depth(np.array([[0.0, 5.0], [10.0, 20.0]]), tmp_path / "d.png", far=10.0)
    d, depth = _read_png(tmp_path / "d.png")
    assert depth == 16 and d.tolist() == [[0, 32768], [65535, 65535]]
    with pytest.raises(IntegrityError):
        hio.write_image(np.array([[np.nan]]), tmp_path / "bad.png")


def test_csv_logs(tmp_path):
    from paper_2512_02932_b200.exchange import ExchangeReport
    p = tmp_path / "x.csv"
    hio.append_exchange_csv(p, 500, ExchangeReport(3, 1, 10, 20))
    hio.append_exchange_csv(p, 1000, ExchangeReport(0, 2, 12, 18))
    lines = p.read_text().strip().splitlines()
    assert lines == ["iteration,n_2d,n_3d,conv_3to2,conv_2to3", "500,10,20,3,1", "1000,12,18,0,2"]
    q = tmp_path / "c.csv"
    hio.append_conflict_csv(q, 7, 45, 100)
    assert q.read_text().strip().splitlines() == ["iteration,n_conflicted,n_total", "7,45,100"]
