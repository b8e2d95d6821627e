"""CPU-side checks of the drop-in boundary: libhgs.so loads, exports every
symbol include/hgs.h declares, and its host-only entry points (sizes, status
strings) behave.  No kernel is launched here."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    inc = os.path.join(REPO, "include")
    src = "".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc))
                  if f.endswith(".h"))
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char \*)\s*(hgs_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2512_02932_b200 import _lib
    so = _lib.LIB_PATH
    if not os.path.exists(so):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    from paper_2512_02932_b200 import _lib
    syms = _header_symbols()
    assert len(syms) >= 10
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s


def test_abi_version_and_status_strings(L):
    from paper_2512_02932_b200 import _lib
    assert L.hgs_abi_version() == _lib.ABI_VERSION
    for code in range(0, 7):
        assert L.hgs_status_string(code)
    assert b"pairs" in L.hgs_status_string(5)


def test_frame_bytes_monotone(L):
    a = L.hgs_frame_bytes(1000, 64, 48, 16, 10000)
    b = L.hgs_frame_bytes(1000, 64, 48, 16, 20000)
    c = L.hgs_frame_bytes(2000, 64, 48, 16, 20000)
    assert 0 < a < b < c
    assert L.hgs_frame_bytes(1000, 64, 48, 8, 10) == 0  # tile size must be 16
    assert L.hgs_backward_scratch_bytes(1000, 1) < L.hgs_backward_scratch_bytes(1000, 3)


def test_struct_sizes_match_header():
    from paper_2512_02932_b200 import _lib
    assert ctypes.sizeof(_lib.Scene) == 8 + 4 + 4 + 10 * 8
    assert ctypes.sizeof(_lib.Camera) == 4 * 8 + 8 + 16 * 8 + 2 * 8
    assert ctypes.sizeof(_lib.FrameInfo) == 4 * 8 + 4 * 4 + 8 + 4 + 4 + 16
    assert ctypes.sizeof(_lib.LossWeights) == 3 * 8
    assert ctypes.sizeof(_lib.Params) == 8 + 4 + 4 + 5 * 8
    assert ctypes.sizeof(_lib.AdamCfg) == 5 * 4 + 3 * 4 + 8


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """sizeof / offsetof of every ABI struct as gcc sees include/*.h equals
    the ctypes mirror in _lib.py."""
    import shutil
    import subprocess
    from paper_2512_02932_b200 import _lib
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("gcc not available")
    pairs = [("hgs_scene", _lib.Scene), ("hgs_camera", _lib.Camera), ("hgs_settings", _lib.Settings),
             ("hgs_images", _lib.Images), ("hgs_frame_info", _lib.FrameInfo),
             ("hgs_exchange_report", _lib.ExchangeReport), ("hgs_frame_export", _lib.FrameExport),
             ("hgs_loss_weights", _lib.LossWeights), ("hgs_params", _lib.Params),
             ("hgs_adam", _lib.AdamCfg), ("hgs_densify_config", _lib.DensifyCfg)]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hgs.h"', '#include "hgs_train.h"',
             'int main(void) {']
    want = []
    for cname, ct in pairs:
        lines.append('printf("%%zu\\n", sizeof(%s));' % cname)
        want.append(ctypes.sizeof(ct))
        for f in ct._fields_:
            lines.append('printf("%%zu\\n", offsetof(%s, %s));' % (cname, f[0]))
            want.append(getattr(ct, f[0]).offset)
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = str(tmp_path / "layout")
    subprocess.run([cc, "-I", os.path.join(REPO, "include"), str(src), "-o", exe], check=True)
    got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert got == want


def test_train_host_entry_points(L):
    # scratch sizes grow with the image; invalid shapes report 0 / CONFIG
    assert L.hgs_loss_scratch_bytes(64, 64, 3) < L.hgs_loss_scratch_bytes(128, 64, 3)
    assert L.hgs_loss_scratch_bytes(0, 64, 3) == 0
    from paper_2512_02932_b200 import _lib
    w = _lib.LossWeights(0.2, 0.2, 0.4)
    assert L.hgs_image_losses(0, 8, 3, None, None, w, None, None, None, 0, None) == 1
    assert L.hgs_combine_gradients(10, 5, None, None, None, None, 0, None, None, None) == 1
    cfg = _lib.AdamCfg((ctypes.c_float * 5)(1, 1, 1, 1, 1), 0.9, 0.999, 1e-15, 0)
    prm = _lib.Params(0, 1, 0, None, None, None, None, None)
    assert L.hgs_adam_step(prm, None, None, None, cfg, None) == 1  # step must be >= 1


def test_errors_are_reference_classes():
    from paper_2512_02932_b200 import _lib, errors
    with pytest.raises(errors.ConfigError):
        _lib.check(1, "x")
    with pytest.raises(errors.InvalidParameterError):
        _lib.check(2, "x")
    with pytest.raises(errors.IntegrityError):
        _lib.check(3, "x")
    with pytest.raises(errors.DegenerateScaleError):
        _lib.check(4, "x")


def _build_c_example(tmp):
    import shutil
    import subprocess
    cc = shutil.which("gcc")
    cuda_inc = "/usr/local/cuda/include"
    if cc is None or not os.path.isdir(cuda_inc):
        pytest.skip("gcc / CUDA headers not available")
    exe = os.path.join(str(tmp), "c_render")
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"), "-I", cuda_inc,
                    os.path.join(REPO, "examples", "c_render.c"), "-L",
                    os.path.join(REPO, "paper_2512_02932_b200"), "-lhgs", "-L", "/usr/local/cuda/lib64",
                    "-lcudart", "-o", exe], check=True)
    return exe


def test_c_example_compiles_against_the_abi(tmp_path, L):
    """The boundary is a plain C ABI: a C program includes hgs.h and links
    libhgs.so without Python or torch (examples/c_render.c)."""
    assert os.path.exists(_build_c_example(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import subprocess
    exe = _build_c_example(tmp_path)
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.pathsep.join([os.path.join(REPO, "paper_2512_02932_b200"),
                                              "/usr/local/cuda/lib64", env.get("LD_LIBRARY_PATH", "")])
    out = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("ok")


@pytest.mark.parametrize("threads", [1, 0])
def test_host_conversions(L, threads):
    """hgs_host_widen / narrow / copy (the host API's staging conversions):
    identical to numpy's casts and copies, specials included, at odd sizes and
    misaligned destinations (head / tail paths of the streaming loops)."""
    import numpy as np
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 9, 1023, 200_003, 1_000_001):
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-40, 40, n)
        if n > 4:
            x[:4] = [np.inf, -np.inf, np.nan, 1e300]  # float32 overflow -> inf, like numpy
        for off in (0, 1, 3):
            d32 = np.empty(n + off, np.float32)[off:]
            assert L.hgs_host_narrow(x.ctypes.data, d32.ctypes.data, n, threads) == 0
            with np.errstate(over="ignore"):
                np.testing.assert_array_equal(d32, x.astype(np.float32))
            d64 = np.empty(n + off, np.float64)[off:]
            assert L.hgs_host_widen(d32.ctypes.data, d64.ctypes.data, n, threads) == 0
            np.testing.assert_array_equal(d64, d32.astype(np.float64))
            b = np.empty(8 * n + off, np.uint8)[off:]
            assert L.hgs_host_copy(x.ctypes.data, b.ctypes.data, 8 * n, threads) == 0
            assert b.tobytes() == x.tobytes()
    assert L.hgs_host_widen(None, None, 5, 0) != 0


def test_host_block_sums(L):
    """The scene-fingerprint sums: the copying and the plain form give the
    same block sums (bit for bit), at any thread count and alignment, and
    the copy is exact."""
    import numpy as np
    B = L.hgs_host_sum_block()
    assert B > 0
    rng = np.random.default_rng(5)
    for n in (0, 1, 9, B - 1, B, 3 * B + 17):
        x = rng.standard_normal(n) * 1e3
        nb = (n + B - 1) // B
        ref = None
        for threads in (1, 0, 3):
            for off in (0, 1):
                s1 = np.zeros(max(nb, 1))
                assert L.hgs_host_block_sums(x.ctypes.data, n, s1.ctypes.data, threads) == 0
                d = np.empty(n + off)[off:]
                s2 = np.zeros(max(nb, 1))
                assert L.hgs_host_copy_block_sums(x.ctypes.data, d.ctypes.data, n, s2.ctypes.data, threads) == 0
                assert d.tobytes() == x.tobytes()
                assert s1.tobytes() == s2.tobytes()
                if ref is None:
                    ref = s1.copy()
                assert s1.tobytes() == ref.tobytes()
        if n:
            np.testing.assert_allclose(sum(ref[:nb]), x.sum(), rtol=1e-12, atol=1e-9)


def test_host_narrow_count(L):
    """Narrowing with the float64 finiteness count (the host backward's
    upstream-gradient check): same float32 values as numpy, inf / NaN counted
    on the float64 inputs (a finite 1e300 is not counted)."""
    import ctypes
    import numpy as np
    rng = np.random.default_rng(7)
    for n in (0, 1, 13, 300_001):
        x = rng.standard_normal(n)
        if n > 10:
            x[[1, 4, 9]] = [np.inf, np.nan, -np.inf]
            x[2] = 1e300
        for off in (0, 1):
            d = np.empty(n + off, np.float32)[off:]
            c = ctypes.c_int64(-1)
            assert L.hgs_host_narrow_count(x.ctypes.data, d.ctypes.data, n, 0, ctypes.byref(c)) == 0
            assert c.value == (3 if n > 10 else 0)
            with np.errstate(over="ignore"):
                np.testing.assert_array_equal(d, x.astype(np.float32))
