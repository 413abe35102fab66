"""CPU-side checks of the C ABI boundary (no GPU needed): the library loads,
exports every symbol include/exmy.h declares, validates arguments before
touching the device, and its host helpers agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exmy():
    import paper_2405_13938_b200 as m
    return m


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "exmy.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(exmy_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_symbols_exported(exmy):
    names = _declared_functions()
    assert len(names) >= 15
    L = ctypes.CDLL(exmy.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(exmy.EXPORTED)


def test_library_is_sm100a(exmy):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", exmy.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(exmy):
    assert "sm_100a" in exmy.version()


def test_formats(exmy):
    fm = exmy.all_formats()
    assert len(fm) == 42
    assert all(exmy.lib().exmy_format_valid(x, y) for x, y in fm)
    assert not exmy.lib().exmy_format_valid(9, 0)
    assert not exmy.lib().exmy_format_valid(1, 0)      # k=2
    assert not exmy.lib().exmy_format_valid(2, 7)      # k=10
    with pytest.raises(ValueError):
        exmy.parse_format("e4m6")


def test_packed_bytes_and_segments(exmy, orc):
    for k in range(3, 10):
        for x in range(0, min(8, k - 1) + 1):
            y = k - 1 - x
            assert exmy.packed_bytes(8 * 37, (x, y)) == 37 * k
    assert exmy.lib().exmy_packed_bytes(12, 3, 3) == -1
    for k in range(1, 16):
        for n in (0, 8, 64, 8 * 1001):
            assert exmy.segments(k, n) == orc.segments(k, n)


def test_bias_emax(exmy, orc):
    for x in range(0, 9):
        for e in (0, 17, 127, 254):
            b = exmy.bias_from_emax(x, e)
            assert b == orc.bias(x, e)
            assert exmy.emax_from_bias(x, b) == e
    with pytest.raises(exmy.ExmyError):
        exmy.bias_from_emax(3, 255)
    with pytest.raises(exmy.ExmyError):
        exmy.emax_from_bias(3, 200)      # e_max would be negative


def test_choose_x_matches_oracle(exmy, orc):
    rng = np.random.default_rng(0)
    for trial in range(300):
        h = np.zeros(256, np.uint64)
        lo = rng.integers(1, 250)
        hi = rng.integers(lo, 255)
        h[lo:hi + 1] = rng.integers(0, 1000, size=hi - lo + 1)
        h[0] = rng.integers(0, 100)
        h[255] = rng.integers(0, 3)
        budget = float(rng.choice([0.0, 1e-3, 0.0011, 0.01, 0.1]))
        assert exmy.choose_x(h.astype(np.int64), budget) == orc.choose_x(h, budget)
        assert exmy.lib().exmy_emax_from_histogram_host(h.ctypes.data_as(ctypes.c_void_p)) == orc.emax(h)


def test_device_ops_validate_before_launch(exmy):
    L = exmy.lib()
    vp = ctypes.c_void_p
    fake = vp(16)   # never dereferenced: validation fails first
    assert L.exmy_quantize(fake, fake, 0, 16, 9, 1, fake, None) == 1          # E_FORMAT
    assert L.exmy_quantize(fake, fake, 7, 16, 3, 2, fake, None) == 4          # E_DTYPE
    assert L.exmy_quantize(fake, fake, 0, -1, 3, 2, fake, None) == 3          # E_SHAPE
    assert L.exmy_quantize(None, fake, 0, 16, 3, 2, fake, None) == 8          # E_ARG
    assert L.exmy_quantize(fake, fake, 0, 0, 3, 2, fake, None) == 0           # n = 0: no-op
    # encode: ROWS needs rows % 8 == 0, COLS cols % 8 == 0
    assert L.exmy_encode(fake, 1, 12, 16, 0, 3, 3, fake, fake, None, None, None, 0, None) == 3
    assert L.exmy_encode(fake, 1, 16, 12, 1, 3, 3, fake, fake, None, None, None, 0, None) == 3
    assert L.exmy_encode(fake, 1, 16, 16, 0, 3, 3, fake, fake, None, None, None, -1, None) == 6
    assert L.exmy_encode(fake, 1, 16, 16, 0, 3, 3, fake, fake, None, None, None, 5, None) == 8
    assert L.exmy_encode(fake, 1, 16, 16, 2, 3, 3, fake, fake, None, None, None, 0, None) == 3
    assert L.exmy_decode(fake, 16, 12, 1, 3, 3, fake, None, None, None, 0, fake, 1, None) == 3
    assert L.exmy_decode(fake, 16, 16, 0, 0, 1, fake, None, None, None, 0, fake, 1, None) == 1
    assert L.exmy_exponent_histogram(fake, 2, 16, fake, None) == 4
    assert L.exmy_emax_from_histogram(None, fake, None) == 8
    for s in range(9):
        assert L.exmy_status_string(s)
