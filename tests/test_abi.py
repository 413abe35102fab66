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


def test_group_plan_host(exmy):
    """exmy_group_plan is host code: chunk bookkeeping and validation
    (include/exmy.h, grouped launch) checked without a device."""
    import struct
    import torch
    A = 0x10000

    def ent(i, rows, cols, **kw):
        e = {"in": A * (i + 1), "packed": A * (i + 100), "meta": A * 1000 + i, "rows": rows, "cols": cols}
        e.update(kw)
        return e

    # bf16: 8 elements per 16-byte vector, 1024 vectors per max chunk; 256 8x4 tiles per tile chunk
    ents = [ent(0, 64, 4096), ent(1, 0, 4), ent(2, 8, 4), ent(3, 8, 512)]
    b = exmy.group_plan(ents, torch.bfloat16, "e3m3")
    assert len(b) == 64 + 4 * 128
    magic, n, dt, x, y, odt, vc, tc, dc, nh, sp = struct.unpack("<Iiiiiiqqqii", b[:56])
    assert (n, dt, x, y, odt, nh, sp) == (4, 1, 3, 3, 1, 1, 0)   # cols 4 -> 8x4 decode tiles
    vchunks = [32, 0, 1, 1]                  # 64*4096/8/1024, -, 32/8 -> 1, 4096/8/1024 -> 1
    tchunks = [(8 * 1024) // 2048, 0, 1, 1]  # encode: CTA chunks of 8 x 256 8x4 tiles
    dchunks = [(8 * 1024) // 256, 0, 1, 1]   # decode: CTA chunks of 256 tiles
    assert vc == sum(vchunks) and tc == sum(tchunks) and dc == sum(dchunks)
    for i in range(4):
        rows, cols, vb, tb, db = struct.unpack("<qqqqq", b[64 + 128 * i + 64:64 + 128 * i + 104])
        assert (rows, cols) == (ents[i]["rows"], ents[i]["cols"])
        assert vb == sum(vchunks[:i]) and tb == sum(tchunks[:i]) and db == sum(dchunks[:i])
    # every cols % 8 == 0 and bf16 output: 8x8 decode tiles, half the chunks
    b = exmy.group_plan([ent(0, 64, 4096), ent(1, 8, 8)], torch.bfloat16, "e3m3")
    tc, dc, nh = struct.unpack("<qqi", b[32:52])
    assert (tc, dc, nh) == (4 + 1, 16 + 1, 2)
    # fp32: 4 elements per vector
    b = exmy.group_plan([ent(0, 64, 4096)], torch.float32, "e2m4", torch.bfloat16)
    assert struct.unpack("<q", b[24:32])[0] == 64 * 4096 // 4 // 1024
    bad = [
        ([ent(0, 12, 8)], 3),                      # rows % 8
        ([ent(0, 8, 6)], 3),                       # cols % 4
        ([ent(0, 8, 8, packed=0)], 8),             # NULL packed
        ([ent(0, 8, 8, meta=0)], 8),               # NULL meta
        ([ent(0, 8, 8, packed=A + 8)], 5),         # misaligned
        ([ent(0, 8, 8, sp_capacity=-1)], 6),
        ([ent(0, 8, 8, sp_capacity=4)], 8),        # capacity without buffers
    ]
    for ents, status in bad:
        with pytest.raises(exmy.ExmyError) as ei:
            exmy.group_plan(ents, torch.bfloat16, "e3m3")
        assert ei.value.status == status
    with pytest.raises(exmy.ExmyError):
        exmy.group_plan([], torch.bfloat16, "e3m3")
    # per-row plans (exmy_group_plan_rows): header flag + row count, each
    # entry's first global row; cols % 8 and 8-byte aligned row bytes
    rents = [ent(0, 64, 4096, meta=A * 1000), ent(1, 0, 8, meta=A * 1001), ent(2, 16, 8, meta=A * 1002),
             ent(3, 8, 512, meta=A * 1003)]
    b = exmy.group_plan(rents, torch.bfloat16, "e3m3", per_row=True)
    sp, per_row, row_total = struct.unpack("<hhq", b[52:64])
    assert (sp, per_row, row_total) == (0, 1, 64 + 16 + 8)
    for i, (rb, fb, fused) in enumerate([(0, 0, 1), (64, 8, 0), (64, 8, 1), (80, 10, 1)]):
        # first global row; first TMA-staged row group and the "rows <= 9216 B" flag
        assert struct.unpack("<qqq", b[64 + 128 * i + 104:64 + 128 * i + 128]) == (rb, fb, fused)
    wide = exmy.group_plan([ent(0, 8, 4616, meta=A * 1000)], torch.bfloat16, "e3m3", per_row=True)
    assert struct.unpack("<q", wide[64 + 120:64 + 128])[0] == 0      # 9232-byte rows: two-pass entry
    assert struct.unpack("<hh", exmy.group_plan(rents, torch.bfloat16, "e3m3")[52:56]) == (0, 0)
    for ents, status in [([ent(0, 8, 4, meta=A * 1000)], 3), ([ent(0, 8, 8, meta=A * 1000 + 4)], 5)]:
        with pytest.raises(exmy.ExmyError) as ei:
            exmy.group_plan(ents, torch.bfloat16, "e3m3", per_row=True)
        assert ei.value.status == status
    assert exmy.group_layout((4096,)) == (8, 512)
    assert exmy.group_layout((3, 5, 8)) == (15, 8)
    # the device calls check the plan before launching anything
    L = exmy.lib()
    junk = (ctypes.c_uint64 * 16)()
    assert L.exmy_group_encode(junk, junk, None) == 8


def test_no_cpu_fallback(exmy, tmp_path):
    """the product path fails loudly: importing without libexmy.so raises, and
    CPU tensors are refused (never computed on the host)"""
    import subprocess
    import sys
    import torch
    code = ("import os, sys; sys.path.insert(0, %r); os.environ['EXMY_LIB_PATH'] = %r\n"
            "try:\n    import paper_2405_13938_b200\nexcept ImportError as e:\n    print('IMPORT-ERROR', e)\n")
    out = subprocess.run([sys.executable, "-c", code % (ROOT, str(tmp_path / "missing.so"))],
                         capture_output=True, text=True, timeout=120)
    assert "IMPORT-ERROR" in out.stdout and "no CPU fallback" in out.stdout
    t = torch.zeros((8, 8), dtype=torch.bfloat16)
    for call in (lambda: exmy.histogram(t), lambda: exmy.quantize(t, "e3m3", 127),
                 lambda: exmy.encode(t, "e3m3", 127), lambda: exmy.encode_fs(t, "e2m1", None, "row"),
                 lambda: exmy.GroupCodec([t], "e3m3")):
        with pytest.raises(ValueError, match="CUDA"):
            call()
