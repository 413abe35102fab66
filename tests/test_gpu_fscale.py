"""GPU parity of the float-scaling scheme (reading D23) against the
oracle: block maxima, emulation, encode bytes + specials and decode to both
dtypes, for every block shape class, extreme block maxima (subnormal, 2^127:
the fp64 fallbacks), x = 8 grids (values below the fp32 range), forced
generic kernels, and the config-2 shape.  Bit-exact."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def exmy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as m
    m.force_generic(False)
    return m


def scaled_bits(shape, seed, dt):
    R, C = shape
    rng = np.random.default_rng(seed)
    t = W.f32_wide(shape, seed=seed).numpy()
    t = t * (2.0 ** rng.integers(-40, 40, size=(R, 1))).astype(np.float32)
    t = torch.from_numpy(t.astype(np.float32))
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t).copy()
    flat = bits.reshape(-1)
    flat[rng.integers(0, flat.size, size=max(1, flat.size // 300))] = 0x7FC0 if dt == "bf16" else 0x7FC00000
    flat[rng.integers(0, flat.size, size=2)] = 0xFF80 if dt == "bf16" else 0xFF800000
    return bits


def extreme_bits(dt):
    """rows whose maxima are fp32-subnormal, tiny, 2^127-ish: the fp64 paths"""
    R, C = 16, 32
    rng = np.random.default_rng(7)
    v = rng.standard_normal((R, C)).astype(np.float64)
    scales = [2.0 ** -140, 2.0 ** -130, 2.0 ** -127, 2.0 ** -100, 1.0, 2.0 ** 100, 2.0 ** 126, 2.0 ** 127] * 2
    v = v / np.abs(v).max(axis=1, keepdims=True) * np.array(scales)[:, None] * 1.5
    t = torch.from_numpy(np.clip(v, -3.0e38, 3.0e38).astype(np.float32))
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t).copy()
    bits[3, :] = 0                       # all-zero row: amax 0
    return bits


BLOCKS = [("tensor", None), ("row", None), ("col", None), ("subrow16", (1, 16)), ("tile8x8", (8, 8)),
          ("odd", (2, 6)), ("subrow32", (1, 32)), ("tile8x64", (8, 64))]


def blk(name, spec, shape):
    R, C = shape
    return {"tensor": (R, C), "row": (1, C), "col": (R, 1)}.get(name, spec)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_block_float_scale(exmy, orc, dt):
    for bits in (scaled_bits((64, 96), 1, dt), extreme_bits(dt)):
        d = W.from_bits(bits).to(DEV)
        for name, spec in BLOCKS:
            b = blk(name, spec, bits.shape)
            if bits.shape[1] % b[1] or bits.shape[0] % b[0]:
                continue
            got = exmy.block_float_scale(d, b).cpu().numpy().view(np.uint32)
            np.testing.assert_array_equal(got, orc.block_float_scale(bits, b), err_msg=name)


FMTS = [(3, 3), (2, 1), (4, 2), (0, 6), (6, 0), (1, 5), (8, 0), (0, 8), (5, 3), (3, 5), (2, 2), (1, 1)]


@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_fs_codecs(exmy, orc, fmt, dt):
    for bits in (scaled_bits((64, 96), fmt[0] * 10 + fmt[1], dt), extreme_bits(dt)):
        shape = bits.shape
        d = W.from_bits(bits).to(DEV)
        for name, spec in BLOCKS:
            b = blk(name, spec, shape)
            if shape[1] % b[1] or shape[0] % b[0]:
                continue
            amax = orc.block_float_scale(bits, b)
            sc = torch.from_numpy(amax.view(np.float32).copy()).to(DEV)
            q = W.to_bits(exmy.quantize_fs(d, fmt, sc, b))
            qref = orc.quantize_fs(bits, fmt, amax, b)
            np.testing.assert_array_equal(q, qref, err_msg=f"quantize {name}")
            for axis in ("rows", "cols"):
                ax = orc.ROWS if axis == "rows" else orc.COLS
                p = exmy.encode_fs(d, fmt, sc, b, axis=axis, specials_capacity=bits.size)
                pref, idx, sb, ns = orc.encode_fs(bits, fmt, amax, b, ax)
                np.testing.assert_array_equal(p.data.cpu().numpy(), pref, err_msg=f"encode {name} {axis}")
                spi, spb, cnt = p.specials()
                assert cnt == ns
                np.testing.assert_array_equal(spi.cpu().numpy(), idx)
                np.testing.assert_array_equal(W.to_bits(exmy.decode(p)), qref, err_msg=f"decode {name} {axis}")
                od = np.uint32 if dt == "bf16" else np.uint16
                other = exmy.decode(p, torch.float32 if dt == "bf16" else torch.bfloat16)
                np.testing.assert_array_equal(W.to_bits(other),
                                              orc.decode_fs(pref, shape, fmt, amax, b, ax, idx, sb, od),
                                              err_msg=f"decode other dtype {name} {axis}")


def test_fs_force_generic(exmy, orc):
    bits = scaled_bits((32, 64), 9, "bf16")
    d = W.from_bits(bits).to(DEV)
    amax = orc.block_float_scale(bits, (1, 64))
    sc = torch.from_numpy(amax.view(np.float32).copy()).to(DEV)
    exmy.force_generic(True)
    try:
        for fmt in [(3, 3), (2, 1), (7, 1)]:
            np.testing.assert_array_equal(W.to_bits(exmy.quantize_fs(d, fmt, sc, (1, 64))),
                                          orc.quantize_fs(bits, fmt, amax, (1, 64)))
            p = exmy.encode_fs(d, fmt, sc, (1, 64), specials_capacity=bits.size)
            np.testing.assert_array_equal(p.data.cpu().numpy(), orc.encode_fs(bits, fmt, amax, (1, 64))[0])
            np.testing.assert_array_equal(W.to_bits(exmy.decode(p)), orc.quantize_fs(bits, fmt, amax, (1, 64)))
    finally:
        exmy.force_generic(False)


def test_fig2_on_gpu(exmy):
    """the block max 3.9 under e2m1 comes back exactly."""
    t = torch.tensor([[3.9, 0.1, -1.0, 2.0, 0.5, 0.25, 3.0, 1.5]] * 8, dtype=torch.float32, device=DEV)
    q = exmy.quantize_fs(t, "e2m1", None, "row")
    assert torch.all(q[:, 0] == torch.tensor(3.9, dtype=torch.float32))
    p = exmy.encode_fs(t, "e2m1", None, "row")
    assert torch.equal(exmy.decode(p), q)


def test_fs_config2_shape_sampled(exmy, orc):
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=DEV)
    sc = exmy.block_float_scale(t, "row")
    p = exmy.encode_fs(t, "e3m3", sc, "row")
    q = exmy.quantize_fs(t, "e3m3", sc, "row")
    assert torch.equal(exmy.decode(p).view(torch.int16), q.view(torch.int16))
    ws, offs = exmy.segments(7, R * C)
    for r0 in (0, 8 * 1234, R - 8):
        rows = W.to_bits(t[r0:r0 + 8])
        amax = sc[r0:r0 + 8].cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(amax, orc.block_float_scale(rows, (1, C)))
        ref = orc.encode_fs(rows, "e3m3", amax, (1, C), orc.ROWS)[0]
        got = torch.cat([p.data[o + r0 * C * w // 8: o + (r0 + 8) * C * w // 8] for w, o in zip(ws, offs)])
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
        np.testing.assert_array_equal(W.to_bits(q[r0:r0 + 8]), orc.quantize_fs(rows, "e3m3", amax, (1, C)))


def amax_rows(k, seed):
    """per-row maxima over the whole fp32 range: fp32-subnormal, tiny, normal,
    huge, and significands divisible by G's odd part (exact binary results)"""
    rng = np.random.default_rng(seed)
    a = list((rng.random(40) * 2.0 ** rng.integers(-149, 128, 40)).astype(np.float32).view(np.uint32))
    a += [1, 3, 0x7FFFFF, 0x00800000, 0x7F7FFFFF, 0x3F800000, 15 * 12345, 0x0D800000, 0x0C000001]
    for _ in range(16):
        e = int(rng.integers(1, 255))
        sig = int(rng.integers(1 << 23, 1 << 24))
        sig -= sig % 7
        a.append((e << 23) | (sig & 0x7FFFFF) if sig >= 1 << 23 else sig)
    a = [int(v) for v in a if v != 0]
    return np.array(a[:64] + [a[0]] * (64 - len(a[:64])), np.uint32)


@pytest.mark.parametrize("fmt", [(3, 3), (2, 1), (4, 2), (0, 6), (6, 0), (1, 5), (8, 0), (7, 1), (2, 5), (5, 3),
                                 (4, 4), (3, 2)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("od", ["f32", "bf16"])
def test_fs_decode_every_code_every_range(exmy, orc, fmt, od):
    """decode = RN32(g amax / G) (reading D23's plain definition): every code
    of the format in every row, rows with maxima across the whole fp32 range
    (results down to fp32 subnormals and zero), ROWS fast kernel and the
    generic (COLS) kernel, both output dtypes -- == the oracle bit for bit."""
    x, y = fmt
    k = 1 + x + y
    C = max(1 << k, 64)
    R = 64
    codes = np.tile(np.arange(C, dtype=np.uint16) % (1 << k), (R, 1))
    amax = amax_rows(k, 100 * k + x)[:, None]
    for axis, ax in (("rows", orc.ROWS), ("cols", orc.COLS)):
        packed = orc.pack(codes, (R, C), ax, k)
        p = exmy.Packed(torch.from_numpy(packed).to(DEV), torch.full((1,), 127, dtype=torch.uint8, device=DEV),
                        torch.zeros(1, dtype=torch.int64, device=DEV), torch.zeros(1, dtype=torch.int32, device=DEV),
                        torch.zeros(1, dtype=torch.int64, device=DEV), (R, C), x, y, exmy.ROWS if ax == orc.ROWS
                        else exmy.COLS, torch.float32, (1, C), None,
                        torch.from_numpy(amax.view(np.float32).copy()).to(DEV), sp_capacity=0, scheme=2)
        dt = torch.float32 if od == "f32" else torch.bfloat16
        got = W.to_bits(exmy.decode(p, dt))
        ref = orc.decode_fs(packed, (R, C), fmt, amax, (1, C), ax, out_dtype=np.uint32 if od == "f32" else np.uint16)
        np.testing.assert_array_equal(got, ref, err_msg=axis)
