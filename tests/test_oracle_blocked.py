"""Pins of the oracle's block-metadata functions:
block metadata before / after rounding, and blocked quantize / encode /
decode -- checked against the paper's Fig. 2 narrative, against the
per-tensor oracle applied block by block (an independent indexing path),
and against library roundings for the "after rounding" exponent."""
import ml_dtypes
import numpy as np
import pytest
import torch

import workloads as W


def f32bits(v):
    return np.asarray(v, dtype=np.float32).view(np.uint32)


def test_fig2_scheme_values(orc):
    """3.9 under e2m1 -> 3.0 with the max exponent taken before
    rounding (metadata 128 = 3.9's exponent), 4.0 after rounding (3.9 rounds
    to 4.0 at y=1, metadata 129).  S:161-164 gives the [3.9, 0.1] block."""
    blk = f32bits([[3.9, 0.1]])
    before = orc.block_max_exponent(blk, (1, 2), y=1, scheme=orc.SCHEME_MAX_BEFORE)
    after = orc.block_max_exponent(blk, (1, 2), y=1, scheme=orc.SCHEME_MAX_AFTER)
    assert before.tolist() == [[128]] and after.tolist() == [[129]]
    qb = orc.quantize_blocked(blk, "e2m1", before, (1, 2)).view(np.float32)
    qa = orc.quantize_blocked(blk, "e2m1", after, (1, 2)).view(np.float32)
    assert qb[0, 0] == 3.0 and qa[0, 0] == 4.0


@pytest.mark.parametrize("y,rnd", [(7, "bf16"), (3, "e4m3"), (2, "e5m2")])
def test_after_rounding_exponent_vs_libraries(orc, y, rnd):
    """The 'after rounding' exponent is the exponent of |v| rounded RTNE to y
    mantissa bits: for y = 7 that is torch's fp32 -> bf16 cast, for y = 3 / 2
    the OCP fp8 casts (in their normal range)."""
    rng = np.random.default_rng(y)
    v = (rng.standard_normal(20000) * 2.0 ** rng.integers(-5, 6, 20000)).astype(np.float32)
    # include exact carries: values just below powers of two
    v[:200] = np.nextafter(np.float32(2.0) ** rng.integers(-5, 6, 200).astype(np.float32), np.float32(0))
    if rnd == "bf16":
        r = torch.from_numpy(np.abs(v)).to(torch.bfloat16).to(torch.float32).numpy()
    else:
        dt, lo, hi = (ml_dtypes.float8_e4m3fn, 2.0 ** -6, 400.0) if rnd == "e4m3" else \
            (ml_dtypes.float8_e5m2, 2.0 ** -14, 50000.0)
        v = v[(np.abs(v) >= lo) & (np.abs(v) < hi)]          # the fp8 normal range
        r = np.abs(v).astype(dt).astype(np.float32)
    expect = ((r.view(np.uint32) >> 23) & 0xFF).astype(np.uint8)
    got = orc.block_max_exponent(f32bits(v).reshape(-1, 1), (1, 1), y=y, scheme=orc.SCHEME_MAX_AFTER).reshape(-1)
    np.testing.assert_array_equal(got, expect)


def test_before_is_exponent_field_max(orc):
    bits = W.random_bits_f32(64 * 48, 3).reshape(64, 48)
    m = orc.block_max_exponent(bits, (8, 16))
    e = ((bits >> 23) & 0xFF).astype(np.int64)
    e[e == 255] = -1
    ref = e.reshape(8, 8, 3, 16).max(axis=(1, 3)).clip(0, 254)
    np.testing.assert_array_equal(m, ref)


def test_schemes_ordering_and_degenerate(orc):
    """after >= before, differing by at most 1; all-zero / all-special
    blocks get metadata 0."""
    bits = W.to_bits(W.f32_wide((32, 64), seed=4))
    for y in (0, 1, 3, 7):
        b = orc.block_max_exponent(bits, (4, 8), y, orc.SCHEME_MAX_BEFORE).astype(int)
        a = orc.block_max_exponent(bits, (4, 8), y, orc.SCHEME_MAX_AFTER).astype(int)
        assert np.all(a >= b) and np.all(a - b <= 1)
    z = np.zeros((8, 8), np.uint32)
    z[0:4] = 0x7FC00000
    assert orc.block_max_exponent(z, (4, 8)).tolist() == [[0], [0]]


@pytest.mark.parametrize("block", [(1, 64), (64, 1), (8, 16), (1, 16), (64, 64)])
@pytest.mark.parametrize("fmt", ["e3m2", "e2m1", "e0m4", "e5m3"])
def test_blocked_equals_per_block_oracle(orc, block, fmt):
    """Blocked quantize/encode/decode == the per-tensor oracle run on each
    block separately (blocks are independent tensors)."""
    t = W.bf16_weights((64, 64), seed=block[0] * 100 + block[1], std=0.02)
    bits = W.to_bits(t)
    # rows of very different magnitude
    scale = (2.0 ** np.arange(-6, 58, 1)).astype(np.float32)[:64, None]
    bits = W.to_bits(torch.from_numpy((t.float().numpy() * scale).astype(np.float32)).to(torch.bfloat16))
    meta = orc.block_max_exponent(bits, block)
    q = orc.quantize_blocked(bits, fmt, meta, block)
    br, bc = block
    for i in range(64 // br):
        for j in range(64 // bc):
            sub = bits[i * br:(i + 1) * br, j * bc:(j + 1) * bc]
            np.testing.assert_array_equal(q[i * br:(i + 1) * br, j * bc:(j + 1) * bc],
                                          orc.quantize(sub, fmt, int(meta[i, j])))
    for axis in (orc.ROWS, orc.COLS):
        p, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, block, axis)
        d = orc.decode_blocked(p, bits.shape, fmt, meta, block, axis, idx, sb, np.uint16)
        np.testing.assert_array_equal(d, q)
        codes = orc.unpack(p, bits.shape, axis, 1 + sum(orc.parse_format(fmt)))
        for i in range(64 // br):
            for j in range(64 // bc):
                sub = bits[i * br:(i + 1) * br, j * bc:(j + 1) * bc]
                np.testing.assert_array_equal(codes[i * br:(i + 1) * br, j * bc:(j + 1) * bc],
                                              orc.encode_codes(sub, fmt, int(meta[i, j])).reshape(sub.shape))


def test_after_scheme_keeps_block_max(orc):
    """with the max exponent after rounding, the block maximum is
    never truncated by saturation: it quantizes to itself rounded to y bits."""
    t = W.f32_wide((16, 32), seed=9)
    bits = W.to_bits(t)
    for fmt in ("e2m1", "e3m2", "e1m2"):
        x, y = orc.parse_format(fmt)
        m = orc.block_max_exponent(bits, (1, 32), y, orc.SCHEME_MAX_AFTER)
        q = orc.quantize_blocked(bits, fmt, m, (1, 32)).view(np.float32)
        a = np.abs(t.numpy())
        rows_max = a.max(axis=1)
        qmax = np.abs(q)[np.arange(16), a.argmax(axis=1)]
        # rounded to y mantissa bits in its own binade
        e = np.floor(np.log2(rows_max.astype(np.float64)))
        ref = np.round(rows_max / 2.0 ** (e - y)) * 2.0 ** (e - y)   # no exact ties in this data
        np.testing.assert_array_equal(qmax.astype(np.float64), ref)


def test_block_shape_validation(orc):
    with pytest.raises(ValueError):
        orc.block_max_exponent(np.zeros((8, 8), np.uint32), (3, 8))
    assert orc.lib().oracle_block_shape_ok(8, 8, 8, 8) == 1


@pytest.mark.parametrize("y", [0, 1, 2, 5])
def test_after_rounding_exponent_fractions(orc, y):
    """Reading D22 with Fractions, every y incl. y = 0: the 'after rounding'
    exponent of a normal fp32 value a in [2^E, 2^(E+1)) is E, or E + 1 when a
    rounds (RTNE with y mantissa bits) up to 2^(E+1); a tie goes to the
    representation whose last kept bit is 0 -- the mantissa LSB for y >= 1,
    the exponent LSB for y = 0 (the same rule as quantize's D6).  Every exact
    tie and its fp32 neighbours are included; a second check uses the paper's
    Eigen procedure on the bits (the exponent field of the rounded pattern)."""
    from fractions import Fraction as F
    rng = np.random.default_rng(70 + y)
    E = rng.integers(1, 250, 3000)
    mant = rng.integers(0, 1 << 23, 3000)
    sh = 23 - y
    mant[::3] = (mant[::3] & ~((1 << sh) - 1)) | (1 << (sh - 1))            # exact ties
    mant[1::3] = (mant[1::3] & ~((1 << sh) - 1)) | ((1 << (sh - 1)) - 1)    # one ulp below a tie
    mant[:40] = (1 << 23) - 1                                             # carries into the next binade
    bits = ((E << 23) | mant).astype(np.uint32)
    got = orc.block_max_exponent(bits.reshape(-1, 1), (1, 1), y=y, scheme=orc.SCHEME_MAX_AFTER).reshape(-1)
    for b, g, e, m in zip(bits.tolist(), got.tolist(), E.tolist(), mant.tolist()):
        frac = F(m, 1 << 23) * (1 << y)               # mantissa in units of the kept LSB
        n, r = divmod(frac, 1)
        n = int(n)
        last_odd = (n & 1) if y >= 1 else (e & 1)     # the last kept bit: mantissa LSB / exponent LSB
        up = r > F(1, 2) or (r == F(1, 2) and last_odd)
        want = e + 1 if (up and n + 1 == 1 << y) else e
        assert g == min(want, 254), (hex(b), g, want)
    eig = eigen_round(bits, y)
    np.testing.assert_array_equal(got, np.minimum((eig >> 23) & 0xFF, 254).astype(np.uint8))


def eigen_round(u, y):
    sh = 23 - y
    u = u.astype(np.uint64)
    r = u + ((1 << (sh - 1)) - 1) + ((u >> sh) & 1)
    return (r & ~np.uint64((1 << sh) - 1)).astype(np.uint64)
