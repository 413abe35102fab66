"""Pins of the oracle's float-scaling scheme (Fig. 2's third scheme, P:254-275,
"float scaling with maximum exponent of 127"; reading D23 in DESIGN.md),
checked against exact rational arithmetic (Python Fractions), the paper's
3.9 example, the other schemes' oracle on inputs where they must agree, and
numpy for the block maxima."""
from fractions import Fraction

import numpy as np
import pytest

import workloads as W

FMTS = [(2, 1), (3, 2), (3, 3), (4, 3), (5, 2), (1, 5), (0, 6), (6, 0), (8, 0), (2, 5), (3, 5), (0, 2)]


def f32(bits):
    return np.array([bits], np.uint32).view(np.float32)[0]


def frac_of_f32(bits):
    return Fraction(float(f32(bits)))


def rn32(fr: Fraction) -> int:
    """fp32 bits of the correctly rounded (ties to even) value of fr; written
    from the IEEE definition with integers, independent of the oracle."""
    if fr == 0:
        return 0
    sign = 0x80000000 if fr < 0 else 0
    a = abs(fr)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                       # subnormal quantum below 2^-126
    q = Fraction(2) ** (e - 23)
    n, r = divmod(a.numerator * q.denominator, a.denominator * q.numerator)
    # a/q = n + r/(den)
    den = a.denominator * q.numerator
    if 2 * r > den or (2 * r == den and n & 1):
        n += 1
    if n == 1 << 24:
        n >>= 1
        e += 1
    if n < 1 << 23:
        return sign | n                    # subnormal
    return sign | ((e + 127) << 23) | (n - (1 << 23))


def test_rn32_helper_against_numpy():
    rng = np.random.default_rng(0)
    v = rng.standard_normal(2000) * 2.0 ** rng.integers(-140, 100, 2000)
    for d in v:
        assert rn32(Fraction(float(d))) == int(np.array([d], np.float64).astype(np.float32).view(np.uint32)[0])


def test_fig2_float_scale_keeps_the_max(orc):
    """P:270-273 / S:537: block [3.9, 0.1] under e2m1 -> 3.0 (max before),
    4.0 (max after), 3.9 exactly (float scaling)."""
    b = np.array([[3.9, 0.1]], np.float32).view(np.uint32)
    amax = orc.block_float_scale(b, (1, 2))
    assert amax[0, 0] == b[0, 0]
    q = orc.quantize_fs(b, "e2m1", amax, (1, 2)).view(np.float32)
    assert q[0, 0] == np.float32(3.9)
    qb = orc.quantize_blocked(b, "e2m1", orc.block_max_exponent(b, (1, 2)), (1, 2)).view(np.float32)
    assert qb[0, 0] == 3.0


def test_grid_top_values(orc):
    """G = the largest magnitude at e_max 127: (2 - 2^-y) for x >= 1 (top
    binade [1, 2)), (2^y - 1) 2^(1-y) for x = 0 (fixed point, bias 0)."""
    for x, y in FMTS:
        g = orc.fs_grid_top((x, y))
        want = (2.0 - 2.0 ** -y) if x >= 1 else (2 ** y - 1) * 2.0 ** (1 - y)
        assert g == want, (x, y)


@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_block_max_decodes_exactly(orc, fmt, dt):
    """'captures the largest value in the block accurately': the
    element holding the block max quantizes back to exactly amax."""
    t = W.f32_wide((32, 64), seed=fmt[0] * 16 + fmt[1])
    if dt == "bf16":
        import torch
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t)
    for block in [(1, 64), (4, 16), (32, 64), (1, 8)]:
        amax = orc.block_float_scale(bits, block)
        q = orc.quantize_fs(bits, fmt, amax, block)
        br, bc = block
        for i in range(32 // br):
            for j in range(64 // bc):
                sub = bits[i * br:(i + 1) * br, j * bc:(j + 1) * bc]
                qs = q[i * br:(i + 1) * br, j * bc:(j + 1) * bc]
                if dt == "bf16":
                    mag = sub & 0x7FFF
                else:
                    mag = sub & 0x7FFFFFFF
                pos = np.unravel_index(np.argmax(mag), mag.shape)
                assert (qs[pos] & (0x7FFF if dt == "bf16" else 0x7FFFFFFF)) == mag[pos]


def test_block_float_scale_is_numpy_max(orc):
    bits = W.to_bits(W.f32_wide((16, 48), seed=3))
    bits[3, 5] = 0x7FC00000           # NaN ignored
    bits[7, :] = 0                    # zero row -> 0
    a = orc.block_float_scale(bits, (1, 48))
    v = np.abs(bits.view(np.float32))
    v[~np.isfinite(v)] = 0
    np.testing.assert_array_equal(a.view(np.float32)[:, 0], v.max(axis=1))


@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f"e{f[0]}m{f[1]}")
def test_scale_in_is_exact_rounding(orc, fmt):
    """u = RN32(v * RN32(G / A1) * 2^-p), amax = A1 2^p: each rounding checked
    with Fractions."""
    rng = np.random.default_rng(fmt[1])
    G = Fraction(orc.fs_grid_top(fmt))
    amaxs = (rng.random(40) * 2.0 ** rng.integers(-140, 120, 40)).astype(np.float32)
    amaxs[:3] = [3.9, 1.0, 2.0 ** -149]
    for a in amaxs:
        ab = int(np.array([a], np.float32).view(np.uint32)[0])
        A = frac_of_f32(ab)
        p = 0
        while A >= 2:
            A /= 2
            p += 1
        while A < 1:
            A *= 2
            p -= 1
        r = frac_of_f32(rn32(G / A))
        vs = (rng.random(20) * float(a) * rng.choice([-1, 1], 20)).astype(np.float32)
        for v in np.append(vs, [a, -a, 0.0]).astype(np.float32):
            vb = int(np.array([v], np.float32).view(np.uint32)[0])
            want = rn32(Fraction(float(v)) * r / Fraction(2) ** p) if p >= 0 else \
                rn32(Fraction(float(v)) * r * Fraction(2) ** (-p))
            if want == 0:
                want = vb & 0x80000000              # a zero product keeps v's sign
            assert orc.fs_scale_in(vb, ab, fmt) == want


def code_value_fr(code: int, x: int, y: int) -> Fraction:
    """exact value of a k-bit code at e_max 127 (bias 2^x - 1, D1), written
    from Table 1 / P:172-175 in Fractions (the oracle's grid is pinned to
    ml_dtypes in test_oracle_pins)"""
    k = 1 + x + y
    s = -1 if (code >> (k - 1)) & 1 else 1
    mag = code & ((1 << (k - 1)) - 1)
    bias = (1 << x) - 1
    e = 0 if x == 0 else mag >> y
    m = mag & ((1 << y) - 1)
    if e == 0:
        return s * Fraction(m) * Fraction(2) ** (1 - bias - y)
    return s * Fraction((1 << y) + m) * Fraction(2) ** (e - bias - y)


def numpy_rn32(fr: Fraction) -> int:
    """RN32 by numpy's float64 -> float32 conversion of RN64(fr).  Exact here:
    for fr = g * amax / G the double rounding could only go wrong if RN64(fr)
    landed on an fp32 midpoint while fr did not; fr's distance from any fp32
    midpoint is either 0 or >= 2^-42 relative (normal results) / >= 2^-33 of
    the value (subnormal results), both far above RN64's 2^-53."""
    return int(np.array([float(fr)], np.float64).astype(np.float32).view(np.uint32)[0])


def amax_sample(rng, fmt, n=48):
    """random maxima over the whole fp32 range (subnormal ones included) plus
    maxima whose significand is divisible by the odd part of G's (so that
    g * amax / G is an exact binary fraction, possibly an fp32 midpoint) and
    the extremes"""
    x, y = fmt
    MG = (2 << y) - 1 if x >= 1 else (1 << y) - 1
    a = list((rng.random(n) * 2.0 ** rng.integers(-149, 128, n)).astype(np.float32).view(np.uint32))
    for _ in range(n // 2):
        q = int(rng.integers(1, (1 << 24) // max(MG, 1)))
        sig = q * max(MG, 1)
        if sig >= 1 << 24:
            continue
        e = int(rng.integers(-149, 104))
        v = np.float32(np.ldexp(float(sig), e))
        if np.isfinite(v) and v > 0:
            a.append(int(np.array([v], np.float32).view(np.uint32)[0]))
    a += [0x00000001, 0x007FFFFF, 0x00800000, 0x7F7FFFFF, 0x3F800000,
          int(np.array([3.9], np.float32).view(np.uint32)[0])]
    return [int(v) for v in a if v != 0]      # amax = 0 is its own case (test_zero_and_special_blocks)


@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f"e{f[0]}m{f[1]}")
def test_scale_out_is_the_plain_definition(orc, fmt):
    """Decode (reading D23) = RN32(g * amax / G) exactly, g the code's exact
    value at e_max 127: for EVERY code (incl. e8m0 values below the fp32
    range and fp32-subnormal results) under maxima spanning the fp32 range,
    against (a) round-to-nearest-even of the exact Fraction, written here from
    the IEEE definition, and (b) numpy's float32 conversion (see numpy_rn32).
    Zero results keep the code's sign."""
    x, y = fmt
    k = 1 + x + y
    rng = np.random.default_rng(100 + k + 10 * x)
    G = code_value_fr((1 << (k - 1)) - 1, x, y)
    assert G == Fraction(orc.fs_grid_top(fmt))
    for ab in amax_sample(rng, fmt):
        A = frac_of_f32(ab)
        for code in range(1 << k):
            g = code_value_fr(code, x, y)
            exact = g * A / G
            got = orc.fs_scale_out(code, ab, fmt)
            sign = 0x80000000 if (code >> (k - 1)) & 1 else 0
            want = rn32(exact) if exact != 0 else sign
            if want & 0x7FFFFFFF == 0:
                want = sign                       # a zero result keeps the code's sign
            assert got == want, (code, hex(ab))
            assert (got & 0x7FFFFFFF) == (numpy_rn32(abs(exact)) if exact != 0 else 0), (code, hex(ab))
        assert orc.fs_scale_out((1 << (k - 1)) - 1, ab, fmt) == ab        # the block max comes back


@pytest.mark.parametrize("fmt", [(2, 3), (3, 3), (1, 5), (3, 5), (0, 6), (2, 1), (4, 3), (7, 1)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
def test_scale_out_ties_only_in_the_subnormal_range(orc, fmt):
    """Where can g * amax / G sit exactly halfway between two fp32 values?
    With g = M_g 2^a, amax = M_a 2^b, G = M_G 2^c (M_* odd-free integers,
    M_g <= M_G, M_a < 2^24), an exact binary fraction needs M_G | M_g M_a and
    then has the integer significand M_g M_a / M_G < 2^24: it is an fp32
    value in the normal range, never a midpoint.  Ties therefore only occur
    among fp32-subnormal results (quantum 2^-149): there the plain definition
    sends them to the even pattern, as numpy's RTNE conversion of the (exactly
    representable) double midpoint does.  (For x <= 1 every code shares G's
    quantum, so even subnormal exact results are fp32 values: no ties.)"""
    x, y = fmt
    k = 1 + x + y
    MG = (2 << y) - 1 if x >= 1 else (1 << y) - 1
    G = code_value_fr((1 << (k - 1)) - 1, x, y)
    rng = np.random.default_rng(7 * k + x)
    ties = 0
    for it in range(3000):
        if it % 2:       # an fp32-subnormal maximum whose significand M_G divides
            ab = MG * int(rng.integers(1, (1 << 23) // MG))
        else:            # a normal one (biased exponent 1..40: small results)
            sig = MG * int(rng.integers(((1 << 23) + MG - 1) // MG, (1 << 24) // MG))
            ab = (int(rng.integers(1, 41)) << 23) | (sig - (1 << 23))
        A = frac_of_f32(ab)
        for code in rng.integers(1, 1 << (k - 1), 6):
            exact = code_value_fr(int(code), x, y) * A / G
            scaled = exact * Fraction(2) ** 150                   # in units of half the subnormal quantum
            if exact >= Fraction(2) ** -126:
                # normal range: exact binary fractions are fp32 values
                if exact.denominator & (exact.denominator - 1) == 0:
                    assert rn32(exact) == numpy_rn32(exact) and frac_of_f32(rn32(exact)) == exact
                continue
            if scaled.denominator == 1 and scaled.numerator % 2 == 1:   # an odd multiple of 2^-150: a tie
                got = orc.fs_scale_out(int(code), ab, fmt)
                assert got == rn32(exact) == numpy_rn32(exact)
                assert got & 1 == 0
                ties += 1
    assert ties >= 3 if x >= 2 else ties == 0, ties


def test_factor_is_correctly_rounded(orc):
    """the encode factor RN32(G / A1) vs numpy (G / A1 is never within 2^-53
    of an fp32 midpoint unless exactly on it) and Fractions"""
    rng = np.random.default_rng(11)
    for fmt in FMTS:
        G = code_value_fr((1 << (fmt[0] + fmt[1])) - 1, *fmt)
        for ab in amax_sample(rng, fmt, 16):
            A = frac_of_f32(ab)
            while A >= 2:
                A /= 2
            while A < 1:
                A *= 2
            assert orc.fs_factor(ab, fmt) == rn32(G / A) == numpy_rn32(G / A), (fmt, hex(ab))


@pytest.mark.parametrize("fmt", [(2, 1), (3, 3), (4, 2), (1, 4), (5, 0), (6, 1)], ids=lambda f: f"e{f[0]}m{f[1]}")
def test_power_of_two_scale_reduces_to_max_before(orc, fmt):
    """If amax = G * 2^s exactly, the scale is the power of two 2^s and float
    scaling coincides with the plain per-block scheme at e_max = 127 + s
    (another oracle path: grid search at a different metadata value)."""
    rng = np.random.default_rng(5)
    G = orc.fs_grid_top(fmt)
    rows = []
    for s in (-20, -3, 0, 5, 40):
        r = (rng.random(16) * 2 - 1) * G * 2.0 ** s
        r[3] = G * 2.0 ** s          # the block max, exactly G 2^s
        rows.append(r)
    t = np.array(rows, np.float32)
    bits = t.view(np.uint32)
    amax = orc.block_float_scale(bits, (1, 16))
    meta = orc.block_max_exponent(bits, (1, 16))
    np.testing.assert_array_equal(meta[:, 0], [107, 124, 127, 132, 167])
    for axis in (orc.ROWS, orc.COLS):
        if axis == orc.ROWS:
            b8 = np.concatenate([bits, bits[:3]])            # 8 rows
            a8 = np.concatenate([amax, amax[:3]])
            m8 = np.concatenate([meta, meta[:3]])
        else:
            b8, a8, m8 = bits, amax, meta
        pf = orc.encode_fs(b8, fmt, a8, (1, 16), axis)[0]
        pb = orc.encode_blocked(b8, fmt, m8, (1, 16), axis)[0]
        np.testing.assert_array_equal(pf, pb)
    np.testing.assert_array_equal(orc.quantize_fs(bits, fmt, amax, (1, 16)),
                                  orc.quantize_blocked(bits, fmt, meta, (1, 16)))


def test_zero_and_special_blocks(orc):
    bits = np.zeros((8, 16), np.uint32)
    bits[0, :] = 0x80000000                  # -0
    bits[1, 2] = 0x7F800000                  # +Inf only (block max stays 0)
    bits[2, :] = W.to_bits(W.f32_wide((1, 16), seed=1))
    bits[2, 7] = 0x7FC00001                  # NaN payload
    amax = orc.block_float_scale(bits, (1, 16))
    assert amax[0, 0] == 0 and amax[1, 0] == 0 and amax[2, 0] != 0
    q = orc.quantize_fs(bits, "e3m2", amax, (1, 16))
    np.testing.assert_array_equal(q[0], bits[0])          # signed zeros kept
    assert q[1, 2] == 0x7F800000 and q[2, 7] == 0x7FC00001
    for axis in (orc.ROWS, orc.COLS):
        p, idx, sb, ns = orc.encode_fs(bits, "e3m2", amax, (1, 16), axis)
        assert ns == 2 and list(idx) == [18, 39]
        d = orc.decode_fs(p, bits.shape, "e3m2", amax, (1, 16), axis, idx, sb, out_dtype=np.uint32)
        np.testing.assert_array_equal(d, q)


@pytest.mark.parametrize("fmt", ["e2m1", "e3m3", "e0m5", "e5m3"])
def test_encode_decode_equals_quantize(orc, fmt):
    t = W.bf16_weights((16, 64), seed=2)
    bits = W.to_bits(t)
    for block in [(1, 64), (8, 8), (16, 1)]:
        amax = orc.block_float_scale(bits, block)
        q = orc.quantize_fs(bits, fmt, amax, block)
        for axis in (orc.ROWS, orc.COLS):
            p = orc.encode_fs(bits, fmt, amax, block, axis)[0]
            np.testing.assert_array_equal(orc.decode_fs(p, bits.shape, fmt, amax, block, axis), q)
