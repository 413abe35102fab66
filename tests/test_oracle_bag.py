"""Pins of the oracle's embedding bag (reading D25): pooled
rows == the oracle's own full decode (an independent unpack path) summed by
numpy in fp32 in index order; weighted pooling == Fraction-exact fused
multiply-add rounding; mean; empty bags; per-row metadata."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import workloads as W


def rn32(fr: Fraction) -> np.float32:
    """correctly rounded fp32 of an exact rational (ties to even), via two
    doubles that bracket it: exact enough here (values have < 80 bits)"""
    f = float(fr)                                    # RN64 (Fraction.__float__ is correctly rounded)
    a = np.float32(f)
    if Fraction(float(a)) == fr:
        return a
    # decide with the exact value against the fp32 neighbours' midpoint
    lo = np.nextafter(a, np.float32(-np.inf)) if Fraction(float(a)) > fr else a
    hi = np.nextafter(lo, np.float32(np.inf))
    mid = (Fraction(float(lo)) + Fraction(float(hi))) / 2
    if fr < mid:
        return lo
    if fr > mid:
        return hi
    return lo if (int(np.array([lo], np.float32).view(np.uint32)[0]) & 1) == 0 else hi


def table(orc, rows, cols, fmt, seed, per_row=False):
    t = W.f32_embedding(rows, cols, seed=seed)
    t = t * torch.exp2(torch.randint(-6, 6, (rows, 1), generator=torch.Generator().manual_seed(seed)).float())
    bits = W.to_bits(t)
    if per_row:
        meta = orc.block_max_exponent(bits, (1, cols))
        packed = orc.encode_blocked(bits, fmt, meta, (1, cols), orc.COLS)[0]
        dec = orc.decode_blocked(packed, (rows, cols), fmt, meta, (1, cols), orc.COLS, out_dtype=np.uint32)
        meta = meta.reshape(-1)
    else:
        e = orc.emax(orc.histogram(bits))
        packed = orc.encode(bits, fmt, e, orc.COLS)[0]
        dec = orc.decode(packed, (rows, cols), fmt, e, orc.COLS, out_dtype=np.uint32)
        meta = np.array([e], np.uint8)
    return packed, meta, dec.view(np.float32)


@pytest.mark.parametrize("fmt", ["e4m2", "e3m1", "e2m4"])
@pytest.mark.parametrize("per_row", [False, True])
def test_bag_sum_mean_vs_numpy(orc, fmt, per_row):
    rows, cols = 200, 64
    packed, meta, dec = table(orc, rows, cols, fmt, 3, per_row)
    rng = np.random.default_rng(1)
    sizes = rng.integers(0, 9, size=40)
    sizes[:3] = [0, 1, 7]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = rng.integers(0, rows, size=int(offsets[-1])).astype(np.int64)
    for mode in ("sum", "mean"):
        got = orc.embedding_bag(packed, (rows, cols), fmt, meta, idx, offsets, mode=mode)
        for b in range(len(sizes)):
            acc = np.zeros(cols, np.float32)
            for i in range(offsets[b], offsets[b + 1]):
                acc = (acc + dec[idx[i]]).astype(np.float32)     # fp32 adds in index order
            if mode == "mean" and sizes[b]:
                acc = (acc / np.float32(sizes[b])).astype(np.float32)
            np.testing.assert_array_equal(got[b], acc, err_msg=f"bag {b} {mode}")
    # a one-row bag is that row's decode
    one = orc.embedding_bag(packed, (rows, cols), fmt, meta, np.array([17], np.int64), np.array([0, 1], np.int64))
    np.testing.assert_array_equal(one[0], dec[17])


def test_bag_weighted_is_exact_fma(orc):
    rows, cols = 50, 16
    packed, meta, dec = table(orc, rows, cols, "e3m3", 5)
    rng = np.random.default_rng(2)
    idx = rng.integers(0, rows, size=6).astype(np.int64)
    w = rng.standard_normal(6).astype(np.float32)
    got = orc.embedding_bag(packed, (rows, cols), "e3m3", meta, idx, np.array([0, 6], np.int64), weights=w)
    for c in range(cols):
        acc = np.float32(0)
        for i in range(6):
            acc = rn32(Fraction(float(w[i])) * Fraction(float(dec[idx[i], c])) + Fraction(float(acc)))
        assert got[0, c] == acc
