"""GPU parity of the fused decode + matrix-vector product (exmy_gemv;
reading D26) against the oracle: the oracle decodes the
packed bytes (exact fp32 values, NaN/Inf restored from the specials list),
numpy forms act @ W.T in fp64, and every finite output must lie within the
fp32 dot-product error bound |err| <= K u / (1 - K u) * sum |act| |W| (+ the
subnormal floor), u = 2^-24, whatever the summation order; NaN / +-Inf
outputs must match exactly.  The bound alone could hide one wrong term, so
test_gemv_one_hot_exact pins the decode inside the product bit for bit:
one-hot activation rows make every output a single exact product, i.e. one
decoded weight.  Per-tensor and per-row metadata, formats of width 3..8,
ragged column tiles, 1..11 activation rows (passes of 8 / 4 / 2 / 1)."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"
U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def exmy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as m
    m.force_generic(False)
    return m


def _weights(shape, seed, specials):
    rng = np.random.default_rng(seed)
    t = W.bf16_weights(shape, seed=seed).float()
    t = t * torch.exp2(torch.from_numpy(rng.integers(-12, 12, size=(shape[0], 1))).float())
    bits = W.to_bits(t.to(torch.bfloat16))
    if specials:
        flat = bits.reshape(-1)
        k = rng.choice(flat.size, 6, replace=False)
        flat[k[:2]] = 0x7FC0          # NaN
        flat[k[2:4]] = 0x7F80         # +Inf
        flat[k[4:]] = 0xFF80          # -Inf
    return bits


def _check(out, ref, bound):
    out = out.astype(np.float64)
    assert np.array_equal(np.isnan(out), np.isnan(ref)), "NaN pattern"
    assert np.array_equal(np.isposinf(out), np.isposinf(ref)), "+Inf pattern"
    assert np.array_equal(np.isneginf(out), np.isneginf(ref)), "-Inf pattern"
    fin = np.isfinite(ref)
    err = np.abs(out[fin] - ref[fin])
    assert np.all(err <= bound[fin]), f"max err / bound {np.max(err / np.maximum(bound[fin], 1e-300)):.3g}"


def _reference(orc, p, bits_shape, fmt, meta, per_row, act):
    pk = p.data.cpu().numpy()
    spi, spb, cnt = p.specials()
    spi, spb = spi.cpu().numpy(), spb.cpu().numpy().view(np.uint32)
    if per_row:
        dec = orc.decode_blocked(pk, bits_shape, fmt, meta, (1, bits_shape[1]), orc.ROWS, spi, spb,
                                 out_dtype=np.uint32)
    else:
        dec = orc.decode(pk, bits_shape, fmt, int(meta[0]), orc.ROWS, spi, spb, out_dtype=np.uint32)
    w = dec.view(np.float32).astype(np.float64)
    a = act.astype(np.float64)
    with np.errstate(invalid="ignore", over="ignore"):
        ref = a @ w.T
        wf = np.where(np.isfinite(w), np.abs(w), 0.0)
        mag = np.abs(a) @ wf.T
    K = bits_shape[1]
    g = K * U32 / (1 - K * U32)
    return ref, g * mag + K * 2.0 ** -149


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (4, 3), (6, 0), (0, 6), (1, 1), (5, 2), (3, 4), (7, 0)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("per_row", [False, True])
def test_gemv_parity(exmy, orc, fmt, per_row):
    for shape, ms, specials in (((64, 1024), (1, 3), False), ((72, 4100), (2, 11), True), ((8, 4), (1, 8), True),
                                ((40, 6160), (1, 5, 8), True)):
        bits = _weights(shape, shape[0] + shape[1], specials)
        d = W.from_bits(bits).to(DEV)
        if per_row:
            meta = orc.block_max_exponent(bits, (1, shape[1]))
            p = exmy.encode_blocked(d, fmt, torch.from_numpy(meta.copy()).to(DEV), (1, shape[1]),
                                    specials_capacity=64)
            meta = meta.reshape(-1)
        else:
            e = orc.emax(orc.histogram(bits))
            p = exmy.encode(d, fmt, e, specials_capacity=64)
            meta = np.array([e], np.uint8)
        for m in ms:
            act = torch.randn(m, shape[1], generator=torch.Generator().manual_seed(m)).numpy().astype(np.float32)
            act[0, :3] = 0.0                     # 0 x Inf = NaN where a special sits there
            out = exmy.gemv(p, torch.from_numpy(act).to(DEV)).cpu().numpy()
            ref, bound = _reference(orc, p, shape, fmt, meta, per_row, act)
            _check(out, ref, bound)


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (4, 3), (6, 0), (0, 6), (1, 1), (7, 0), (0, 7), (2, 5)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("per_row", [False, True])
@pytest.mark.parametrize("shape", [(96, 2052), (96, 2064)], ids=["regs", "bulk"])
def test_gemv_one_hot_exact(exmy, orc, fmt, per_row, shape):
    """act = one-hot rows e_c: out[m, n] = 1 * W[n, c] + 0 + ... exactly, so
    every column the rows select equals the oracle's decode bit for bit (the
    table, the byte extraction, the per-row rescale; every code of the format
    occurs at this size).  2052 columns: the register-pipelined kernel; 2064:
    the bulk-staged one with a 16-column last stage"""
    bits = _weights(shape, 17, False)
    d = W.from_bits(bits).to(DEV)
    if per_row:
        meta = orc.block_max_exponent(bits, (1, shape[1]))
        p = exmy.encode_blocked(d, fmt, torch.from_numpy(meta.copy()).to(DEV), (1, shape[1]))
        dec = orc.decode_blocked(p.data.cpu().numpy(), shape, fmt, meta, (1, shape[1]), orc.ROWS, out_dtype=np.uint32)
    else:
        e = orc.emax(orc.histogram(bits))
        p = exmy.encode(d, fmt, e)
        dec = orc.decode(p.data.cpu().numpy(), shape, fmt, e, orc.ROWS, out_dtype=np.uint32)
    for cols in ([0, 1, 2, 3, 4, 5, 6, 7], [1023, 1024, 1025, 2047, 2048, 2049, 2050, shape[1] - 1], [9, 500, 1500],
                 [77]):
        act = np.zeros((len(cols), shape[1]), np.float32)
        act[np.arange(len(cols)), cols] = 1.0
        out = exmy.gemv(p, torch.from_numpy(act).to(DEV)).cpu().numpy()
        want = dec[:, cols].T.copy().view(np.float32)
        # +0 and -0 weights sum to +0 (0 + -0): compare values, and bits where nonzero
        np.testing.assert_array_equal(out, want)
        nz = want != 0
        np.testing.assert_array_equal(out[nz].view(np.uint32), want[nz].view(np.uint32))


def test_gemv_config2_sampled(exmy, orc):
    """config 2's weight (16384 x 16384 bf16, e3m3, per tensor), 4 activation
    rows: 64 sampled output rows against the oracle's decode of those rows"""
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=DEV)
    h = exmy.histogram(t)
    meta = exmy.emax(h)
    p = exmy.encode(t, "e3m3", meta, strict=False)
    act = torch.randn(4, C, generator=torch.Generator().manual_seed(9)).to(DEV)
    out = exmy.gemv(p, act).cpu().numpy()
    rows = np.random.default_rng(3).choice(R, 64, replace=False)
    e = int(meta.item())
    dec = exmy.decode(p, torch.float32)[torch.from_numpy(rows).to(DEV)].cpu().numpy().astype(np.float64)
    # the sampled rows' decode is itself checked bit-exactly against the oracle
    bits = W.to_bits(t[torch.from_numpy(rows).to(DEV)].cpu())
    want = orc.quantize(bits, "e3m3", e).astype(np.uint32) << 16      # bf16 bits widened to fp32
    np.testing.assert_array_equal(dec.astype(np.float32).view(np.uint32), want)
    a = act.cpu().numpy().astype(np.float64)
    ref = a @ dec.T
    bound = C * U32 / (1 - C * U32) * (np.abs(a) @ np.abs(dec).T) + C * 2.0 ** -149
    assert np.all(np.abs(out[:, rows] - ref) <= bound)


def test_gemv_kernels_agree(exmy):
    """the bulk-staged and the register-pipelined kernels sum in the same
    order: identical outputs (config-2-like rows, 2 row groups per CTA)"""
    t = W.bf16_weights((2048, 8192), seed=4, device=DEV)
    p = exmy.encode(t, "e2m3", exmy.emax(exmy.histogram(t)))
    act = torch.randn(3, 8192, generator=torch.Generator().manual_seed(2)).to(DEV)
    a = exmy.gemv(p, act)
    prev = exmy.gemv_bulk(False)
    try:
        b = exmy.gemv(p, act)
    finally:
        exmy.gemv_bulk(prev)
    assert torch.equal(a, b)


def test_gemv_guards(exmy):
    t = W.bf16_weights((16, 64), seed=2, device=DEV)
    p = exmy.encode(t, "e3m3", exmy.emax(exmy.histogram(t)))
    with pytest.raises(ValueError):
        exmy.gemv(p, torch.zeros(2, 63, device=DEV))
    q = exmy.encode(t, "e4m4", exmy.emax(exmy.histogram(t)))       # k = 9: not supported by the table kernel
    with pytest.raises(exmy.ExmyError):
        exmy.gemv(q, torch.zeros(1, 64, device=DEV))
    c = exmy.encode(t, "e3m3", exmy.emax(exmy.histogram(t)), axis="cols")
    with pytest.raises(ValueError):
        exmy.gemv(c, torch.zeros(1, 64, device=DEV))
