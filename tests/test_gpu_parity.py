"""GPU parity: every sm_100a kernel vs the CPU oracle on the same seeded
inputs.  Tolerance is 0: histograms, codes and packed bytes byte-identical,
quantized/decoded outputs bit-identical (incl. -0 and NaN payloads)."""
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


def dev_bits(bits: np.ndarray) -> torch.Tensor:
    return W.from_bits(bits).to(DEV)


def np_bits(t: torch.Tensor) -> np.ndarray:
    return W.to_bits(t)


ALL_FMTS = [(x, k - 1 - x) for k in range(3, 10) for x in range(0, min(8, k - 1) + 1)]


def fmt_id(f):
    return f"e{f[0]}m{f[1]}"


def emax_set(x):
    return sorted({0, min((1 << x) - 1, 254), 100, 127, 200, 254})


def oracle_boundary_f32(orc, fmt, e_max):
    """Boundary suite B(x,y,e_max) built from the oracle's grid."""
    g = np.abs(orc.grid(fmt, e_max))
    g = np.unique(g)
    mids = (g[1:] + g[:-1]) / 2
    cand = np.concatenate([g, mids, [g[-1] * 2, g[-1] * 1.75, g[1] / 2, g[1] / 4, 2.0 ** -149, 1e38]])
    with np.errstate(over="ignore"):
        f = cand.astype(np.float32)
    f = f[np.isfinite(f)]
    f = np.concatenate([f, np.nextafter(f, np.float32(0)), np.nextafter(f, np.float32(np.inf))])
    f = f[np.isfinite(f)]
    b = f.view(np.uint32)
    b = np.concatenate([b, b | np.uint32(0x80000000), np.array(W.SPECIAL_F32_BITS, np.uint32)])
    pad = (-b.size) % 64
    return np.concatenate([b, np.zeros(pad, np.uint32)])


# ----------------------------------------------------------------- K1 / K1b
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("n", [0, 1, 7, 8 * 1000 + 5, 1 << 20, (1 << 22) + 3])
def test_histogram_parity(exmy, orc, dt, n, mode):
    prev = exmy.hist_mode(mode)
    try:
        bits = W.random_bits_bf16(n, n) if dt == "bf16" else W.random_bits_f32(n, n)
        h = exmy.histogram(dev_bits(bits)).cpu().numpy().astype(np.uint64)
        np.testing.assert_array_equal(h, orc.histogram(bits))
    finally:
        exmy.hist_mode(prev)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_histogram_peaked_and_misaligned(exmy, orc, dt):
    t = W.bf16_weights((4096, 1024), seed=3) if dt == "bf16" else W.f32_gradients(1 << 22)
    bits = W.to_bits(t).reshape(-1)
    d = dev_bits(bits)
    np.testing.assert_array_equal(exmy.histogram(d).cpu().numpy().astype(np.uint64), orc.histogram(bits))
    # misaligned view (offset by one element) takes the scalar kernel
    sub = d[1:]
    np.testing.assert_array_equal(exmy.histogram(sub).cpu().numpy().astype(np.uint64), orc.histogram(bits[1:]))
    # accumulation into an existing histogram
    h = exmy.histogram(d)
    exmy.histogram(d, out=h)
    np.testing.assert_array_equal(h.cpu().numpy().astype(np.uint64), 2 * orc.histogram(bits))


def peaked_mix(n, seed, dt="bf16"):
    """bf16 weights-like values (peaked exponents) with far
    clusters, exact zeros, subnormals and NaN/Inf sprinkled in"""
    rng = np.random.default_rng(seed)
    v = (rng.standard_normal(n) * 0.02).astype(np.float32)
    blk = rng.integers(0, 4, size=(n + 4095) // 4096).repeat(4096)[:n]
    v = np.where(blk == 1, v * np.float32(2.0 ** 60), v)       # whole 4K runs in another window
    v = np.where(blk == 2, v * np.float32(2.0 ** -100), v)     # runs near the subnormal range
    m = rng.random(n)
    v = np.where(m < 0.01, np.float32(0), v)
    v = np.where((m > 0.01) & (m < 0.012), v * np.float32(2.0 ** 30), v)   # single far elements
    bits = (v.view(np.uint32) >> 16).astype(np.uint16) if dt == "bf16" else v.view(np.uint32).copy()
    k = rng.choice(n, size=min(n, 50), replace=False)
    bits[k[:25]] = 0x7FC0 if dt == "bf16" else 0x7FC00000
    bits[k[25:]] = 0xFF80 if dt == "bf16" else 0xFF800000
    return bits


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("blocks", [0, 1, 3])
@pytest.mark.parametrize("n", [8 * 1000 + 5, (1 << 22) + 3, 20_000_011])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_histogram_peaked_epochs(exmy, orc, mode, blocks, n, dt):
    """peaked bf16 data (most elements in a few bins: the lane-private 16-bit
    counters fill fastest), far clusters, zeros, specials; a grid capped at
    1 / 3 CTAs makes every lane run past the counter epoch, so the flush
    before overflow is exercised at test sizes"""
    prev = exmy.hist_mode(mode)
    exmy.hist_blocks(blocks)
    try:
        bits = peaked_mix(n, n % 97, dt)
        h = exmy.histogram(dev_bits(bits)).cpu().numpy().astype(np.uint64)
        np.testing.assert_array_equal(h, orc.histogram(bits))
    finally:
        exmy.hist_mode(prev)
        exmy.hist_blocks(0)


def test_histogram_wide_and_shifting_exponents(exmy, orc):
    """17+ distinct exponents per warp in the first half, any bin (zeros,
    subnormals, bin 255) in the second, both orders: the lane-pair counters
    (MODE 3: bins of equal parity from a lane pair share a bank) count
    exactly"""
    prev = exmy.hist_mode(3)
    try:
        rng = np.random.default_rng(5)
        n = 1 << 22
        e = rng.integers(100, 117, n).astype(np.uint16)        # 17 distinct exponents: one always outside
        e[n // 2:] = rng.integers(0, 256, n // 2).astype(np.uint16)   # second half: anything
        bits = (e << 7) | rng.integers(0, 1 << 7, n).astype(np.uint16) | (rng.integers(0, 2, n).astype(np.uint16) << 15)
        for b in (bits, bits[::-1].copy()):
            h = exmy.histogram(dev_bits(b)).cpu().numpy().astype(np.uint64)
            np.testing.assert_array_equal(h, orc.histogram(b))
    finally:
        exmy.hist_mode(prev)


def test_emax_parity(exmy, orc):
    rng = np.random.default_rng(1)
    for trial in range(50):
        h = np.zeros(256, np.int64)
        k = rng.integers(0, 6)
        h[rng.integers(0, 256, size=k)] = rng.integers(1, 100, size=k)
        m = exmy.emax(torch.from_numpy(h).to(DEV))
        assert int(m.item()) == orc.emax(h.astype(np.uint64))


# --------------------------------------------------------------- K2 quantize
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("fmt", ALL_FMTS, ids=fmt_id)
def test_quantize_exhaustive_bf16(exmy, orc, fmt, generic):
    """Every bf16 pattern (65,536) x e_max sweep, every format k=3..9."""
    bits = W.all_bf16_bits()
    d = dev_bits(bits)
    exmy.force_generic(generic)
    try:
        for e in emax_set(fmt[0]):
            q = np_bits(exmy.quantize(d, fmt, e))
            ref = orc.quantize(bits, fmt, e)
            np.testing.assert_array_equal(q, ref, err_msg=f"{fmt_id(fmt)} e_max={e}")
    finally:
        exmy.force_generic(False)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("fmt", ALL_FMTS, ids=fmt_id)
def test_quantize_f32_boundaries(exmy, orc, fmt, generic):
    exmy.force_generic(generic)
    try:
        for e in emax_set(fmt[0]):
            b = np.concatenate([oracle_boundary_f32(orc, fmt, e), W.random_bits_f32(4096, e)])
            q = np_bits(exmy.quantize(dev_bits(b), fmt, e))
            np.testing.assert_array_equal(q, orc.quantize(b, fmt, e), err_msg=f"{fmt_id(fmt)} e_max={e}")
    finally:
        exmy.force_generic(False)


def test_quantize_misaligned_and_ragged(exmy, orc):
    bits = W.random_bits_bf16(1000 + 3, 5)
    d = dev_bits(bits)
    for fmt in [(3, 3), (0, 6), (8, 0)]:
        np.testing.assert_array_equal(np_bits(exmy.quantize(d[1:], fmt, 125)), orc.quantize(bits[1:], fmt, 125))
        np.testing.assert_array_equal(np_bits(exmy.quantize(d, fmt, 125)), orc.quantize(bits, fmt, 125))


# ------------------------------------------------------ K3 / K4 encode-decode
SHAPES = [(8, 8), (64, 512), (24, 40), (16, 264), (40, 96), (8, 4104)]


def _check_roundtrip(exmy, orc, bits2d, fmt, e, axis, out_dtypes=("same",)):
    ax = orc.ROWS if axis == "rows" else orc.COLS
    d = dev_bits(bits2d)
    p = exmy.encode(d, fmt, e, axis=axis, specials_capacity=bits2d.size)
    ref_packed, ref_idx, ref_bits, ref_n = orc.encode(bits2d, fmt, e, ax)
    np.testing.assert_array_equal(p.data.cpu().numpy(), ref_packed, err_msg=f"packed {fmt_id(fmt)} {axis} e={e}")
    spi, spb, cnt = p.specials()
    assert cnt == ref_n
    np.testing.assert_array_equal(spi.cpu().numpy(), ref_idx)
    np.testing.assert_array_equal(spb.cpu().numpy().view(np.uint32), ref_bits)
    for od in out_dtypes:
        if od == "same":
            out = exmy.decode(p)
            ref = orc.decode(ref_packed, bits2d.shape, fmt, e, ax, ref_idx, ref_bits, bits2d.dtype)
        else:
            tdt = torch.float32 if od == "f32" else torch.bfloat16
            out = exmy.decode(p, tdt)
            ref = orc.decode(ref_packed, bits2d.shape, fmt, e, ax, ref_idx, ref_bits,
                             np.uint32 if od == "f32" else np.uint16)
        np.testing.assert_array_equal(np_bits(out), ref, err_msg=f"decode {fmt_id(fmt)} {axis} e={e} {od}")


@pytest.mark.parametrize("fmt", ALL_FMTS, ids=fmt_id)
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_encode_decode_all_formats(exmy, orc, fmt, dt):
    rng = np.random.default_rng(fmt[0] * 16 + fmt[1])
    for shape in SHAPES:
        n = shape[0] * shape[1]
        if dt == "bf16":
            t = W.bf16_weights(shape, seed=n, std=float(rng.choice([0.02, 1.0, 100.0])))
            bits = W.to_bits(t)
            bits.reshape(-1)[: n // 50] = W.random_bits_bf16(n // 50, n)
        else:
            bits = W.to_bits(W.f32_wide(shape, seed=n))
            bits.reshape(-1)[: n // 50] = W.random_bits_f32(n // 50, n)
        e = orc.emax(orc.histogram(bits))
        for axis in ("rows", "cols"):
            if axis == "rows" and shape[0] % 8:
                continue
            _check_roundtrip(exmy, orc, bits, fmt, e, axis, ("same", "f32", "bf16"))
        for e2 in (0, 254, min((1 << fmt[0]) - 1, 254)):
            _check_roundtrip(exmy, orc, bits, fmt, e2, "cols", ("same",))


@pytest.mark.parametrize("generic", [False, True])
def test_encode_decode_exhaustive_bf16_7bit(exmy, orc, generic):
    """all 65,536 bf16 patterns through every 7-bit format (config 2 formats)."""
    bits = W.all_bf16_bits().reshape(256, 256)
    exmy.force_generic(generic)
    try:
        for x in range(0, 7):
            fmt = (x, 6 - x)
            for e in emax_set(x):
                for axis in ("rows", "cols"):
                    _check_roundtrip(exmy, orc, bits, fmt, e, axis)
    finally:
        exmy.force_generic(False)


def test_config1_all_codes(exmy, orc):
    """Config 1: every code of e3m2 and e2m3 decodes like the oracle and
    re-encodes to itself, at e_max in {0,64,127,129,131,200,254}."""
    for fmt in [(3, 2), (2, 3)]:
        for e in (0, 64, 127, 129, 131, 200, 254):
            codes = np.tile(np.arange(64, dtype=np.uint16), 2).reshape(16, 8)
            packed = orc.pack(codes, (16, 8), orc.COLS, 6)
            dp = torch.from_numpy(packed).to(DEV)
            out = exmy.decode_raw(dp, 16, 8, fmt, e, axis="cols", dtype=torch.float32)
            ref = orc.decode(packed, (16, 8), fmt, e, orc.COLS, out_dtype=np.uint32)
            np.testing.assert_array_equal(np_bits(out), ref)
            p2 = exmy.encode(out, fmt, e, axis="cols")
            np.testing.assert_array_equal(p2.data.cpu().numpy(), packed)


def test_config1_wide_f32_roundtrip(exmy, orc):
    """Config 1: 65,536 fp32 (256x256) bulk + boundary block, e3m2 with e_max
    from the histogram and forced 131, both axes."""
    bulk = W.to_bits(W.f32_wide((256, 256), seed=0)).reshape(-1)
    bnd = oracle_boundary_f32(orc, (3, 2), 131)
    bulk[: bnd.size] = bnd
    bits = bulk.reshape(256, 256)
    e_hist = orc.emax(orc.histogram(bits))
    d = dev_bits(bits)
    assert int(exmy.max_exponent(d).item()) == e_hist
    for e in (e_hist, 131):
        for axis in ("rows", "cols"):
            _check_roundtrip(exmy, orc, bits, (3, 2), e, axis, ("same", "bf16"))


def test_empty_and_degenerate(exmy, orc):
    z = torch.empty((0, 16), dtype=torch.bfloat16, device=DEV)
    p = exmy.encode(z, "e3m3", 127)
    assert p.data.numel() == 0
    assert exmy.decode(p).shape == (0, 16)
    assert exmy.quantize(z, "e3m3", 127).numel() == 0
    # all zeros / all specials tensors
    for v in (0.0, -0.0, float("nan"), float("-inf")):
        t = torch.full((8, 16), v, dtype=torch.float32)
        bits = W.to_bits(t)
        _check_roundtrip(exmy, orc, bits, (4, 3), 127, "rows")
    # ragged ROWS (C % V != 0) and misaligned input -> generic kernels
    bits = W.random_bits_bf16(16 * 36, 3).reshape(16, 36)
    _check_roundtrip(exmy, orc, bits, (3, 3), 125, "rows")
    big = dev_bits(W.random_bits_bf16(16 * 64 + 1, 4))
    sub = big[1:].view(16, 64)
    p = exmy.encode(sub, "e2m4", 124, axis="rows")
    ref = orc.encode(W.to_bits(sub), "e2m4", 124, orc.ROWS)[0]
    np.testing.assert_array_equal(p.data.cpu().numpy(), ref)


def test_specials_sorted_and_capacity(exmy, orc):
    rng = np.random.default_rng(9)
    bits = W.to_bits(W.f32_wide((64, 256), seed=2))
    flat = bits.reshape(-1)
    pos = rng.choice(flat.size, size=3000, replace=False)
    flat[pos] = np.array(W.SPECIAL_F32_BITS[:5], np.uint32)[rng.integers(0, 5, size=pos.size)]
    _check_roundtrip(exmy, orc, bits, (4, 4), 130, "rows", ("same", "bf16"))
    # more specials than capacity: count still total, first entries dropped
    d = dev_bits(bits)
    p = exmy.encode(d, "e4m4", 130, specials_capacity=10, strict=False)
    spi, spb, cnt = p.specials()
    assert cnt == 3000 and spi.numel() == 10
    # the list is index-ordered compaction: exactly the FIRST 10 specials by index
    assert spi.cpu().numpy().tolist() == sorted(pos.tolist())[:10]
    assert spb.cpu().numpy().view(np.uint32).tolist() == flat[sorted(pos.tolist())[:10]].tolist()
    # > 4096 specials: global-memory sort path
    flat[:] = 0x7FC00000
    flat[::3] = 0x3F800000
    _check_roundtrip(exmy, orc, bits, (3, 3), 127, "cols")


def test_row_shard_decodes_independently(exmy, orc):
    """byte ranges of a row shard decode on their own."""
    t = W.bf16_weights((256, 1024), seed=4)
    d = t.to(DEV)
    p = exmy.encode(d, "e3m3", axis="rows")
    e = int(p.meta.item())
    q = exmy.quantize(d, "e3m3", e)
    C, k = 1024, 7
    ws, offs = exmy.segments(k, 256 * C)
    r0, r1 = 64, 192
    shard = torch.cat([p.data[o + r0 * C * w // 8: o + r1 * C * w // 8] for w, o in zip(ws, offs)])
    out = exmy.decode_raw(shard, r1 - r0, C, "e3m3", e, axis="rows", dtype=torch.bfloat16)
    assert torch.equal(out.view(torch.int16), q[r0:r1].view(torch.int16))


def test_config2_full_size_sampled(exmy, orc):
    """Config 2 at full size (16384 x 16384 bf16, all 7-bit formats), in the
    launch configuration bench.py times; parity on sampled row-group windows
    (their packed bytes are contiguous ranges) + decode==quantize
    on the whole tensor (a property that holds at any size)."""
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=DEV)
    hist = exmy.histogram(t)
    meta = exmy.emax(hist)
    e = int(meta.item())
    windows = [0, 8 * 517, 8 * 1024, R - 8]
    for x in range(0, 7):
        fmt = (x, 6 - x)
        p = exmy.encode(t, fmt, meta, axis="rows")
        dec = exmy.decode(p)
        q = exmy.quantize(t, fmt, meta)
        assert torch.equal(dec.view(torch.int16), q.view(torch.int16)), fmt
        ws, offs = exmy.segments(7, R * C)
        for r0 in windows:
            rows = W.to_bits(t[r0:r0 + 8])
            ref = orc.encode(rows, fmt, e, orc.ROWS)[0]
            got = torch.cat([p.data[o + r0 * C * w // 8: o + (r0 + 8) * C * w // 8] for w, o in zip(ws, offs)])
            np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"{fmt} window {r0}")
            np.testing.assert_array_equal(W.to_bits(q[r0:r0 + 8]), orc.quantize(rows, fmt, e))
        del p, dec, q


def test_host_codec_roundtrip(exmy, orc):
    t = W.bf16_weights((128, 512), seed=6)
    hc = exmy.HostCodec(t.shape, torch.bfloat16, "e2m4")
    hin = t.pin_memory()
    hp = torch.empty(hc.nbytes_packed, dtype=torch.uint8).pin_memory()
    hm = torch.empty(1, dtype=torch.uint8).pin_memory()
    hc.encode(hin, hp, hm)
    hout = torch.empty_like(hin).pin_memory()
    hc.decode(hp, hout)
    torch.cuda.synchronize()
    bits = W.to_bits(t)
    e = orc.emax(orc.histogram(bits))
    assert int(hm.item()) == e
    np.testing.assert_array_equal(hp.numpy(), orc.encode(bits, "e2m4", e, orc.ROWS)[0])
    np.testing.assert_array_equal(W.to_bits(hout), orc.quantize(bits, "e2m4", e))


@pytest.mark.parametrize("axis", ["rows", "cols"])
def test_beyond_2e32_elements(exmy, orc, axis):
    """Maximum-size edge case: n > 2^32 elements (64-bit indexing everywhere).
    Parity on windows past the 2^32 boundary (rows are contiguous byte ranges
    per segment) + decode == quantize on sampled rows."""
    if torch.cuda.get_device_properties(0).total_memory < 60e9:
        pytest.skip("needs a large-memory GPU")
    R, C = 65536 + 64, 65536
    t = W.bf16_weights((R, C), seed=21, device=DEV)
    meta = exmy.max_exponent(t)
    e = int(meta.item())
    p = exmy.encode(t, "e3m3", meta, axis=axis)
    ws, offs = exmy.segments(7, R * C)
    for r0 in (0, 65536 - 8, 65536 + 8, R - 8):
        rows = W.to_bits(t[r0:r0 + 8])
        ref = orc.encode(rows, "e3m3", e, orc.ROWS if axis == "rows" else orc.COLS)[0]
        got = torch.cat([p.data[o + r0 * C * w // 8: o + (r0 + 8) * C * w // 8] for w, o in zip(ws, offs)])
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"window {r0}")
    d = exmy.decode(p)
    del p
    torch.cuda.empty_cache()
    q = exmy.quantize(t, "e3m3", meta)
    for r0 in (0, 65536 - 8, 65536 + 8, R - 8):
        assert torch.equal(d[r0:r0 + 8].view(torch.int16), q[r0:r0 + 8].view(torch.int16))
        np.testing.assert_array_equal(W.to_bits(q[r0:r0 + 8]), orc.quantize(W.to_bits(t[r0:r0 + 8]), "e3m3", e))
    h = exmy.histogram(t).cpu().numpy().astype(np.uint64)
    assert int(h.sum()) == R * C


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("n", [1, 7, 8 * 1000 + 5, 1 << 20, (1 << 22) + 3])
def test_max_exponent_reduction(exmy, orc, dt, n):
    """exmy_max_exponent == top populated histogram bin in [0,254]"""
    bits = W.random_bits_bf16(n, n + 1) if dt == "bf16" else W.random_bits_f32(n, n + 1)
    d = dev_bits(bits)
    assert int(exmy.max_exponent(d).item()) == orc.emax(orc.histogram(bits))
    # peaked data, NaN/Inf-only and zero-only tensors
    t = W.bf16_weights((n,), seed=n) if dt == "bf16" else W.f32_gradients(n, seed=n)
    b2 = W.to_bits(t)
    assert int(exmy.max_exponent(t.to(DEV)).item()) == orc.emax(orc.histogram(b2))
    sp = np.full(n, 0x7FC0 if dt == "bf16" else 0x7F800000, bits.dtype)
    assert int(exmy.max_exponent(dev_bits(sp)).item()) == 0
    z = np.zeros(n, bits.dtype)
    z[-1] = 0x0001    # one subnormal at the tail
    assert int(exmy.max_exponent(dev_bits(z)).item()) == 0


def test_max_exponent_preserves_neighbour_bytes(exmy):
    """the byte compare-and-swap touches only the addressed metadata byte"""
    t = W.bf16_weights((4096,), seed=2).to(DEV)
    metas = torch.tensor([11, 22, 33, 44, 55, 66, 77, 88], dtype=torch.uint8, device=DEV)
    for i in range(8):
        exmy.max_exponent(t, out=metas[i:i + 1])
    ref = int(exmy.emax(exmy.histogram(t)).item())
    assert metas.tolist() == [ref] * 8
    m2 = torch.tensor([1, 2, 3, 4], dtype=torch.uint8, device=DEV)
    exmy.max_exponent(t, out=m2[2:3])
    assert m2.tolist() == [1, 2, ref, 4]


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_all_nan_tensor_is_fast_and_ordered(exmy, dt):
    """a NaN-heavy tensor (a diverged gradient) encodes in
    under 2x the clean tensor's time -- the fast kernels mask NaN/Inf lanes
    to code 0 and count them per warp, the ordered list is a stream
    compaction (no sort) that stops re-reading at the capacity -- and the
    list holds the first `capacity` specials by index."""
    n_rows, cols = (16384, 16384) if dt == "bf16" else (8192, 16384)
    clean = W.bf16_weights((n_rows, cols), seed=1, device=DEV) if dt == "bf16" else \
        W.f32_gradients(n_rows * cols, device=DEV).view(n_rows, cols)
    nan = torch.full_like(clean, float("nan"))
    nan.view(-1)[1::7] = float("-inf")
    meta = exmy.max_exponent(clean)
    cap = 4096

    def t_enc(x):
        for _ in range(2):
            exmy.encode(x, "e3m3", meta, specials_capacity=cap, strict=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p = exmy.encode(x, "e3m3", meta, specials_capacity=cap, strict=False)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts)[2], p

    t_clean, pc = t_enc(clean)
    t_nan, pn = t_enc(nan)
    idx, bits, cnt = pn.specials()
    assert cnt == clean.numel()
    assert idx.cpu().numpy().tolist() == list(range(cap))
    want = [0xFF800000 if i % 7 == 1 else int(W.to_bits(nan.view(-1)[i:i + 1].cpu())[0]) << (16 if dt == "bf16" else 0)
            for i in range(cap)]
    assert bits.cpu().numpy().view(np.uint32).tolist() == [w & 0xFFFFFFFF for w in want]
    assert int(pc.sp_count[0].item()) == 0
    assert t_nan < 2.0 * t_clean, (t_nan, t_clean)
    # the packed stream holds code 0 for every special; decode restores the listed ones
    assert int(pn.data.max().item()) == 0
