"""GPU parity of the block-metadata path against the
oracle: block max exponent (both schemes), blocked quantize / encode /
decode, every block shape class (tensor, row, column, sub-row, 2-D tile),
fast and scalar kernels, bit-exact."""
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


def rowscaled_bits(shape, seed, dt="bf16"):
    """rows of very different magnitude (per-row metadata matters) + specials"""
    R, C = shape
    rng = np.random.default_rng(seed)
    t = W.bf16_weights(shape, seed=seed, std=0.02).float().numpy()
    t = t * (2.0 ** rng.integers(-20, 20, size=(R, 1))).astype(np.float32)
    t = torch.from_numpy(t.astype(np.float32))
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t)
    flat = bits.reshape(-1)
    flat[rng.integers(0, flat.size, size=max(1, flat.size // 500))] = (0x7FC0 if dt == "bf16" else 0x7FC00000)
    return bits


BLOCKS = [("tensor", None), ("row", None), ("col", None), ("subrow32", (1, 32)), ("tile8x16", (8, 16)),
          ("tile16x64", (16, 64)), ("odd", (2, 12))]


def block_of(name, spec, shape):
    R, C = shape
    return {"tensor": (R, C), "row": (1, C), "col": (R, 1)}.get(name, spec)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("scheme", [0, 1])
def test_block_max_exponent(exmy, orc, dt, scheme):
    shape = (64, 192)
    bits = rowscaled_bits(shape, 3, dt)
    d = W.from_bits(bits).to(DEV)
    for name, spec in BLOCKS:
        blk = block_of(name, spec, shape)
        for y in (0, 1, 3, 6):
            got = exmy.block_max_exponent(d, blk, y, scheme).cpu().numpy()
            ref = orc.block_max_exponent(bits, blk, y, scheme)
            np.testing.assert_array_equal(got, ref, err_msg=f"{name} y={y}")
    # fp32 subnormals / carries at the exponent-254 edge for the after scheme
    edge = np.array([0x007FFFFF, 0x007FFFFE, 0x00400000, 0x7F7FFFFF, 0x00000001, 0x7F800000, 0, 0x80000000],
                    np.uint32).reshape(1, 8)
    for y in (0, 1, 2, 5, 22):
        got = exmy.block_max_exponent(W.from_bits(edge).to(DEV), (1, 1), y, scheme).cpu().numpy()
        np.testing.assert_array_equal(got, orc.block_max_exponent(edge, (1, 1), y, scheme))


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("scheme", [0, 1])
def test_block_max_exponent_tiles(exmy, orc, dt, scheme):
    """2-D blocks with short rows (k_block_max_tile: a warp reads 32 vectors
    of each block row, covering 32 / (bc / V) blocks side by side): block
    heights not a multiple of the 8 rows in flight, 1..16 vectors per block
    row, NaN/Inf, zeros and subnormal rows"""
    shape = (96, 1024)
    bits = rowscaled_bits(shape, 7, dt)
    rng = np.random.default_rng(11)
    flat = bits.reshape(-1)
    k = rng.choice(flat.size, 40, replace=False)
    flat[k[:20]] = 0x7FC0 if dt == "bf16" else 0x7FC00000
    flat[k[20:30]] = 0xFF80 if dt == "bf16" else 0xFF800000
    bits[5] = 0                                             # an all-zero row
    bits[6, :64] = 1                                        # smallest subnormals
    d = W.from_bits(bits).to(DEV)
    V = 8 if dt == "bf16" else 4
    for blk in [(32, 32), (8, 16), (3, 8 * V), (12, V), (96, 2 * V), (1 * 2, 4 * V), (24, 16 * V)]:
        if shape[0] % blk[0] or shape[1] % blk[1]:
            continue
        for y in (0, 2, 5):
            got = exmy.block_max_exponent(d, blk, y, scheme).cpu().numpy()
            ref = orc.block_max_exponent(bits, blk, y, scheme)
            np.testing.assert_array_equal(got, ref, err_msg=f"{blk} y={y}")


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("scheme", [0, 1])
def test_block_max_exponent_bands(exmy, orc, dt, scheme):
    """Shapes large enough for the band kernel (k_block_max_band: a CTA
    streams br rows x 256*U vectors; U = 8 / 4 / 2 picked by the work count)
    incl. a column chunk that ends mid-way (4352 columns), and tall blocks
    that take the warp-per-block kernel's flattened path"""
    V = 8 if dt == "bf16" else 4
    for shape in ((4096, 4352), (2048, 8192)):
        bits = rowscaled_bits(shape, 13, dt)
        bits[7, :] = 0
        d = W.from_bits(bits).to(DEV)
        for blk in [(2, 4 * V), (4, 16 * V), (2, V), (8, 2 * V), (128, 32 * V), (64, 16 * V)]:
            if shape[0] % blk[0] or shape[1] % blk[1]:
                continue
            got = exmy.block_max_exponent(d, blk, 3, scheme).cpu().numpy()
            ref = orc.block_max_exponent(bits, blk, 3, scheme)
            np.testing.assert_array_equal(got, ref, err_msg=f"{shape} {blk}")


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (4, 2), (6, 0), (1, 5), (0, 6), (2, 2), (5, 3), (2, 1), (0, 7),
                                 (1, 7), (8, 0)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_blocked_codecs(exmy, orc, fmt, dt):
    shape = (64, 192)
    bits = rowscaled_bits(shape, fmt[0] * 10 + fmt[1], dt)
    d = W.from_bits(bits).to(DEV)
    x, y = fmt
    for name, spec in BLOCKS:
        blk = block_of(name, spec, shape)
        for scheme in (0, 1):
            meta = orc.block_max_exponent(bits, blk, y, scheme)
            dm = torch.from_numpy(meta.copy()).to(DEV)
            q = W.to_bits(exmy.quantize_blocked(d, fmt, dm, blk))
            qref = orc.quantize_blocked(bits, fmt, meta, blk)
            np.testing.assert_array_equal(q, qref, err_msg=f"quantize {name} scheme {scheme}")
            for axis in ("rows", "cols"):
                ax = orc.ROWS if axis == "rows" else orc.COLS
                p = exmy.encode_blocked(d, fmt, dm, blk, axis=axis, specials_capacity=bits.size)
                pref, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, blk, ax)
                np.testing.assert_array_equal(p.data.cpu().numpy(), pref, err_msg=f"encode {name} {axis}")
                spi, spb, cnt = p.specials()
                assert cnt == ns
                np.testing.assert_array_equal(spi.cpu().numpy(), idx)
                out = exmy.decode(p)
                np.testing.assert_array_equal(W.to_bits(out), qref, err_msg=f"decode {name} {axis}")
                od = np.uint32 if dt == "bf16" else np.uint16
                other = exmy.decode(p, torch.float32 if dt == "bf16" else torch.bfloat16)
                np.testing.assert_array_equal(W.to_bits(other),
                                              orc.decode_blocked(pref, shape, fmt, meta, blk, ax, idx, sb, od))


def test_blocked_forced_metadata_edges(exmy, orc):
    """metadata outside the fast preconditions (e_max 0, 254, below the data)
    per row: the tiles fall back to the integer path, results unchanged."""
    shape = (16, 64)
    bits = rowscaled_bits(shape, 77)
    d = W.from_bits(bits).to(DEV)
    meta = np.array([0, 254, 1, 100, 127, 131, 200, 3] * 2, np.uint8).reshape(16, 1)
    dm = torch.from_numpy(meta.copy()).to(DEV)
    for fmt in [(3, 3), (7, 1), (6, 0), (0, 6)]:
        q = W.to_bits(exmy.quantize_blocked(d, fmt, dm, (1, 64)))
        np.testing.assert_array_equal(q, orc.quantize_blocked(bits, fmt, meta, (1, 64)))
        for axis in ("rows", "cols"):
            ax = orc.ROWS if axis == "rows" else orc.COLS
            p = exmy.encode_blocked(d, fmt, dm, (1, 64), axis=axis, specials_capacity=bits.size)
            pref = orc.encode_blocked(bits, fmt, meta, (1, 64), ax)[0]
            np.testing.assert_array_equal(p.data.cpu().numpy(), pref)
            np.testing.assert_array_equal(W.to_bits(exmy.decode(p)), orc.quantize_blocked(bits, fmt, meta, (1, 64)))


def test_per_row_config2_shape_sampled(exmy, orc):
    """per-row metadata on the config-2 tensor (16384^2 bf16), the shape the
    bench measures; parity on sampled row-group windows + decode == quantize."""
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=DEV)
    meta = exmy.block_max_exponent(t, "row")
    ws, offs = exmy.segments(7, R * C)
    p = exmy.encode_blocked(t, "e3m3", meta, "row")
    q = exmy.quantize_blocked(t, "e3m3", meta, "row")
    assert torch.equal(exmy.decode(p).view(torch.int16), q.view(torch.int16))
    for r0 in (0, 8 * 777, R - 8):
        rows = W.to_bits(t[r0:r0 + 8])
        m = meta[r0:r0 + 8].cpu().numpy()
        np.testing.assert_array_equal(m, orc.block_max_exponent(rows, (1, C)))
        ref = orc.encode_blocked(rows, "e3m3", m, (1, C), orc.ROWS)[0]
        got = torch.cat([p.data[o + r0 * C * w // 8: o + (r0 + 8) * C * w // 8] for w, o in zip(ws, offs)])
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", [(4, 2), (3, 1), (5, 3), (2, 4), (8, 0), (0, 8)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("per_row", [False, True])
def test_row_gather_decode(exmy, orc, fmt, dt, per_row):
    """Embedding lookup (config 5 access pattern): decode an arbitrary list of
    rows of a COLS-packed table == the same rows of the full decode."""
    R, C = 1000, 136
    t = W.f32_embedding(R, C, seed=5)
    t = t * torch.exp2(torch.randint(-8, 8, (R, 1)).float())
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t)
    d = t.to(DEV)
    rng = np.random.default_rng(1)
    idx = rng.integers(0, R, size=777)
    idx[:5] = [0, R - 1, 3, 3, 3]
    if per_row:
        meta = orc.block_max_exponent(bits, (1, C))
        p = exmy.encode_blocked(d, fmt, torch.from_numpy(meta.copy()).to(DEV), (1, C), axis="cols")
        full = orc.decode_blocked(orc.encode_blocked(bits, fmt, meta, (1, C), orc.COLS)[0], (R, C), fmt, meta, (1, C),
                                  orc.COLS, out_dtype=bits.dtype)
    else:
        e = orc.emax(orc.histogram(bits))
        p = exmy.encode(d, fmt, e, axis="cols")
        full = orc.decode(orc.encode(bits, fmt, e, orc.COLS)[0], (R, C), fmt, e, orc.COLS, out_dtype=bits.dtype)
    got = exmy.decode_rows(p, torch.from_numpy(idx))
    np.testing.assert_array_equal(W.to_bits(got), full[idx])
    other = torch.bfloat16 if dt == "f32" else torch.float32
    got2 = exmy.decode_rows(p, torch.from_numpy(idx), dtype=other)
    np.testing.assert_array_equal(W.to_bits(got2), W.to_bits(exmy.decode(p, other))[idx])


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (6, 0), (0, 6), (5, 3), (3, 1), (1, 7), (8, 0)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_encode_rowwise_fused(exmy, orc, fmt, dt):
    """fused per-row metadata + encode == block max (row) + blocked encode"""
    # (4096, 264): more row groups than CTAs (each CTA reuses its staging buffer);
    # (16, 2304): fp32 rows of exactly the shared-memory staging limit (9216 B)
    for shape in [(64, 192), (24, 40), (8, 4104), (4096, 264), (16, 2304)]:
        bits = rowscaled_bits(shape, shape[1] + fmt[1], dt)
        d = W.from_bits(bits).to(DEV)
        for scheme in (0, 1):
            meta = orc.block_max_exponent(bits, (1, shape[1]), fmt[1], scheme)
            for axis in ("rows", "cols"):
                if axis == "cols" and shape[1] % 8:
                    continue
                ax = orc.ROWS if axis == "rows" else orc.COLS
                p = exmy.encode_rowwise(d, fmt, axis=axis, scheme=scheme, specials_capacity=bits.size)
                np.testing.assert_array_equal(p.meta.cpu().numpy(), meta, err_msg=f"meta {shape} {axis}")
                pref, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, (1, shape[1]), ax)
                np.testing.assert_array_equal(p.data.cpu().numpy(), pref, err_msg=f"packed {shape} {axis} {scheme}")
                spi, spb, cnt = p.specials()
                assert cnt == ns
                np.testing.assert_array_equal(spi.cpu().numpy(), idx)
                np.testing.assert_array_equal(W.to_bits(exmy.decode(p)),
                                              orc.quantize_blocked(bits, fmt, meta, (1, shape[1])))


def test_encode_rowwise_config2_shape(exmy, orc):
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=DEV)
    p = exmy.encode_rowwise(t, "e3m3")
    m = exmy.block_max_exponent(t, "row")
    assert torch.equal(p.meta, m)
    p2 = exmy.encode_blocked(t, "e3m3", m, "row")
    assert torch.equal(p.data, p2.data)


@pytest.mark.parametrize("cols", [64, 128, 256, 512])
@pytest.mark.parametrize("fmt", [(4, 2), (3, 1), (2, 4), (6, 0), (5, 3), (0, 6), (4, 3)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_per_row_cols_narrow_rows(exmy, orc, cols, fmt, dt):
    """Embedding-width tables (config 5: 128 columns) with one metadata byte per
    row, COLS packing: the narrow-row kernels (a warp tile = 128/gpr whole rows,
    one pipelined metadata load per tile) == the oracle, with a ragged last
    tile, rows of wildly different scale, NaN rows and bytes forced outside the
    fast ranges (0, 254) on some rows (integer path inside the tile)"""
    rows = 8 * 128 // (cols // 8) * 3 + 24          # three whole tiles and a ragged fourth
    bits = rowscaled_bits((rows, cols), cols + fmt[0], dt)
    d = W.from_bits(bits).to(DEV)
    meta = orc.block_max_exponent(bits, (1, cols))
    meta[5, 0], meta[17, 0], meta[rows - 1, 0] = 0, 254, 0
    m = torch.from_numpy(meta.copy()).to(DEV)
    p = exmy.encode_blocked(d, fmt, m, "row", axis="cols", specials_capacity=bits.size)
    pref, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, (1, cols), orc.COLS)
    np.testing.assert_array_equal(p.data.cpu().numpy(), pref)
    spi, spb, cnt = p.specials()
    assert cnt == ns and np.array_equal(spi.cpu().numpy(), idx)
    for od in (np.uint16, np.uint32):
        out = exmy.decode(p, torch.bfloat16 if od == np.uint16 else torch.float32)
        ref = orc.decode_blocked(pref, bits.shape, fmt, meta, (1, cols), orc.COLS, idx, sb, out_dtype=od)
        np.testing.assert_array_equal(W.to_bits(out), ref)


@pytest.mark.parametrize("fmt", [(3, 3), (6, 0), (2, 4), (4, 4), (1, 7)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_encode_rowwise_cluster_wide_rows(exmy, orc, fmt, dt):
    """With the A/B knob on, rows of 9 KB .. 72 KB take the thread-block-cluster kernel (column slabs
    in distributed shared memory, CL = 2 / 4 / 8): bytes, metadata, specials
    == the oracle's per-row encode (both schemes), and == the two-pass path
    (knob off)"""
    es = 2 if dt == "bf16" else 4
    for C in (9216 * 2 // es, 32768 // es, 73728 // es):    # CL = 2, 4, 8
        R = 24 if C * es <= 32768 else 16
        bits = rowscaled_bits((R, C), C + fmt[0], dt)
        d = W.from_bits(bits).to(DEV)
        for scheme in (0, 1):
            meta = orc.block_max_exponent(bits, (1, C), fmt[1], scheme)
            prev = exmy.rowwise_cluster(True)
            try:
                p = exmy.encode_rowwise(d, fmt, scheme=scheme, specials_capacity=bits.size)
            finally:
                exmy.rowwise_cluster(prev)
            np.testing.assert_array_equal(p.meta.cpu().numpy(), meta, err_msg=f"meta {C}")
            pref, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, (1, C), orc.ROWS)
            np.testing.assert_array_equal(p.data.cpu().numpy(), pref, err_msg=f"packed {C} scheme {scheme}")
            spi, spb, cnt = p.specials()
            assert cnt == ns and np.array_equal(spi.cpu().numpy(), idx)
            prev = exmy.rowwise_cluster(False)
            try:
                q = exmy.encode_rowwise(d, fmt, scheme=scheme, specials_capacity=bits.size)
            finally:
                exmy.rowwise_cluster(prev)
            assert torch.equal(p.data, q.data) and torch.equal(p.meta, q.meta)


def test_encode_rowwise_cluster_config2(exmy):
    """config 2 (16384^2 bf16, 32 KB rows): the cluster kernel == block max +
    blocked encode, many row groups per cluster"""
    t = W.bf16_weights((16384, 16384), seed=1, device=DEV)
    prev = exmy.rowwise_cluster(True)
    try:
        p = exmy.encode_rowwise(t, "e3m3", strict=False)
    finally:
        exmy.rowwise_cluster(prev)
    m = exmy.block_max_exponent(t, "row")
    assert torch.equal(p.meta, m)
    assert torch.equal(p.data, exmy.encode_blocked(t, "e3m3", m, "row", strict=False).data)
