"""GPU parity of the grouped launch with per-row metadata
(exmy_group_plan_rows; the paper's Llama recipe, "the maximum
exponent of each row"): every row's byte == exmy_block_max_exponent with
block (1, cols), the bytes == exmy_encode_blocked and the decode ==
exmy_decode_blocked on every entry's group_layout (those are pinned to the
oracle in test_gpu_blocked), and == the oracle directly on small entries."""
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


# per-row plans need cols % 8 == 0: Llama-like mix of wide / tall / tiny
# matrices, 1-D vectors (packed as (8, n/8)), an empty entry
# (encode with derived metadata = exmy_group_encode_rowwise: rows <= 9216 B are
# staged in shared memory, (8, 4616) bf16 / the wide fp32 rows take two passes)
SHAPES = [(64, 4096), (8, 8), (0, 16), (4096,), (200, 40), (1024, 136), (8, 1032), (24, 8), (512,), (16, 2048),
          (8, 4616)]


def table(dt, seed, specials=False, extreme=False):
    """rows scaled by 2^U(-40, 40) so the per-row bytes differ; extreme: a few
    rows at the top / bottom of the range (metadata outside the fast paths)"""
    rng = np.random.default_rng(seed)
    ts = []
    for i, s in enumerate(SHAPES):
        if len(s) == 1:
            t = torch.ones(s, dtype=torch.float32) * float(rng.uniform(0.5, 2.0))
        else:
            t = W.f32_wide(s, seed=seed + i) if s[0] else torch.zeros(s)
            if s[0]:
                sc = torch.from_numpy(np.exp2(rng.integers(-40, 40, size=(s[0], 1))).astype(np.float32))
                t = t * sc
                if extreme and s[0] >= 8:
                    t[1] = t[1] / t[1].abs().max() * 2.0 ** 120
                    t[2] = t[2] / t[2].abs().max() * 2.0 ** -120
                    t[3] = 0.0
        if specials and t.numel() >= 64:
            flat = t.view(-1)
            idx = torch.from_numpy(rng.choice(t.numel(), size=5, replace=False))
            flat[idx] = torch.tensor([float("nan"), float("inf"), float("-inf"), float("nan"), 3.0])
        ts.append(t.to(torch.bfloat16 if dt == "bf16" else torch.float32).to(DEV))
    return ts


def check_against_blocked(exmy, ts, g, fmt, cap=0):
    packed = g.encode()
    fused_meta = g.meta.clone()
    g.max_exponent()                      # the separate row-bytes pass agrees with the fused one
    assert torch.equal(g.meta, fused_meta)
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        v = t.reshape(lay) if t.numel() else t.reshape(0, lay[1])
        if v.numel() == 0:
            continue
        m = exmy.block_max_exponent(v, "row")
        assert torch.equal(p.meta.reshape(-1), m.reshape(-1)), tuple(t.shape)
        ref = exmy.encode_blocked(v, fmt, m, "row", axis="rows", specials_capacity=max(cap, 1))
        assert torch.equal(p.data, ref.data), (tuple(t.shape), fmt)
        if cap:
            a, b, c = p.specials()
            ra, rb, rc = ref.specials()
            assert c == rc and torch.equal(a, ra) and torch.equal(b, rb)
        d = exmy.decode(ref, o.dtype)
        assert torch.equal(o.reshape(lay).view(torch.uint8), d.view(torch.uint8)), (tuple(t.shape), fmt)
        assert torch.equal(o.view(torch.uint8), exmy.decode(p, o.dtype).view(torch.uint8))


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (4, 2), (6, 0), (0, 6), (1, 1), (3, 0), (5, 3), (3, 5), (8, 0),
                                 (0, 8), (2, 1)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("odt", ["same", "other"])
def test_group_rows_equals_blocked(exmy, fmt, dt, odt):
    ts = table(dt, 10 * fmt[0] + fmt[1])
    out = None if odt == "same" else (torch.float32 if dt == "bf16" else torch.bfloat16)
    g = exmy.GroupCodec(ts, fmt, out_dtype=out, per_row=True)
    check_against_blocked(exmy, ts, g, fmt)


@pytest.mark.parametrize("fmt", [(3, 3), (2, 2), (4, 3), (0, 7)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_group_rows_oracle_small(exmy, orc, fmt, dt):
    """entries small enough for the oracle: per-row bytes, packed bytes and
    decode against oracle_block_max_exponent / encode_blocked / decode_blocked"""
    ts = table(dt, 7 + fmt[1])
    g = exmy.GroupCodec(ts, fmt, out_dtype=torch.float32, per_row=True)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        if t.numel() == 0 or t.numel() > 300000:
            continue
        bits = W.to_bits(t.cpu()).reshape(lay)
        meta = orc.block_max_exponent(bits, (1, lay[1]))
        np.testing.assert_array_equal(p.meta.cpu().numpy().reshape(-1), meta.reshape(-1))
        pref = orc.encode_blocked(bits, fmt, meta, (1, lay[1]), orc.ROWS)[0]
        np.testing.assert_array_equal(p.data.cpu().numpy(), pref)
        dref = orc.decode_blocked(pref, lay, fmt, meta, (1, lay[1]), orc.ROWS, out_dtype=np.uint32)
        np.testing.assert_array_equal(W.to_bits(o.cpu()).reshape(lay), dref)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("fmt", [(3, 2), (2, 5), (5, 2)], ids=lambda f: f"e{f[0]}m{f[1]}")
def test_group_rows_specials_and_extreme_rows(exmy, dt, fmt):
    """NaN/Inf (per-entry sorted specials lists, restored by decode) and rows
    whose metadata is outside the fast ranges (2^120, 2^-120, all-zero rows)"""
    ts = table(dt, 3, specials=True, extreme=True)
    g = exmy.GroupCodec(ts, fmt, specials_capacity=64, per_row=True)
    check_against_blocked(exmy, ts, g, fmt, cap=64)


def test_group_rows_forced_meta_force_generic_and_graph(exmy):
    ts = table("bf16", 5)
    g = exmy.GroupCodec(ts, "e2m3", per_row=True)
    ref = [p.data.clone() for p in g.encode()]
    dref = [o.clone() for o in g.decode()]
    exmy.force_generic(True)
    try:
        g2 = exmy.GroupCodec(ts, "e2m3", per_row=True)
        assert all(torch.equal(a.data, b) for a, b in zip(g2.encode(), ref))
        assert all(torch.equal(a, b) for a, b in zip(g2.decode(), dref))
    finally:
        exmy.force_generic(False)
    # caller-supplied row bytes (every row 0 / 254 / a ramp)
    n = g.meta.numel()
    for meta in (torch.zeros(n, dtype=torch.uint8), torch.full((n,), 254, dtype=torch.uint8),
                 (torch.arange(n) % 255).to(torch.uint8)):
        packed = g.encode(meta.to(DEV))
        outs = g.decode()
        for t, p, o, lay in zip(ts, packed, outs, g.layouts):
            if t.numel() == 0:
                continue
            v = t.reshape(lay)
            r = exmy.encode_blocked(v, "e2m3", p.meta.reshape(lay[0], 1), "row", specials_capacity=1)
            assert torch.equal(p.data, r.data)
            assert torch.equal(o.reshape(lay).view(torch.uint8), exmy.decode(r).view(torch.uint8))
    # CUDA-graph capture of max + encode + decode
    g.encode()
    for p in g.packed:
        p.zero_()
    g.meta.zero_()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.encode()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(graph):
        g.encode()
        g.decode()
    for p in g.packed:
        p.zero_()
    for o in g.outs:
        o.zero_()
    g.meta.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(g.packed, ref))
    assert all(torch.equal(a, b) for a, b in zip(g.outs, dref))


def test_group_rows_llama_shapes_sampled(exmy):
    """Config 3's table (first 2 layers + embeddings / head) under the
    per-row recipe: row bytes, packed bytes and decode == per-tensor calls"""
    shapes = [s for s in W.llama3_8b_shapes() if not s[0].startswith("layers.") or int(s[0].split(".")[1]) < 2]
    ts = []
    for i, (name, shp) in enumerate(shapes):
        ts.append(torch.ones(shp, dtype=torch.bfloat16, device=DEV) if len(shp) == 1
                  else W.bf16_weights(shp, seed=1000 + i, device=DEV))
    g = exmy.GroupCodec(ts, "e3m3", per_row=True)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        v = t.reshape(lay)
        m = exmy.block_max_exponent(v, "row")
        assert torch.equal(p.meta.reshape(-1), m.reshape(-1))
        ref = exmy.encode_blocked(v, "e3m3", m, "row", specials_capacity=1)
        assert torch.equal(p.data, ref.data)
        assert torch.equal(o.reshape(lay), exmy.decode(ref))
