"""GPU parity of the grouped launch (include/exmy.h "grouped launch", SURVEY
8(f) row 4): per-tensor metadata, ROWS encode and decode of a whole tensor
table == the per-tensor calls on every entry (which are themselves pinned
to the oracle), and == the oracle directly on the small entries."""
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


# a Llama-like mix: wide and tall matrices spanning many chunks, small ones
# inside one chunk, a 1-D norm vector, an empty tensor, ragged chunk tails
SHAPES = [(64, 4096), (8, 4), (0, 16), (4096,), (200, 36), (1024, 136), (8, 1028), (24, 4), (512,), (16, 2048)]


SHAPES8 = [s for s in SHAPES if len(s) == 1 or s[1] % 8 == 0]   # bf16 output: 8x8 decode tiles


def table(dt, seed, specials=False, shapes=SHAPES):
    rng = np.random.default_rng(seed)
    ts = []
    for i, s in enumerate(shapes):
        if len(s) == 1:
            t = torch.ones(s, dtype=torch.float32) * float(rng.uniform(0.5, 2.0))
        else:
            t = W.f32_wide(s, seed=seed + i) if s[0] else torch.zeros(s)
            t = t * float(2.0 ** rng.integers(-30, 30))
        if specials and t.numel() >= 64:
            flat = t.view(-1)
            idx = torch.from_numpy(rng.choice(t.numel(), size=5, replace=False))
            flat[idx] = torch.tensor([float("nan"), float("inf"), float("-inf"), float("nan"), 3.0])
        ts.append(t.to(torch.bfloat16 if dt == "bf16" else torch.float32).to(DEV))
    return ts


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (4, 2), (6, 0), (0, 6), (1, 1), (3, 0), (5, 3), (3, 5), (8, 0),
                                 (0, 8), (2, 1)], ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("shapes", ["mixed", "cols8"])
def test_group_equals_per_tensor(exmy, fmt, dt, shapes):
    ts = table(dt, 10 * fmt[0] + fmt[1], shapes=SHAPES if shapes == "mixed" else SHAPES8)
    g = exmy.GroupCodec(ts, fmt)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        v = t.reshape(lay) if t.numel() else t.reshape(0, lay[1])
        m = exmy.max_exponent(t)
        assert p.meta.item() == m.item()
        ref = exmy.encode(v, fmt, m, axis="rows", specials_capacity=0)
        assert torch.equal(p.data, ref.data), (tuple(t.shape), fmt)
        assert torch.equal(o.view(torch.uint8), exmy.decode(p).view(torch.uint8))
        assert torch.equal(o.reshape(lay).view(torch.uint8), exmy.decode(ref).view(torch.uint8))


@pytest.mark.parametrize("fmt", [(3, 3), (2, 1), (0, 7), (4, 4)], ids=lambda f: f"e{f[0]}m{f[1]}")
def test_group_oracle_small(exmy, orc, fmt):
    """entries small enough for the oracle: bytes and decode against it"""
    ts = table("bf16", 7 + fmt[1])
    g = exmy.GroupCodec(ts, fmt, out_dtype=torch.float32)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        if t.numel() == 0 or t.numel() > 300000:
            continue
        bits = W.to_bits(t.cpu()).reshape(lay)
        e = orc.emax(orc.histogram(bits))
        assert p.meta.item() == e
        pref = orc.encode(bits, fmt, e, orc.ROWS)[0]
        np.testing.assert_array_equal(p.data.cpu().numpy(), pref)
        dref = orc.decode(pref, lay, fmt, e, orc.ROWS, out_dtype=np.uint32)
        np.testing.assert_array_equal(W.to_bits(o.cpu()).reshape(lay), dref)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_group_specials_and_forced_meta(exmy, dt):
    """NaN/Inf: per-entry sorted specials lists == exmy.encode's, restored by
    decode; metadata outside the fast range (0, 254) -> integer paths."""
    ts = table(dt, 3, specials=True)
    g = exmy.GroupCodec(ts, "e3m2", specials_capacity=64)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        v = t.reshape(lay) if t.numel() else t.reshape(0, lay[1])
        ref = exmy.encode(v, "e3m2", p.meta, specials_capacity=64)
        assert torch.equal(p.data, ref.data)
        a, b, c = p.specials()
        ra, rb, rc = ref.specials()
        assert c == rc and torch.equal(a, ra) and torch.equal(b, rb)
        assert torch.equal(o.view(torch.uint8), exmy.decode(ref).reshape(t.shape).view(torch.uint8))
    # forced metadata: every entry under e_max 0 / 254 / 100
    for e in (0, 254, 100):
        meta = torch.full((len(ts),), e, dtype=torch.uint8, device=DEV)
        packed = g.encode(meta)
        outs = g.decode()
        for t, p, o, lay in zip(ts, packed, outs, g.layouts):
            v = t.reshape(lay) if t.numel() else t.reshape(0, lay[1])
            ref = exmy.encode(v, "e3m2", e, specials_capacity=64)
            assert torch.equal(p.data, ref.data), (e, tuple(t.shape))
            assert torch.equal(o.view(torch.uint8), exmy.decode(ref).reshape(t.shape).view(torch.uint8))


def test_group_force_generic_and_graph(exmy):
    ts = table("bf16", 5)
    g = exmy.GroupCodec(ts, "e2m3")
    ref = [p.data.clone() for p in g.encode()]
    dref = [o.clone() for o in g.decode()]
    exmy.force_generic(True)
    try:
        g2 = exmy.GroupCodec(ts, "e2m3")
        assert all(torch.equal(a.data, b) for a, b in zip(g2.encode(), ref))
        assert all(torch.equal(a, b) for a, b in zip(g2.decode(), dref))
    finally:
        exmy.force_generic(False)
    # CUDA-graph capture of the whole-model encode + decode
    for p in g.packed:
        p.zero_()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.encode()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        g.encode()
        g.decode()
    for p in g.packed:
        p.zero_()
    for o in g.outs:
        o.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(g.packed, ref))
    assert all(torch.equal(a, b) for a, b in zip(g.outs, dref))


def test_group_llama_shapes_sampled(exmy):
    """Config 3's table (Llama-3-8B, 291 tensors, first 2 layers here): meta
    and bytes of every tensor == per-tensor calls."""
    shapes = [s for s in W.llama3_8b_shapes() if not s[0].startswith("layers.") or int(s[0].split(".")[1]) < 2]
    ts = []
    for i, (name, shp) in enumerate(shapes):
        ts.append(torch.ones(shp, dtype=torch.bfloat16, device=DEV) if len(shp) == 1
                  else W.bf16_weights(shp, seed=1000 + i, device=DEV))
    g = exmy.GroupCodec(ts, "e3m3", decode_outputs=True)
    packed = g.encode()
    outs = g.decode()
    for t, p, o, lay in zip(ts, packed, outs, g.layouts):
        m = exmy.max_exponent(t)
        assert p.meta.item() == m.item()
        ref = exmy.encode(t.reshape(lay), "e3m3", m, specials_capacity=0)
        assert torch.equal(p.data, ref.data)
        assert torch.equal(o.reshape(lay), exmy.decode(ref))
