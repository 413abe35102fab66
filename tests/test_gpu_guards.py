"""Out-of-bounds write guards (compute-sanitizer is closed on the GPU pool):
every output buffer is a view into a larger allocation whose 4 KB before and
after are filled with a canary pattern; after each op on ragged shapes the
canaries must be intact and the result must equal the op on a plain buffer."""
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"
PAD = 4096
CANARY = 0xA5


@pytest.fixture(scope="module")
def exmy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as m
    m.force_generic(False)
    return m


class Guarded:
    """a tensor of `shape` / `dtype` carved out of a canary-filled byte slab"""

    def __init__(self, shape, dtype):
        n = 1
        for s in shape:
            n *= s
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        self.slab = torch.full((nbytes + 2 * PAD,), CANARY, dtype=torch.uint8, device=DEV)
        self.nbytes = nbytes
        self.t = self.slab[PAD:PAD + nbytes].view(dtype).view(shape)

    def intact(self):
        torch.cuda.synchronize()
        return bool((self.slab[:PAD] == CANARY).all()) and bool((self.slab[PAD + self.nbytes:] == CANARY).all())


SHAPES = [(8, 8 * 35), (24, 8 * 37), (64, 8 * 129)]     # ragged against 256-thread column blocks


@pytest.mark.parametrize("shape", SHAPES, ids=str)
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("fmt", ["e3m3", "e6m0", "e4m3", "e3m5", "e8m0", "e1m1"])
def test_codec_writes_stay_in_bounds(exmy, shape, dt, fmt):
    R, C = shape
    t = W.f32_wide(shape, seed=R + C).to(dt).to(DEV)
    t.view(-1)[3] = float("inf")
    m = exmy.max_exponent(t)
    k = 1 + sum(exmy.parse_format(fmt))
    q = Guarded(shape, dt)
    exmy.quantize(t, fmt, m, out=q.t)
    assert q.intact() and torch.equal(q.t, exmy.quantize(t, fmt, m))
    for axis in ("rows", "cols"):
        pk = Guarded((R * C * k // 8,), torch.uint8)
        p = exmy.encode(t, fmt, m, axis=axis, out=pk.t)
        assert pk.intact() and torch.equal(pk.t, exmy.encode(t, fmt, m, axis=axis).data)
        for odt in (torch.bfloat16, torch.float32):
            o = Guarded(shape, odt)
            exmy.decode(p, odt, out=o.t)
            assert o.intact() and torch.equal(o.t, exmy.decode(p, odt))
        for blk in ("row", (1, 8), (8, 4)):
            meta = exmy.block_max_exponent(t, blk)
            pb = Guarded((R * C * k // 8,), torch.uint8)
            pp = exmy.encode_blocked(t, fmt, meta, blk, axis=axis, out=pb.t)
            assert pb.intact()
            ob = Guarded(shape, dt)
            exmy.decode(pp, out=ob.t)
            assert ob.intact() and torch.equal(ob.t, exmy.quantize_blocked(t, fmt, meta, blk))
        pf = Guarded((R * C * k // 8,), torch.uint8)
        pfs = exmy.encode_fs(t, fmt, None, "row", axis=axis, out=pf.t)
        assert pf.intact()
        of = Guarded(shape, dt)
        exmy.decode(pfs, out=of.t)
        assert of.intact() and torch.equal(of.t, exmy.quantize_fs(t, fmt, None, "row"))


@pytest.mark.parametrize("fmt", ["e3m3", "e4m2", "e3m5"])
def test_gather_bag_push_pull_in_bounds(exmy, fmt):
    R, C = 64, 8 * 37
    t = W.f32_wide((R, C), seed=2).to(DEV)
    m = exmy.max_exponent(t)
    k = 1 + sum(exmy.parse_format(fmt))
    pc = exmy.encode(t, fmt, m, axis="cols")
    idx = torch.tensor([5, 63, 0, 5, 17], dtype=torch.int64)
    g = Guarded((5, C), torch.float32)
    exmy.decode_rows(pc, idx, out=g.t)
    assert g.intact() and torch.equal(g.t, exmy.decode_rows(pc, idx))
    b = Guarded((3, C), torch.float32)
    off = torch.tensor([0, 2, 2, 5], dtype=torch.int64)
    exmy.embedding_bag(pc, idx, off, out=b.t)
    assert b.intact() and torch.equal(b.t, exmy.embedding_bag(pc, idx, off))
    dsts = [Guarded((R * C * k // 8,), torch.uint8) for _ in range(3)]
    for r in range(4):
        exmy.encode_push(t[16 * r:16 * (r + 1)], fmt, m, 16 * r, R, [d.t for d in dsts])
    whole = exmy.encode(t, fmt, m).data
    assert all(d.intact() and torch.equal(d.t, whole) for d in dsts)
    shards = [exmy.encode(t[16 * r:16 * (r + 1)], fmt, m).data for r in range(4)]
    o = Guarded((R, C), torch.float32)
    exmy.decode_pull(shards, 16, C, fmt, m, out=o.t)
    assert o.intact() and torch.equal(o.t, exmy.decode(exmy.encode(t, fmt, m), torch.float32))


def test_roofline_probe_runs_and_validates(exmy):
    """exmy_debug_probe (SURVEY 8(d) roofline probe): streams the bytes it is
    given; the output share of each chunk lands inside the output buffer"""
    src = torch.zeros(64 * 1024, dtype=torch.uint8, device=DEV)
    o = Guarded((7 * 1024 + 16 * 5,), torch.uint8)
    exmy.roofline_probe(src, o.nbytes, out=o.t)
    assert o.intact()
    with pytest.raises(exmy.ExmyError):
        exmy.roofline_probe(src[:1000], 16)          # input not a multiple of 16 KB
    with pytest.raises(exmy.ExmyError):
        exmy.roofline_probe(src, 17)                 # output not a multiple of 16 B


def test_capacity_zero_specials_never_scatter(exmy):
    """an encode with specials capacity 0 still counts NaN/Inf;
    the decode must scatter min(count, capacity) = 0 entries (no write through
    an unwritten index), and strict encodes refuse the overflow."""
    t = W.bf16_weights((64, 256), seed=3, device=DEV)
    t.view(-1)[[7, 300, 5000]] = torch.tensor([float("nan"), float("inf"), float("-inf")], dtype=torch.bfloat16,
                                               device=DEV)
    p = exmy.encode(t, "e3m3", specials_capacity=0, strict=False)
    assert int(p.sp_count[0].item()) == 3 and p.capacity == 0
    p.sp_index.fill_(1 << 40)      # garbage an unguarded scatter would write through
    g = Guarded(t.shape, torch.bfloat16)
    exmy.decode(p, out=g.t)
    assert g.intact()
    ref = exmy.decode(exmy.encode(t, "e3m3", p.meta))          # with the lists
    keep = torch.ones(t.numel(), dtype=torch.bool, device=DEV)
    keep[[7, 300, 5000]] = False
    assert torch.equal(g.t.reshape(-1)[keep].view(torch.int16), ref.reshape(-1)[keep].view(torch.int16))
    assert int(g.t.reshape(-1)[7].view(torch.int16)) == 0      # in-band code 0 -> +0
    with pytest.raises(exmy.ExmyError) as ei:
        exmy.encode(t, "e3m3", specials_capacity=2)
    assert ei.value.status == 6
    q = exmy.encode(t, "e3m3", specials_capacity=3)            # exactly enough
    idx, bits, cnt = q.specials()
    assert cnt == 3 and idx.tolist() == [7, 300, 5000]


def test_group_codec_default_capacity_zero(exmy):
    """GroupCodec's default capacity 0 with NaN in a member: decode stays in bounds"""
    a = W.bf16_weights((64, 128), seed=4, device=DEV)
    a.view(-1)[11] = float("nan")
    g = exmy.GroupCodec([a, W.bf16_weights((32, 64), seed=5, device=DEV)], "e2m4")
    ps = g.encode()
    assert ps[0].capacity == 0 and int(ps[0].sp_count[0].item()) == 1
    outs = g.decode()
    torch.cuda.synchronize()
    d = exmy.decode(ps[0])
    assert int(d.reshape(-1)[11].view(torch.int16)) == 0 and torch.equal(d, outs[0])


def test_gather_index_validation(exmy):
    t = W.f32_embedding(100, 128, seed=9).to(DEV)
    p = exmy.encode(t, "e4m2", axis="cols")
    with pytest.raises(IndexError):
        exmy.decode_rows(p, torch.tensor([0, 100]))
    with pytest.raises(IndexError):
        exmy.decode_rows(p, torch.tensor([-1]))
    with pytest.raises(IndexError):
        exmy.embedding_bag(p, torch.tensor([3, 1000]), torch.tensor([0, 2]))
    with pytest.raises(ValueError):
        exmy.embedding_bag(p, torch.tensor([3, 4]), torch.tensor([0, 3]))
