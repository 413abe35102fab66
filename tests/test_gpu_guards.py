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
