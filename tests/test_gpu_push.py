"""GPU parity of the fused encode + all-gather (exmy_encode_push; SURVEY 8(f)
row 2): every rank's shard encode writes its bytes into every destination
buffer at the global offsets.  On one GPU the "peers" are local buffers: after
all shards ran, each buffer == the single-GPU encode of the whole tensor ==
the oracle, and the shards' specials lists (global indices) concatenate to
the whole tensor's list."""
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


def bits_with_specials(shape, seed, dt):
    t = W.f32_wide(shape, seed=seed)
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t).copy()
    rng = np.random.default_rng(seed)
    flat = bits.reshape(-1)
    idx = rng.choice(flat.size, size=9, replace=False)
    flat[idx[:5]] = 0x7FC0 if dt == "bf16" else 0x7FC00000
    flat[idx[5:]] = 0xFF80 if dt == "bf16" else 0xFF800000
    return bits


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (6, 0), (0, 6), (4, 3), (3, 5), (8, 0), (2, 1)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("G", [1, 4])
def test_push_equals_whole_encode(exmy, orc, fmt, dt, G):
    R, C = 256, 192
    bits = bits_with_specials((R, C), fmt[0] * 7 + fmt[1], dt)
    t = W.from_bits(bits).to(DEV)
    e = orc.emax(orc.histogram(bits))
    k = 1 + fmt[0] + fmt[1]
    ndst = 3
    bufs = [torch.full((R * C * k // 8,), 0xA5, dtype=torch.uint8, device=DEV) for _ in range(ndst)]
    per = R // G
    idxs = []
    for r in range(G):
        spi, spb, spc = exmy.encode_push(t[r * per:(r + 1) * per], fmt, e, r * per, R, bufs,
                                         specials_capacity=R * C)
        cnt = int(spc[0].item())
        idxs.append(spi[:cnt].cpu().numpy())
    torch.cuda.synchronize()
    pref, idx, sb, ns = orc.encode(bits, fmt, e, orc.ROWS)
    whole = exmy.encode(t, fmt, e, specials_capacity=R * C)
    for b in bufs:
        np.testing.assert_array_equal(b.cpu().numpy(), pref)
        assert torch.equal(b, whole.data)
    np.testing.assert_array_equal(np.concatenate(idxs), idx)


def test_push_forced_meta_generic_tiles(exmy, orc):
    """metadata outside the fast range -> the integer path stores to every buffer"""
    R, C = 64, 96
    bits = bits_with_specials((R, C), 3, "bf16")
    t = W.from_bits(bits).to(DEV)
    for e in (0, 254):
        bufs = [torch.zeros(R * C * 7 // 8, dtype=torch.uint8, device=DEV) for _ in range(2)]
        for r in range(2):
            exmy.encode_push(t[r * 32:(r + 1) * 32], "e3m3", e, r * 32, R, bufs, specials_capacity=R * C)
        ref = orc.encode(bits, "e3m3", e, orc.ROWS)[0]
        for b in bufs:
            np.testing.assert_array_equal(b.cpu().numpy(), ref)


def test_push_large_shards(exmy):
    """config-2-like width, 8 shards of 2048 rows, 8 destinations"""
    R, C = 16384, 4096
    t = W.bf16_weights((R, C), seed=4, device=DEV)
    m = exmy.max_exponent(t)
    whole = exmy.encode(t, "e3m3", m)
    bufs = [torch.zeros(R * C * 7 // 8, dtype=torch.uint8, device=DEV) for _ in range(8)]
    for r in range(8):
        exmy.encode_push(t[r * 2048:(r + 1) * 2048], "e3m3", m, r * 2048, R, bufs)
    for b in bufs:
        assert torch.equal(b, whole.data)


def test_push_argument_errors(exmy):
    t = torch.zeros((16, 8), dtype=torch.bfloat16, device=DEV)
    buf = torch.zeros(64 * 8 * 7 // 8, dtype=torch.uint8, device=DEV)
    with pytest.raises(exmy.ExmyError):
        exmy.encode_push(t, "e3m3", 100, 4, 64, [buf])          # row0 % 8
    with pytest.raises(exmy.ExmyError):
        exmy.encode_push(t, "e3m3", 100, 56, 64, [buf])         # past the end
    with pytest.raises(exmy.ExmyError):
        exmy.encode_push(t, "e3m3", 100, 0, 64, [buf] * 9)      # > 8 destinations


@pytest.mark.parametrize("fmt", [(3, 3), (2, 4), (6, 0), (4, 3), (3, 5), (8, 0), (0, 8), (1, 7)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_pull_decode_equals_whole_decode(exmy, orc, fmt, dt):
    """exmy_decode_pull over G independently encoded row shards (global e_max)
    == decode of the whole tensor == the oracle's quantize (no specials)"""
    R, C = 256, 192
    t = W.f32_wide((R, C), seed=fmt[0] * 3 + fmt[1])
    if dt == "bf16":
        t = t.to(torch.bfloat16)
    bits = W.to_bits(t)
    d = t.to(DEV)
    e = orc.emax(orc.histogram(bits))
    ref = orc.quantize(bits, fmt, e)
    for G in (1, 4, 8):
        per = R // G
        shards = [exmy.encode(d[r * per:(r + 1) * per], fmt, e).data for r in range(G)]
        for odt in (torch.bfloat16, torch.float32):
            out = exmy.decode_pull(shards, per, C, fmt, e, dtype=odt)
            whole = exmy.decode(exmy.encode(d, fmt, e), odt)
            assert torch.equal(out.view(torch.uint8), whole.view(torch.uint8)), (G, odt)
        same = exmy.decode_pull(shards, per, C, fmt, e, dtype=t.dtype)
        np.testing.assert_array_equal(W.to_bits(same), ref)


def test_pull_decode_large_emax_two_multiplies(exmy):
    """o > 127 (metadata near the top): the two-multiply fast path"""
    t = (torch.randn(64, 256) * 2.0 ** 120).to(torch.bfloat16).to(DEV)
    m = exmy.max_exponent(t)
    shards = [exmy.encode(t[i * 16:(i + 1) * 16], "e2m3", m).data for i in range(4)]
    out = exmy.decode_pull(shards, 16, 256, "e2m3", m, dtype=torch.bfloat16)
    assert torch.equal(out, exmy.quantize(t, "e2m3", m))
