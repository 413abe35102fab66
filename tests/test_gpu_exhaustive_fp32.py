"""Exhaustive fp32 parity (SURVEY 8(c) coverage plan):
every one of the 2^32 fp32 bit patterns, generated on the device
(torch.arange reinterpreted as fp32), through quantize and ROWS encode for
the six (format, e_max) pairs the plan names -- e3m2@131 (OCP FP6 E3M2),
e2m3@129 (FP6 E2M3), e4m3@135 (OCP E4M3 scale), e5m3@116, e6m0@124 (y = 0
ties, reading D6) and e0m6@120 (linear) -- compared bit for bit, chunk by
chunk, with the CPU oracle run on all host cores: quantized values, packed
bytes, and the ordered NaN/Inf lists.  The fp32 fast path (one FADD per
element) is what the RTNE claim rests on; this checks it on
every input, subnormals, ties, saturation and specials included."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAIRS = [((3, 2), 131), ((2, 3), 129), ((4, 3), 135), ((5, 3), 116), ((6, 0), 124), ((0, 6), 120)]
CHUNK = 1 << 26          # patterns per chunk: a (16384, 4096) fp32 tensor
COLS = 4096


@pytest.fixture(scope="module")
def exmy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as m
    m.force_generic(False)
    return m


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


@pytest.mark.parametrize("fmt,e_max", PAIRS, ids=lambda v: f"e{v[0]}m{v[1]}" if isinstance(v, tuple) else str(v))
def test_all_fp32_patterns(exmy, orc, fmt, e_max):
    x, y = fmt
    k = 1 + x + y
    rows = CHUNK // COLS
    nthr = max(1, min(_cores(), 32))
    slab = rows // nthr // 8 * 8 or 8
    starts = list(range(0, rows, slab))
    ws, offs = exmy.segments(k, CHUNK)
    meta = torch.tensor([e_max], dtype=torch.uint8, device="cuda")
    cap = 1 << 23
    pool = ThreadPoolExecutor(max_workers=len(starts))
    total_specials = 0
    for c in range((1 << 32) // CHUNK):
        lo = c * CHUNK
        d = torch.arange(lo, lo + CHUNK, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.float32)
        d = d.view(rows, COLS)
        q = exmy.quantize(d, fmt, meta).view(torch.int32).cpu().numpy().view(np.uint32)
        p = exmy.encode(d, fmt, meta, specials_capacity=cap)
        pk = p.data.cpu().numpy()
        gi, gb, gn = p.specials()
        gi, gb = gi.cpu().numpy(), gb.cpu().numpy().view(np.uint32)
        bits = np.arange(lo, lo + CHUNK, dtype=np.uint64).astype(np.uint32).reshape(rows, COLS)

        def one(r0):
            # the oracle's encode, and its decode of those bytes to fp32 (decode(encode(x)) ==
            # quantize(x) is pinned in test_oracle_pins): half the oracle time of a separate quantize
            sb = bits[r0:r0 + slab]
            enc = orc.encode(sb, fmt, e_max, orc.ROWS)
            dq = orc.decode(enc[0], sb.shape, fmt, e_max, orc.ROWS, enc[1], enc[2], out_dtype=np.uint32)
            return r0, dq, enc

        idx_all, bits_all = [], []
        for r0, oq, (opk, oi, ob, ons) in pool.map(one, starts):
            np.testing.assert_array_equal(q[r0:r0 + slab], oq, err_msg=f"quantize chunk {c:#x} rows {r0}")
            n_s = slab * COLS
            got = np.concatenate([pk[o + r0 * COLS * w // 8: o + r0 * COLS * w // 8 + n_s * w // 8]
                                  for w, o in zip(ws, offs)])
            np.testing.assert_array_equal(got, opk, err_msg=f"encode chunk {c:#x} rows {r0}")
            idx_all.append(oi + r0 * COLS)
            bits_all.append(ob)
        oi = np.concatenate(idx_all)
        ob = np.concatenate(bits_all)
        assert gn == oi.size
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gb, ob)
        total_specials += gn
    pool.shutdown()
    assert total_specials == 2 << 23      # every NaN payload and both infinities, each sign
