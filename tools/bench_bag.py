"""Embedding bag fused with decode vs the unfused pipeline (row gather-decode
to HBM, then a torch pool), config 5 at one shard of 8: a (12.5 M, 128) fp32
table packed COLS, DLRM-style bags.
python tools/bench_bag.py [--rows 12500000] [--bags 65536] [--pool 32] [--fmt e4m2]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=12_500_000)
    ap.add_argument("--cols", type=int, default=128)
    ap.add_argument("--bags", type=int, default=65536)
    ap.add_argument("--pool", type=int, default=32)
    ap.add_argument("--fmt", default="e4m2")
    ap.add_argument("--per-row", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    t = W.f32_embedding(a.rows, a.cols, device=dev)
    if a.per_row:
        p = exmy.encode_blocked(t, a.fmt, None, "row", axis="cols")
    else:
        p = exmy.encode(t, a.fmt, axis="cols")
    del t
    g = torch.Generator(device=dev).manual_seed(1)
    nidx = a.bags * a.pool
    idx = torch.randint(0, a.rows, (nidx,), device=dev, generator=g, dtype=torch.int64)
    off = torch.arange(0, nidx + 1, a.pool, device=dev, dtype=torch.int64)
    out = torch.empty((a.bags, a.cols), dtype=torch.float32, device=dev)
    rows_buf = torch.empty((nidx, a.cols), dtype=torch.float32, device=dev)
    k = p.k
    fused = timeit(lambda: exmy.embedding_bag(p, idx, off, out=out))
    unfused = timeit(lambda: (exmy.decode_rows(p, idx, out=rows_buf), torch.sum(rows_buf.view(a.bags, a.pool, a.cols), 1, out=out)))
    packed_b = nidx * a.cols * k / 8 + nidx * 8            # gathered packed rows + indices
    res = {"rows": a.rows, "cols": a.cols, "bags": a.bags, "pool": a.pool, "fmt": a.fmt, "per_row": a.per_row,
           "fused_ms": round(fused, 4), "fused_Glookups_s": round(nidx / fused / 1e6, 3),
           "fused_gbs": round((packed_b + a.bags * a.cols * 4) / fused / 1e6, 1),
           "unfused_ms": round(unfused, 4), "unfused_Glookups_s": round(nidx / unfused / 1e6, 3),
           "speedup": round(unfused / fused, 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
