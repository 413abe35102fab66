"""Embedding lookup throughput (config 5 access pattern): a COLS-packed fp32
table (rows x 128) decoded at B random row indices per call.
python tools/bench_gather.py [--rows 10000000] [--fmt e4m2] [--per-row]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402
from tools.bench_ops import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--cols", type=int, default=128)
    ap.add_argument("--fmt", default="e4m2")
    ap.add_argument("--per-row", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    t = W.f32_embedding(a.rows, a.cols, seed=5, device=dev)
    x, y = exmy.parse_format(a.fmt)
    k = 1 + x + y
    if a.per_row:
        p = exmy.encode_blocked(t, a.fmt, None, "row", axis="cols")
    else:
        p = exmy.encode(t, a.fmt, axis="cols")
    del t
    torch.cuda.empty_cache()
    peak = 6555.5
    res = {}
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for B in (2048, 65536, 1 << 20):
        idx = torch.randint(0, a.rows, (B,), device=dev, generator=g)
        out = torch.empty((B, a.cols), dtype=torch.float32, device=dev)
        ms = timeit(lambda: exmy.decode_rows(p, idx, out=out), reps=50)
        alg = B * (a.cols * k // 8 + a.cols * 4 + 8)
        res[B] = {"us": ms * 1e3, "rows_per_s": B / ms * 1e3, "hbm_gbs": alg / ms / 1e6, "frac": alg / ms / 1e6 / peak}
        print(f"B={B:8d} {ms * 1e3:9.1f} us {B / ms * 1e3 / 1e6:9.2f} Mrows/s {alg / ms / 1e6:8.1f} GB/s "
              f"{100 * alg / ms / 1e6 / peak:5.1f}% of copy")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
