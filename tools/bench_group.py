"""Grouped launch vs per-tensor calls, kernel by kernel (CUDA events, back to
back reps).  python tools/bench_group.py [--shapes 16384x16384,4096x4096]
[--llama LAYERS] [--fmt e3m3]"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def timeit(fn, reps=10, warm=2):
    for _ in range(warm):
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
    ap.add_argument("--shapes", default="16384x16384")
    ap.add_argument("--llama", type=int, default=0, help="use the Llama-3-8B table with this many layers")
    ap.add_argument("--fmt", default="e3m3")
    a = ap.parse_args()
    dev = torch.device("cuda")
    if a.llama:
        shapes = [s for (nm, s) in W.llama3_8b_shapes()
                  if not nm.startswith("layers.") or int(nm.split(".")[1]) < a.llama]
    else:
        shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
    ts = [torch.ones(s, dtype=torch.bfloat16, device=dev) if len(s) == 1 else
          W.bf16_weights(s, seed=i, device=dev) for i, s in enumerate(shapes)]
    n = sum(t.numel() for t in ts)
    x, y = exmy.parse_format(a.fmt)
    k = 1 + x + y
    g = exmy.GroupCodec(ts, a.fmt)
    g.encode()
    L, P = exmy.lib(), exmy._ptr
    ph, pd = g._ph, P(g.plan_dev)
    per = []
    for t, lay in zip(ts, g.layouts):
        per.append((t, lay, torch.zeros(1, dtype=torch.uint8, device=dev),
                    torch.empty(t.numel() * k // 8, dtype=torch.uint8, device=dev), torch.empty_like(t)))

    def st():
        return exmy._stream(dev)

    def p_max():
        for t, lay, m, p, o in per:
            L.exmy_max_exponent(P(t), exmy.BF16, t.numel(), P(m), st())

    def p_enc():
        for t, (R, C), m, p, o in per:
            L.exmy_encode(P(t), exmy.BF16, R, C, exmy.ROWS, x, y, P(m), P(p), None, None, None, 0, st())

    def p_dec():
        for t, (R, C), m, p, o in per:
            L.exmy_decode(P(p), R, C, exmy.ROWS, x, y, P(m), None, None, None, 0, P(o), exmy.BF16, st())

    rows = [("max", n * 2, lambda: L.exmy_group_max_exponent(ph, pd, st()), p_max),
            ("encode", n * (2 + k / 8), lambda: L.exmy_group_encode(ph, pd, st()), p_enc),
            ("decode", n * (2 + k / 8), lambda: L.exmy_group_decode(ph, pd, st()), p_dec)]
    p_max()
    print(f"{len(ts)} tensors, {n / 1e9:.3f} G elements, {a.fmt}")
    for name, nb, fg, fp in rows:
        tg, tp = timeit(fg), timeit(fp)
        print(f"{name:8s} group {tg * 1e3:9.1f} us {nb / tg / 1e6:7.0f} GB/s   per-tensor {tp * 1e3:9.1f} us "
              f"{nb / tp / 1e6:7.0f} GB/s")


if __name__ == "__main__":
    main()
