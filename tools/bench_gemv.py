"""Fused decode + GEMV (exmy_gemv) on config 2's weight (16384 x 16384 bf16,
encoded e3m3 / e2m2 / e4m3, per tensor and per row) for m = 1..16 activation
rows, against (a) cuBLAS bf16 GEMV on the uncompressed weight and (b) decode
to bf16 + cuBLAS.  CUDA events, L2 flushed between calls (the weight alone
exceeds L2 in bf16, not in packed form).  Usage: python tools/bench_gemv.py"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def timeit(fn, flush, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmts", default="e3m3,e2m2,e4m3")
    ap.add_argument("--ms", default="1,2,4,8,16")
    a = ap.parse_args()
    dev = torch.device("cuda")
    R = C = 16384
    t = W.bf16_weights((R, C), seed=1, device=dev)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: scratch.zero_()   # noqa: E731
    res = {}
    for m in [int(v) for v in a.ms.split(",")]:
        act = torch.randn(m, C, device=dev)
        actb = act.to(torch.bfloat16)
        ms = timeit(lambda: torch.matmul(actb, t.t()), flush)
        res[f"cublas_bf16_m{m}"] = {"us": ms * 1e3, "weight_gbs": R * C * 2 / ms / 1e6}
        print(f"cublas bf16      m={m:2d} {ms * 1e3:8.1f} us  {R * C * 2 / ms / 1e6:7.1f} GB/s of weight")
        for f in a.fmts.split(","):
            x, y = exmy.parse_format(f)
            k = 1 + x + y
            for per_row in (False, True):
                if per_row:
                    p = exmy.encode_rowwise(t, f, strict=False)
                else:
                    p = exmy.encode(t, f, exmy.emax(exmy.histogram(t)), strict=False)
                ms = timeit(lambda: exmy.gemv(p, act), flush)
                wb = R * C * k / 8
                tag = f"gemv_{f}_{'row' if per_row else 'tensor'}_m{m}"
                res[tag] = {"us": ms * 1e3, "packed_gbs": wb / ms / 1e6}
                print(f"gemv {f} {'row   ' if per_row else 'tensor'} m={m:2d} {ms * 1e3:8.1f} us  {wb / ms / 1e6:7.1f} GB/s of packed weight")
                if not per_row and f == "e3m3":
                    def two_step():
                        d = exmy.decode(p, torch.bfloat16)
                        return torch.matmul(actb, d.t())
                    ms2 = timeit(two_step, flush)
                    res[f"decode_then_cublas_{f}_m{m}"] = {"us": ms2 * 1e3}
                    print(f"decode+cublas {f} m={m:2d} {ms2 * 1e3:8.1f} us")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
