"""A/B of the ROWS encode kernels (exmy_debug_enc_tma: TMA-staged ring vs
register pipeline) on the config-2 tensor (16384^2 bf16) and a fp32 tensor,
CUDA events, interleaved; asserts identical bytes.
Usage: python tools/enc_ab.py [--fmts e3m3,e6m0,e4m3,e3m5] [--reps 20]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmts", default="e3m3,e6m0,e4m3,e3m5,e0m6")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--f32", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    t = W.bf16_weights((16384, 16384), seed=1, device=dev)
    cases = [("bf16", t)]
    if a.f32:
        cases.append(("f32", W.f32_gradients(1 << 28, device=dev).view(16384, 16384)))
    for name, x in cases:
        n = x.numel()
        meta = exmy.max_exponent(x)
        for f in a.fmts.split(","):
            k = 1 + sum(exmy.parse_format(f))
            out = {m: torch.empty(n * k // 8, dtype=torch.uint8, device=dev) for m in (0, 1)}
            times = {0: [], 1: []}
            for r in range(a.reps + 3):
                for m in (0, 1):
                    exmy.enc_tma(m)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    exmy.encode(x, f, meta, out=out[m], strict=False)
                    e.record()
                    torch.cuda.synchronize()
                    if r >= 3:
                        times[m].append(s.elapsed_time(e) * 1e3)
            assert torch.equal(out[0], out[1]), (name, f)
            alg = n * x.element_size() + n * k // 8
            line = [f"{name} {f}:"]
            for m in (0, 1):
                v = sorted(times[m])
                med = v[len(v) // 2]
                line.append(f"{'tma' if m else 'reg'} {med:.1f} us ({alg / med / 1e3:.0f} GB/s)")
            print("  ".join(line), flush=True)
    exmy.enc_tma(0)


if __name__ == "__main__":
    main()
