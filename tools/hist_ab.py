"""A/B of the histogram kernels (exmy_debug_hist_mode) on the config-2 tensor
(16384^2 bf16 ~N(0, 0.02^2)) and on a wide-exponent tensor, CUDA events,
interleaved repetitions.  Usage: python tools/hist_ab.py [--modes 2,3] [--reps 20]"""
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
    ap.add_argument("--modes", default="3,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    modes = [int(m) for m in a.modes.split(",")]
    dev = torch.device("cuda")
    tensors = {"config2": W.bf16_weights((16384, 16384), seed=1, device=dev)}
    if not a.only:
        tensors["wide"] = W.bf16_weights((16384, 16384), seed=2, device=dev) * torch.exp2(
            torch.randint(-20, 20, (16384, 1), device=dev).float()).to(torch.bfloat16)
    h = torch.zeros(256, dtype=torch.int64, device=dev)
    n = 16384 * 16384
    for name, t in tensors.items():
        ref = None
        times = {m: [] for m in modes}
        for r in range(a.reps + 3):
            for m in modes:
                exmy.hist_mode(m)
                h.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                exmy.histogram(t, out=h)
                e.record()
                torch.cuda.synchronize()
                if r >= 3:
                    times[m].append(s.elapsed_time(e) * 1e3)
                if ref is None:
                    ref = h.clone()
                assert torch.equal(h, ref), (name, m)
        for m in modes:
            v = sorted(times[m])
            med = v[len(v) // 2]
            print(f"{name} mode {m}: median {med:.1f} us  min {v[0]:.1f}  ({2 * n / med / 1e3:.0f} GB/s)")
    exmy.hist_mode(4)


if __name__ == "__main__":
    main()
