"""Run each codec op on the config-2 tensor (16384^2 bf16) a few times, for
ncu captures.  Usage: python tools/prof_ops.py [--fmt e3m3] [--axis rows] [--reps 3]"""
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
    ap.add_argument("--fmt", default="e3m3")
    ap.add_argument("--axis", default="rows")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--cols", type=int, default=16384)
    a = ap.parse_args()
    dev = torch.device("cuda")
    if a.dtype == "bf16":
        t = W.bf16_weights((a.rows, a.cols), seed=1, device=dev)
    else:
        t = W.f32_gradients(a.rows * a.cols, device=dev).view(a.rows, a.cols)
    for _ in range(a.reps):
        h = exmy.histogram(t)
        m = exmy.emax(h)
        q = exmy.quantize(t, a.fmt, m)
        p = exmy.encode(t, a.fmt, m, axis=a.axis)
        d = exmy.decode(p)
    torch.cuda.synchronize()
    assert torch.equal(d.view(torch.int16) if a.dtype == "bf16" else d.view(torch.int32),
                       q.view(torch.int16) if a.dtype == "bf16" else q.view(torch.int32))
    print("ok", int(m.item()))


if __name__ == "__main__":
    main()
