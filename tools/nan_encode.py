"""Encode a clean and an all-NaN/Inf 16384^2 bf16 tensor (e3m3, ROWS, specials
capacity 4096) a few times -- for ncu launch lists of the NaN-heavy path
(main kernel, fix-up pass, ordered-list compaction).  Prints CUDA-event ms."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def main():
    dev = torch.device("cuda")
    clean = W.bf16_weights((16384, 16384), seed=1, device=dev)
    nan = torch.full_like(clean, float("nan"))
    nan.view(-1)[1::7] = float("-inf")
    meta = exmy.max_exponent(clean)
    for name, t in (("clean", clean), ("nan", nan)):
        for _ in range(2):
            exmy.encode(t, "e3m3", meta, specials_capacity=4096, strict=False)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            exmy.encode(t, "e3m3", meta, specials_capacity=4096, strict=False)
        b.record()
        torch.cuda.synchronize()
        print(name, round(a.elapsed_time(b) / 5, 4), "ms per encode")


if __name__ == "__main__":
    main()
