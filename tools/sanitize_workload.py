"""Small ragged workload touching every kernel family once (for
compute-sanitizer memcheck / racecheck / synccheck / initcheck where it is
available: `compute-sanitizer --tool racecheck python tools/sanitize_workload.py`;
the round-1 GPU pool has the sanitizer closed, so out-of-bounds and race
safety rest on the bit-exact parity tests over ragged shapes instead)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402


def main():
    dev = torch.device("cuda")
    R, C = 64, 576        # ragged: 144 four-column tiles per row, not a multiple of 256
    for dt in (torch.bfloat16, torch.float32):
        t = W.f32_wide((R, C), seed=1).to(dt).to(dev)
        t.view(-1)[[5, 77]] = float("nan")
        for mode in (0, 1, 2, 3, 4):
            exmy.hist_mode(mode)
            exmy.histogram(t)
        exmy.hist_mode(4)
        m = exmy.max_exponent(t)
        for fmt in ("e3m3", "e6m0", "e4m3", "e3m5", "e8m0"):
            exmy.quantize(t, fmt, m)
            for axis in ("rows", "cols"):
                p = exmy.encode(t, fmt, m, axis=axis)
                exmy.decode(p)
                exmy.decode(p, torch.float32 if dt == torch.bfloat16 else torch.bfloat16)
            for blk in ("row", (1, 48), (8, 8)):
                meta = exmy.block_max_exponent(t, blk, 3, "after")
                exmy.quantize_blocked(t, fmt, meta, blk)
                for axis in ("rows", "cols"):
                    exmy.decode(exmy.encode_blocked(t, fmt, meta, blk, axis=axis))
            for blk in ("row", (1, 48), (1, 32), (1, 64)):
                exmy.quantize_fs(t, fmt, None, blk)
                exmy.decode(exmy.encode_fs(t, fmt, None, blk))
            exmy.decode(exmy.encode_rowwise(t, fmt))
            pc = exmy.encode(t, fmt, m, axis="cols")
            exmy.decode_rows(pc, torch.tensor([3, 0, 63, 3]))
            exmy.embedding_bag(pc, torch.tensor([3, 0, 63, 3, 9]), torch.tensor([0, 2, 2, 5]),
                               torch.rand(5), mode="mean")
            k = exmy.parse_format(fmt)
            nb = R * C * (1 + k[0] + k[1]) // 8
            bufs = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
            for r in range(2):
                exmy.encode_push(t[32 * r:32 * (r + 1)], fmt, m, 32 * r, R, bufs)
            shards = [exmy.encode(t[32 * r:32 * (r + 1)], fmt, m).data for r in range(2)]
            exmy.decode_pull(shards, 32, C, fmt, m, dtype=dt)
        g = exmy.GroupCodec([t, t[:8].clone(), torch.ones(64, dtype=dt, device=dev)], "e3m3", specials_capacity=16)
        g.encode()
        g.decode()
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
