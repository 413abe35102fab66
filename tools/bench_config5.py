"""Config 5 at full size on ONE B200 (BASELINE configs[4]):
a DLRM-style 100M x 128 fp32 embedding table (51.2 GB) ~ U(-1e-4, 1e-4),
COLS packing (row-addressable), e4m2 / e3m1:
  * whole-table max exponent, encode, decode (per-tensor metadata);
  * per-row metadata (the paper's recipe): row maxima, encode,
    decode through the narrow-row kernels;
  * row gathers of B = 2048 (captured as one CUDA graph of 100 gathers, so
    the per-call Python overhead is gone), 65536 and 2^20 random rows;
  * oracle parity of sampled row windows of every packed table.
Generated in place on the device (peak ~115 GB).  Prints one JSON line.
python tools/bench_config5.py [--rows 100000000]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_13938_b200 as exmy  # noqa: E402
import workloads as W  # noqa: E402

PEAK = 6546.6


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def table(rows, cols, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    t = torch.rand((rows, cols), generator=g, device=dev)
    return t.mul_(2.0).sub_(1.0).mul_(1e-4)     # == workloads.f32_embedding, in place


def check_windows(orc, t, p, fmt, meta, per_row, cols, windows):
    ok = True
    k = 1 + sum(exmy.parse_format(fmt))
    n = t.shape[0] * cols
    ws, offs = exmy.segments(k, n)
    for r0 in windows:
        bits = W.to_bits(t[r0:r0 + 64].cpu())
        got = torch.cat([p.data[o + r0 * cols * w // 8: o + (r0 + 64) * cols * w // 8] for w, o in zip(ws, offs)])
        if per_row:
            m = p.meta[r0:r0 + 64].cpu().numpy()
            ref = orc.encode_blocked(bits, fmt, m, (1, cols), orc.COLS)[0]
        else:
            ref = orc.encode(bits, fmt, int(meta), orc.COLS)[0]
        ok = ok and bool(np.array_equal(got.cpu().numpy(), ref))
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000_000)
    ap.add_argument("--cols", type=int, default=128)
    ap.add_argument("--fmts", default="e4m2,e3m1")
    a = ap.parse_args()
    import oracle as orc
    orc.lib()
    dev = torch.device("cuda")
    R, C = a.rows, a.cols
    n = R * C
    free, total = torch.cuda.mem_get_info()
    need = n * 4 * 2 + n * 9 // 8 + (2 << 30)
    if need > free:
        R = int(R * free / need * 0.9) // 1024 * 1024
        n = R * C
    t = table(R, C, dev)
    out = torch.empty_like(t)
    res = {"rows": R, "cols": C, "bytes_fp32": n * 4}
    windows = [0, R // 3 // 64 * 64, R - 64]
    meta = exmy.max_exponent(t)
    res["max_exponent_ms"] = timeit(lambda: exmy.max_exponent(t, out=meta))
    for fmt in a.fmts.split(","):
        k = 1 + sum(exmy.parse_format(fmt))
        pk = torch.empty(n * k // 8, dtype=torch.uint8, device=dev)
        r = {}
        ms = timeit(lambda: exmy.encode(t, fmt, meta, axis="cols", out=pk, strict=False))
        r["encode"] = {"ms": ms, "hbm_gbs": n * (4 + k / 8) / ms / 1e6, "frac": n * (4 + k / 8) / ms / 1e6 / PEAK}
        p = exmy.encode(t, fmt, meta, axis="cols", out=pk, strict=False)
        ms = timeit(lambda: exmy.decode(p, out=out))
        r["decode"] = {"ms": ms, "hbm_gbs": n * (4 + k / 8) / ms / 1e6, "frac": n * (4 + k / 8) / ms / 1e6 / PEAK}
        r["parity_windows_ok"] = check_windows(orc, t, p, fmt, int(meta.item()), False, C, windows)
        # per-row metadata (narrow-row kernels)
        rm = torch.empty((R, 1), dtype=torch.uint8, device=dev)
        ms = timeit(lambda: exmy.block_max_exponent(t, "row", 0, "before", out=rm))
        r["row_max"] = {"ms": ms, "hbm_gbs": n * 4 / ms / 1e6, "frac": n * 4 / ms / 1e6 / PEAK}
        ms = timeit(lambda: exmy.encode_blocked(t, fmt, rm, "row", axis="cols", out=pk, strict=False))
        r["encode_per_row"] = {"ms": ms, "hbm_gbs": n * (4 + k / 8) / ms / 1e6,
                               "frac": n * (4 + k / 8) / ms / 1e6 / PEAK}
        pr = exmy.encode_blocked(t, fmt, rm, "row", axis="cols", out=pk, strict=False)
        ms = timeit(lambda: exmy.decode(pr, out=out))
        r["decode_per_row"] = {"ms": ms, "hbm_gbs": n * (4 + k / 8) / ms / 1e6,
                               "frac": n * (4 + k / 8) / ms / 1e6 / PEAK}
        r["parity_windows_per_row_ok"] = check_windows(orc, t, pr, fmt, 0, True, C, windows)
        # row gathers (the serving access pattern), per-tensor metadata
        p = exmy.encode(t, fmt, meta, axis="cols", out=pk, strict=False)
        gen = torch.Generator(device=dev)
        gen.manual_seed(0)
        gat = {}
        for B in (2048, 65536, 1 << 20):
            idx = torch.randint(0, R, (B,), device=dev, generator=gen)
            o = torch.empty((B, C), dtype=torch.float32, device=dev)
            exmy.decode_rows(p, idx, out=o, check=True)          # validated once
            if B == 2048:   # 100 gathers in one CUDA graph: no per-call host overhead
                graph = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    exmy.decode_rows(p, idx, out=o, check=False)
                    with torch.cuda.graph(graph, stream=s):
                        for _ in range(100):
                            exmy.decode_rows(p, idx, out=o, check=False)
                torch.cuda.current_stream().wait_stream(s)
                ms = timeit(lambda: graph.replay()) / 100
                how = "CUDA graph of 100 gathers"
            else:
                ms = timeit(lambda: exmy.decode_rows(p, idx, out=o, check=False))
                how = "one call"
            alg = B * (C * k // 8 + C * 4 + 8)
            gat[B] = {"us": ms * 1e3, "mrows_per_s": B / ms / 1e3, "hbm_gbs": alg / ms / 1e6, "how": how}
        r["gather"] = gat
        res[fmt] = r
        del pk, p, pr
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
