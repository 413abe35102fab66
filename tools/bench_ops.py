"""Per-op timing (CUDA events, median of reps) for kernel tuning.
python tools/bench_ops.py [--dtype bf16|f32] [--fmts e3m3,e6m0] [--axis rows|cols] [--hist-modes 0,1]"""
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


def timeit(fn, reps=20, warm=3):
    """average device time per call over `reps` back-to-back calls (the
    launch queue stays ahead of the GPU, so host overhead is hidden)"""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--cols", type=int, default=16384)
    ap.add_argument("--fmts", default="e0m6,e1m5,e2m4,e3m3,e4m2,e5m1,e6m0")
    ap.add_argument("--axis", default="rows")
    ap.add_argument("--hist-modes", default="4")
    ap.add_argument("--probe", action="store_true", help="also time the roofline probe for each op's byte mix")
    ap.add_argument("--fs", action="store_true", help="with --block: also time the float-scaling scheme")
    ap.add_argument("--block", default=None, help="row | col | tensor | BRxBC: time the block-metadata path")
    a = ap.parse_args()
    dev = torch.device("cuda")
    R, C = a.rows, a.cols
    n = R * C
    if a.dtype == "bf16":
        t = W.bf16_weights((R, C), seed=1, device=dev)
        es = 2
    else:
        t = W.f32_gradients(n, device=dev).view(R, C)
        es = 4
    peak = 6555.5
    res = {}
    h = torch.zeros(256, dtype=torch.int64, device=dev)
    for m in [int(v) for v in a.hist_modes.split(",")]:
        exmy.hist_mode(m)
        ms = timeit(lambda: exmy.histogram(t, out=h))
        res[f"hist_mode{m}"] = {"ms": ms, "gbs": n * es / ms / 1e6, "frac": n * es / ms / 1e6 / peak}
    exmy.hist_mode(4)
    meta = exmy.max_exponent(t)
    q = torch.empty_like(t)
    d = torch.empty_like(t)
    for f in a.fmts.split(","):
        x, y = exmy.parse_format(f)
        k = 1 + x + y
        ms = timeit(lambda: exmy.quantize(t, f, meta, out=q))
        res[f"quantize_{f}"] = {"ms": ms, "gbs": 2 * n * es / ms / 1e6, "frac": 2 * n * es / ms / 1e6 / peak}
        buf = torch.empty(n * k // 8, dtype=torch.uint8, device=dev)
        ms = timeit(lambda: exmy.encode(t, f, meta, axis=a.axis, out=buf, strict=False))
        res[f"encode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6, "frac": n * (es + k / 8) / ms / 1e6 / peak}
        p = exmy.encode(t, f, meta, axis=a.axis, out=buf, strict=False)
        ms = timeit(lambda: exmy.decode(p, out=d))
        res[f"decode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6, "frac": n * (es + k / 8) / ms / 1e6 / peak}
    if a.block:
        blk = a.block if a.block in ("row", "col", "tensor") else tuple(int(v) for v in a.block.split("x"))
        br, bc = exmy.block_shape(t.shape, blk)
        for f in a.fmts.split(","):
            x, y = exmy.parse_format(f)
            k = 1 + x + y
            m = torch.empty((R // br, C // bc), dtype=torch.uint8, device=dev)
            ms = timeit(lambda: exmy.block_max_exponent(t, (br, bc), y, "before", out=m))
            res[f"blkmax_{f}"] = {"ms": ms, "gbs": n * es / ms / 1e6, "frac": n * es / ms / 1e6 / peak}
            ms = timeit(lambda: exmy.quantize_blocked(t, f, m, (br, bc), out=q))
            res[f"bquant_{f}"] = {"ms": ms, "gbs": 2 * n * es / ms / 1e6, "frac": 2 * n * es / ms / 1e6 / peak}
            buf = torch.empty(n * k // 8, dtype=torch.uint8, device=dev)
            ms = timeit(lambda: exmy.encode_blocked(t, f, m, (br, bc), axis=a.axis, out=buf, strict=False))
            res[f"bencode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6,
                                   "frac": n * (es + k / 8) / ms / 1e6 / peak}
            if (br, bc) == (1, C):
                ms = timeit(lambda: exmy.encode_rowwise(t, f, axis=a.axis, out=buf, meta_out=m, strict=False))
                res[f"rowwise_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6,
                                       "frac": n * (es + k / 8) / ms / 1e6 / peak}
            p = exmy.encode_blocked(t, f, m, (br, bc), axis=a.axis, out=buf, strict=False)
            ms = timeit(lambda: exmy.decode(p, out=d))
            res[f"bdecode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6,
                                   "frac": n * (es + k / 8) / ms / 1e6 / peak}
            if a.fs:   # float scaling (reading D23)
                sc = torch.empty((R // br, C // bc), dtype=torch.float32, device=dev)
                ms = timeit(lambda: exmy.block_float_scale(t, (br, bc), out=sc))
                res[f"fsmax_{f}"] = {"ms": ms, "gbs": n * es / ms / 1e6, "frac": n * es / ms / 1e6 / peak}
                ms = timeit(lambda: exmy.quantize_fs(t, f, sc, (br, bc), out=q))
                res[f"fsquant_{f}"] = {"ms": ms, "gbs": 2 * n * es / ms / 1e6, "frac": 2 * n * es / ms / 1e6 / peak}
                ms = timeit(lambda: exmy.encode_fs(t, f, sc, (br, bc), axis=a.axis, out=buf, strict=False))
                res[f"fsencode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6,
                                        "frac": n * (es + k / 8) / ms / 1e6 / peak}
                pf = exmy.encode_fs(t, f, sc, (br, bc), axis=a.axis, out=buf, strict=False)
                ms = timeit(lambda: exmy.decode(pf, out=d))
                res[f"fsdecode_{f}"] = {"ms": ms, "gbs": n * (es + k / 8) / ms / 1e6,
                                        "frac": n * (es + k / 8) / ms / 1e6 / peak}
    if a.probe:   # roofline probe: the same read:write bytes with no arithmetic
        src = t.reshape(-1).view(torch.uint8)
        mixes = {"hist": 0.0, "quantize": float(es)}
        for f in a.fmts.split(","):
            k = 1 + sum(exmy.parse_format(f))
            mixes[f"encode_{f}"] = k / 8
        for name, wpe in mixes.items():   # write bytes per element
            ob = int(n * wpe)
            o = torch.empty(max(ob, 16), dtype=torch.uint8, device=dev)
            ms = timeit(lambda: exmy.roofline_probe(src, ob, out=o))
            tot = n * es + ob
            res[f"probe_{name}"] = {"ms": ms, "gbs": tot / ms / 1e6, "frac": tot / ms / 1e6 / peak}
        for f in a.fmts.split(","):   # decode's mix: read k/8, write es (probe reads the packed bytes' size)
            k = 1 + sum(exmy.parse_format(f))
            pk = torch.empty(n * k // 8, dtype=torch.uint8, device=dev)
            o = torch.empty(n * es, dtype=torch.uint8, device=dev)
            ms = timeit(lambda: exmy.roofline_probe(pk, n * es, out=o))
            tot = n * k // 8 + n * es
            res[f"probe_decode_{f}"] = {"ms": ms, "gbs": tot / ms / 1e6, "frac": tot / ms / 1e6 / peak}
    for k_, v in res.items():
        print(f"{k_:16s} {v['ms']*1e3:9.1f} us {v['gbs']:8.1f} GB/s  {v['frac']*100:5.1f}%")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
