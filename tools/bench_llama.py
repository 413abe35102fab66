"""Config 3 at one GPU: Llama-3-8B-shaped bf16 weights (291 tensors, 8.03 G
params, N(0,0.02^2), norms = 1), per-tensor metadata from the histogram,
ROWS packing to e2m2 / e3m3 / e2m4.  Times the whole model: histogram ->
e_max -> encode per tensor, then decode, with eager launches and with the
same launches captured in a CUDA graph; and the grouped launch
(GroupCodec: max exponent + encode of all tensors in 3 launches, decode in 1).
python tools/bench_llama.py [--fmt e3m3] [--layers 32]"""
import argparse
import json
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
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="", help="comma list of timings to run (default: all)")
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    shapes = [s for s in W.llama3_8b_shapes() if not s[0].startswith("layers.") or
              int(s[0].split(".")[1]) < a.layers]
    x, y = exmy.parse_format(a.fmt)
    k = 1 + x + y
    L = exmy.lib()
    P = exmy._ptr
    tensors, hists, metas, packed, outs = [], [], [], [], []
    for i, (name, shp) in enumerate(shapes):
        if len(shp) == 1:
            t = torch.ones(shp, dtype=torch.bfloat16, device=dev)
            shp2 = (1, shp[0])
        else:
            t = W.bf16_weights(shp, seed=1000 + i, device=dev)
            shp2 = shp
        tensors.append((t, shp2))
        hists.append(torch.zeros(256, dtype=torch.int64, device=dev))
        metas.append(torch.zeros(1, dtype=torch.uint8, device=dev))
        n = shp2[0] * shp2[1]
        packed.append(torch.empty(n * k // 8, dtype=torch.uint8, device=dev))
        outs.append(torch.empty_like(t))
    nparams = sum(t.numel() for t, _ in tensors)

    def encode_all():
        sp = exmy._stream(dev)   # the current stream (the capture stream inside a graph)
        for (t, (R, C)), h, m, p in zip(tensors, hists, metas, packed):
            h.zero_()
            L.exmy_exponent_histogram(P(t), exmy.BF16, R * C, P(h), sp)
            L.exmy_emax_from_histogram(P(h), P(m), sp)
            ax = exmy.ROWS if R % 8 == 0 else exmy.COLS
            L.exmy_encode(P(t), exmy.BF16, R, C, ax, x, y, P(m), P(p), None, None, None, 0, sp)

    def encode_all_max():   # metadata by the read-only max reduction instead of the histogram
        sp = exmy._stream(dev)
        for (t, (R, C)), m, p in zip(tensors, metas, packed):
            L.exmy_max_exponent(P(t), exmy.BF16, R * C, P(m), sp)
            ax = exmy.ROWS if R % 8 == 0 else exmy.COLS
            L.exmy_encode(P(t), exmy.BF16, R, C, ax, x, y, P(m), P(p), None, None, None, 0, sp)

    def decode_all():
        sp = exmy._stream(dev)
        for (t, (R, C)), m, p, o in zip(tensors, metas, packed, outs):
            ax = exmy.ROWS if R % 8 == 0 else exmy.COLS
            L.exmy_decode(P(p), R, C, ax, x, y, P(m), None, None, None, 0, P(o), exmy.BF16, sp)

    def time(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / a.reps

    grp = exmy.GroupCodec([t for t, _ in tensors], (x, y))

    # the paper's quality recipe: one metadata byte per row; 1-D norms as one row
    row_metas = [torch.zeros((R, 1), dtype=torch.uint8, device=dev) for (_, (R, C)) in tensors]

    def encode_all_rowwise():   # per-row max exponent + encode (fused kernel for rows <= 16 KB)
        sp = exmy._stream(dev)
        for (t, (R, C)), rm, p in zip(tensors, row_metas, packed):
            ax = exmy.ROWS if R % 8 == 0 else exmy.COLS
            L.exmy_encode_rowwise(P(t), exmy.BF16, R, C, ax, x, y, 0, P(rm), P(p), None, None, None, 0, sp)

    def decode_all_rowwise():
        sp = exmy._stream(dev)
        for (t, (R, C)), rm, p, o in zip(tensors, row_metas, packed, outs):
            ax = exmy.ROWS if R % 8 == 0 else exmy.COLS
            L.exmy_decode_blocked(P(p), R, C, ax, 1, C, x, y, P(rm), None, None, None, 0, P(o), exmy.BF16, sp)

    def group_encode():   # grouped launch: meta (2 launches) + encode (1)
        grp.encode()

    def group_decode():
        grp.decode()

    grp_rows = exmy.GroupCodec([t for t, _ in tensors], (x, y), per_row=True)   # per-row recipe, grouped

    def group_rows_encode():   # row bytes (1 launch) + encode (1)
        grp_rows.encode()

    def group_rows_decode():
        grp_rows.decode()

    res = {"tensors": len(tensors), "params": nparams, "fmt": a.fmt}
    nl = {"encode": 3 * len(tensors), "encode_maxexp": 2 * len(tensors), "decode": len(tensors),
          "encode_rowwise": len(tensors), "decode_rowwise": len(tensors),
          "group_encode": 3, "group_decode": 1, "group_rows_encode": 2, "group_rows_decode": 1}
    for name, fn in (("encode", encode_all), ("encode_maxexp", encode_all_max), ("decode", decode_all),
                     ("encode_rowwise", encode_all_rowwise), ("decode_rowwise", decode_all_rowwise),
                     ("group_encode", group_encode), ("group_decode", group_decode),
                     ("group_rows_encode", group_rows_encode), ("group_rows_decode", group_rows_decode)):
        if a.only and name not in a.only.split(","):
            continue
        ms = time(fn)
        if a.no_graph:
            print(f"{name}: eager {ms:.3f} ms")
            continue
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            fn()
        torch.cuda.current_stream().wait_stream(st)
        with torch.cuda.graph(g):
            fn()
        ms_g = time(g.replay)
        alg = nparams * ((2 + 2 + k / 8) if "encode" in name else (k / 8 + 2))
        res[name] = {"eager_ms": ms, "graph_ms": ms_g, "eager_hbm_gbs": alg / ms / 1e6,
                     "graph_hbm_gbs": alg / ms_g / 1e6,
                     "launches": nl[name]}
        print(f"{name}: eager {ms:.3f} ms ({alg / ms / 1e6:.0f} GB/s)  graph {ms_g:.3f} ms ({alg / ms_g / 1e6:.0f} GB/s)")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
