"""Config 4 (BASELINE.json configs[3]): fp32 gradients and Adam optimizer state
(1 B elements each) to the 9-bit formats e5m3 and e4m4, encode + decode with
the per-tensor exponent histogram, one B200.  Per tensor and format: histogram
-> e_max -> encode (ROWS) and decode, CUDA events, back-to-back reps.
python tools/bench_config4.py [--n 1073741824] [--reps 5]"""
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

PEAK = 6555.5


def timeit(fn, reps):
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
    ap.add_argument("--n", type=int, default=1 << 30)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda")
    n = a.n
    C = 16384
    R = n // C
    tensors = {"gradients": W.f32_gradients(n, device=dev).view(R, C),
               "adam_m": W.f32_adam_m(n, device=dev).view(R, C),
               "adam_v": W.f32_adam_v(n, device=dev).view(R, C)}
    res = {"config": "config 4: fp32 gradients / Adam m / Adam v, %d elements each, (%d, %d) ROWS" % (n, R, C)}
    L, P = exmy.lib(), exmy._ptr
    for name, t in tensors.items():
        h = torch.zeros(256, dtype=torch.int64, device=dev)
        m = torch.zeros(1, dtype=torch.uint8, device=dev)
        for fmt in ("e5m3", "e4m4"):
            x, y = exmy.parse_format(fmt)
            k = 1 + x + y
            packed = torch.empty(n * k // 8, dtype=torch.uint8, device=dev)
            out = torch.empty_like(t)
            st = exmy._stream(dev)

            def enc():
                h.zero_()
                L.exmy_exponent_histogram(P(t), exmy.F32, n, P(h), st)
                L.exmy_emax_from_histogram(P(h), P(m), st)
                L.exmy_encode(P(t), exmy.F32, R, C, exmy.ROWS, x, y, P(m), P(packed), None, None, None, 0, st)

            def dec():
                L.exmy_decode(P(packed), R, C, exmy.ROWS, x, y, P(m), None, None, None, 0, P(out), exmy.F32, st)

            te, td = timeit(enc, a.reps), timeit(dec, a.reps)
            enc_bytes = n * 4 + n * 4 + n * k / 8          # histogram read + encode read + packed write
            dec_bytes = n * k / 8 + n * 4
            ref = exmy.quantize(t, fmt, m)
            exact = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
            res[f"{name}/{fmt}"] = {
                "encode_ms": round(te, 3), "encode_hbm_gbs": round(enc_bytes / te / 1e6, 1),
                "encode_frac": round(enc_bytes / te / 1e6 / PEAK, 3),
                "encode_input_gbs": round(2 * n * 4 / te / 1e6, 1),
                "decode_ms": round(td, 3), "decode_hbm_gbs": round(dec_bytes / td / 1e6, 1),
                "decode_frac": round(dec_bytes / td / 1e6 / PEAK, 3),
                "e_max": int(m.item()), "decode_equals_quantize": exact}
            print(f"{name:10s} {fmt}: hist+encode {te:7.3f} ms ({enc_bytes / te / 1e6:6.0f} GB/s, "
                  f"{enc_bytes / te / 1e6 / PEAK * 100:4.1f} %)  decode {td:7.3f} ms ({dec_bytes / td / 1e6:6.0f} GB/s, "
                  f"{dec_bytes / td / 1e6 / PEAK * 100:4.1f} %)  e_max {int(m.item())}  exact {exact}")
            del packed, out, ref
    print(json.dumps(res))


if __name__ == "__main__":
    main()
