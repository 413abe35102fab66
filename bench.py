#!/usr/bin/env python
"""bench.py -- eXmY codec throughput on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1], "config 2"): a 16384 x 16384 bf16 tensor
~ N(0, 0.02^2) (LLM-weight-like, seed 1), packed along rows, through every
7-bit format e0m6 .. e6m0.  One STEP is one pass of the whole hot path
(SURVEY 8(a)):  exponent histogram (A1) -> e_max (A2) -> for each of the 7
formats: quantize (A3), encode (A4+A5), decode (A6+A7); at N > 1 also the
histogram all-reduce and the all-gather of packed shards (A8).

value = input GB/s of the step: sum over the codec calls of the bytes of each
call's input buffer (histogram 2n, quantize 2n, encode 2n, decode n*k/8 per
format), divided by the device time of the step; at N>1 summed over ranks
over the max rank time.

N > 1 (one process per GPU, NCCL, call stack 4): every rank owns
one 16384^2 shard (weak scaling of the encode side), histograms it, the
histograms are all-reduced into the global e_max, and per format the rank
quantizes and encodes its shard, all-gathers the packed shards (the
compressed exchange, P:298 / P:536) and decodes every received shard, each
one independently -- so each rank's decode input grows with N.
`python bench.py --gpus N` without a launcher re-executes itself under
torch.distributed.run; the driver's own torchrun launch is used as is.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "encode/decode input-GB/s per B200 and at 8 GPUs; % of HBM roofline"
R = C = 16384
FORMATS = [(x, 6 - x) for x in range(0, 7)]           # e0m6 .. e6m0 (k = 7)
K_BITS = 7
SEED = 1
FALLBACK_HBM_GBS = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------ clock sampling
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting", 0x10: "sync_boost"}


class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons through NVML every
    ~2 ms in a background thread while the timed region runs (nvidia-smi's
    own polling cannot start fast enough for a tens-of-ms region); falls back
    to `nvidia-smi -lms 100` if NVML is unavailable."""

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.samples = []
        self.stop = threading.Event()
        self.thread = None
        self.proc = None
        self.src = "nvml"

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self.stop.is_set():
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.samples.append((sm, self.max_mhz, rs))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            time.sleep(0.01)
        except Exception:
            self.src = "nvidia-smi"
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.thread = threading.Thread(target=self._read_smi, daemon=True)
                self.thread.start()
            except Exception:
                self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "source": self.src}
        sm = [s[0] for s in self.samples]
        reasons = set()
        for s in self.samples:
            for bit, name in REASON_BITS.items():
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_min_mhz": min(sm), "reasons": sorted(reasons), "samples": len(sm), "source": self.src}


# ------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, local, backend="nccl"):
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
        return dist
    return None


def device_index(local):
    """One process per GPU.  (--dist-backend gloo exists only to smoke-test the
    N>1 host logic on a 1-GPU box; ranks then share the device, and their
    collectives run on the CPU, so no kernel waits on another rank.)"""
    n = torch.cuda.device_count()
    return local % n if n else local


def self_launch(args) -> int:
    """`bench.py --gpus N` run directly: re-execute under torch.distributed.run
    with N ranks (127.0.0.1 rendezvous).  NCCL needs N visible GPUs."""
    n_dev = torch.cuda.device_count()
    if args.dist_backend == "nccl" and n_dev < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {n_dev} CUDA device(s) visible "
                         "(one process per GPU; --dist-backend gloo shares one GPU for a host-logic smoke run)")
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # rank / channel / NVLS lines for the driver's logs
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------- our arm
def run_ours(args):
    import paper_2405_13938_b200 as exmy
    from paper_2405_13938_b200 import dist as xdist
    import workloads as W

    ws, rank, local = dist_env()
    di = device_index(local)
    torch.cuda.set_device(di)
    dev = torch.device("cuda", di)
    dist = init_dist(ws, di, args.dist_backend)
    group = None

    n = R * C
    t = W.bf16_weights((R, C), seed=SEED + rank, device=dev)            # weak scaling: one shard per rank
    hist = torch.zeros(256, dtype=torch.int64, device=dev)
    meta = torch.zeros(1, dtype=torch.uint8, device=dev)
    packed = [torch.empty(n * K_BITS // 8, dtype=torch.uint8, device=dev) for _ in FORMATS]
    qout = torch.empty_like(t)
    dout = torch.empty_like(t)
    cap = 4096
    spi = torch.empty(cap, dtype=torch.int64, device=dev)
    spb = torch.empty(cap, dtype=torch.int32, device=dev)
    spc = exmy.specials_workspace(dev)
    packed_b = n * K_BITS // 8
    gathered = torch.empty(ws * packed_b, dtype=torch.uint8, device=dev) if ws > 1 else None
    # at N > 1 every received shard is decoded (into its rows of the full tensor)
    dout_all = torch.empty((ws * R, C), dtype=torch.bfloat16, device=dev) if ws > 1 else None
    L = exmy.lib()
    st = torch.cuda.current_stream(dev)
    sp = exmy._stream(dev)
    P = exmy._ptr
    ops = ["hist", "emax", "allreduce", "quantize", "encode", "allgather", "decode"]
    ev = {o: [] for o in ops}

    def rec(name, fn):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev[name].append((a, b))

    def chk(s):
        if s != 0:
            raise exmy.ExmyError(s, "bench")

    def step(timed):
        hist.zero_()
        f = rec if timed else (lambda name, fn: fn())
        f("hist", lambda: chk(L.exmy_exponent_histogram(P(t), exmy.BF16, n, P(hist), sp)))
        if ws > 1:
            f("allreduce", lambda: xdist.allreduce_histogram(hist, group))
        f("emax", lambda: chk(L.exmy_emax_from_histogram(P(hist), P(meta), sp)))
        for i, (x, y) in enumerate(FORMATS):
            f("quantize", lambda: chk(L.exmy_quantize(P(t), P(qout), exmy.BF16, n, x, y, P(meta), sp)))
            f("encode", lambda: chk(L.exmy_encode(P(t), exmy.BF16, R, C, exmy.ROWS, x, y, P(meta), P(packed[i]),
                                                  P(spi), P(spb), P(spc), cap, sp)))
            if ws > 1:
                f("allgather", lambda: xdist.allgather_bytes(packed[i], gathered, group))

                def dec_all():
                    for r in range(ws):      # shards decode independently; no specials in the data
                        chk(L.exmy_decode(ctypes.c_void_p(gathered.data_ptr() + r * packed_b), R, C, exmy.ROWS, x,
                                          y, P(meta), None, None, None, 0,
                                          ctypes.c_void_p(dout_all.data_ptr() + r * n * 2), exmy.BF16, sp))
                f("decode", dec_all)
            else:
                f("decode", lambda: chk(L.exmy_decode(P(packed[i]), R, C, exmy.ROWS, x, y, P(meta), P(spi), P(spb),
                                                      P(spc), cap, P(dout), exmy.BF16, sp)))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(dev)
    for k in ev:
        ev[k].clear()

    with ClockSampler(di) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.steps):
            step(True)
        t1.record(st)
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
    ms_total = t0.elapsed_time(t1)
    if dist:
        tt = torch.tensor([ms_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    per_op_ms = {k: sum(a.elapsed_time(b) for a, b in v) / args.steps for k, v in ev.items() if v}
    launches = {k: len(v) / args.steps for k, v in ev.items() if v}

    # bytes per step (one rank); at N > 1 the rank decodes all ws received shards
    nf = len(FORMATS)
    in_bytes = {"hist": 2 * n, "quantize": nf * 2 * n, "encode": nf * 2 * n, "decode": nf * ws * packed_b}
    alg_bytes = {"hist": 2 * n, "emax": 2048, "quantize": nf * 4 * n, "encode": nf * (2 * n + packed_b),
                 "decode": nf * ws * (packed_b + 2 * n)}
    step_in = sum(in_bytes.values())
    value = ws * step_in / (ms_step * 1e-3) / 1e9

    peak, peak_src = peaks()
    per_op = {}
    for k in ("hist", "quantize", "encode", "decode"):
        ms = per_op_ms[k]
        nl = launches[k]
        per_op[k] = {"ms_per_launch": ms / nl, "input_gbs": in_bytes[k] / (ms * 1e-3) / 1e9,
                     "hbm_gbs": alg_bytes[k] / (ms * 1e-3) / 1e9,
                     "frac_of_measured": alg_bytes[k] / (ms * 1e-3) / 1e9 / peak,
                     "frac_of_8tbs": alg_bytes[k] / (ms * 1e-3) / 1e9 / 8000.0}
        # per-launch distribution over the timed steps (median, p10 / p90)
        us = sorted(1e3 * a.elapsed_time(b) for a, b in ev[k])
        pct = lambda q: us[min(len(us) - 1, int(round(q * (len(us) - 1))))]
        per_op[k]["launch_us"] = {"p10": round(pct(0.1), 2), "median": round(pct(0.5), 2),
                                  "p90": round(pct(0.9), 2), "n": len(us)}
    dom = max(("quantize", "encode", "decode", "hist"), key=lambda k: per_op_ms[k])
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None
    achieved = per_op[dom]["hbm_gbs"]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "algorithmic_bytes_per_launch": alg_bytes[dom] / launches[dom], "peak_source": peak_src}

    # gpu launches of OUR kernels per step: hist 1, emax 1; per format quantize 1,
    # encode 3 (encode, NaN/Inf fix-up pass, ordered-list compaction; the last two
    # return at once on this data), decode 2 (decode + specials scatter) or, at N > 1,
    # one decode per received shard
    gpu_launches = args.steps * (2 + nf * (4 + (2 if ws == 1 else ws)))

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "config2: 16384x16384 bf16 ~N(0,0.02^2) seed 1 (+rank), ROWS packing, "
                               "7-bit formats e0m6..e6m0; step = histogram, e_max, 7x(quantize, encode, decode)"
                               + (", + hist all-reduce and packed all-gather (NCCL)" if ws > 1 else ""),
                   "elements_per_gpu": n, "formats": [f"e{x}m{y}" for x, y in FORMATS], "axis": "rows",
                   "l2": "inputs (512 MiB) larger than L2 (126 MB); no flush needed",
                   "parallelism": f"shard-per-rank x{ws}, all-gather of packed shards + decode of all {ws}"
                                  if ws > 1 else "single GPU",
                   "value_definition": "sum of codec-call input bytes per step / device step time"},
        # the metric's own per-codec numbers (input bytes of the call / its device time)
        "encode_input_gbs": round(per_op["encode"]["input_gbs"], 1),
        "decode_input_gbs": round(per_op["decode"]["input_gbs"], 1),
        "per_op": per_op, "per_op_ms_per_step": {k: round(v, 4) for k, v in per_op_ms.items()},
        "roofline": roofline, "gpu_launches": gpu_launches,
    }
    result["clocks"] = clk.summary()
    if ws > 1:
        result["multi_gpu"] = multi_gpu_report(dist, dev, t, packed[0], gathered, ev, per_op_ms, ms_total, args, ws,
                                               rank, nf, packed_b)

    # ---------------- block metadata: per-row e_max, e3m3,
    # same tensor; timed separately (not part of `value`)
    if not args.no_blocked:
        result["per_row_metadata"] = bench_blocked(exmy, t, args, peak, st)

    # ---------------- e2e through the C ABI with host buffers (rank-local).
    # Formats alternate between two streams, so one format's device->host
    # copies overlap the next format's host->device copies (PCIe is full
    # duplex; each stream keeps its own pinned buffers and device scratch).
    e2e_steps = max(1, min(args.steps, 3))
    hc = {}
    t_host = t.cpu().pin_memory()
    NS = int(os.environ.get("EXMY_E2E_STREAMS", "2"))
    host_packed = [torch.empty(packed_b, dtype=torch.uint8).pin_memory() for _ in range(NS)]
    host_meta = [torch.empty(1, dtype=torch.uint8).pin_memory() for _ in range(NS)]
    host_out = [torch.empty_like(t_host).pin_memory() for _ in range(NS)]
    e2e_streams = [torch.cuda.Stream(dev) for _ in range(NS)]
    for x, y in FORMATS:
        hc[(x, y)] = exmy.HostCodec((R, C), torch.bfloat16, (x, y), device=dev, specials_capacity=cap)
    parity = parity_of_timed_outputs(exmy, t, packed, qout, dout if ws == 1 else dout_all[rank * R:(rank + 1) * R],
                                     packed_b) if rank == 0 else None
    del qout, packed
    torch.cuda.empty_cache()

    def e2e_step():
        go = torch.cuda.Event()
        go.record(st)
        for s in e2e_streams:
            s.wait_event(go)
        for i, (x, y) in enumerate(FORMATS):
            j = i % NS
            with torch.cuda.stream(e2e_streams[j]):
                c = hc[(x, y)]
                c.encode(t_host, host_packed[j], host_meta[j])
                c.decode(host_packed[j], host_out[j])
        for s in e2e_streams:
            st.wait_stream(s)

    e2e_step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    b.record(st)
    torch.cuda.synchronize(dev)
    _ = float(host_out[(nf - 1) % NS][0, 0])   # the step's result, read on the host
    e2e_ms = a.elapsed_time(b) / e2e_steps
    if dist:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_in = nf * (2 * n + packed_b)     # per format: the encode call's host input, the decode call's host input
    result["e2e"] = {"value": round(ws * e2e_in / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                     "h2d_bytes_per_step": nf * (2 * n + packed_b), "d2h_bytes_per_step": nf * (packed_b + 1 + 2 * n),
                     "ms_per_step": round(e2e_ms, 3), "steps": e2e_steps,
                     "path": "exmy_encode_host (H2D, histogram, e_max, encode, D2H) + exmy_decode_host (H2D, decode, "
                             "D2H) per format, pinned host buffers, formats alternating over 2 streams (H2D and D2H "
                             "copies overlap); value = the two calls' host input bytes / time"}

    if rank == 0:
        result["parity"] = parity
        result["config1_latency_us"] = config1_latency(exmy, dev)
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(t[:args.cpu_rows].cpu())
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def parity_of_timed_outputs(exmy, t, packed, qout, dout, packed_b, windows=(0, 6144, 12000, 16376)):
    """parity checked on the timed outputs.  After the timed
    steps every format's packed buffer, and the last format's quantize and
    decode outputs, are still in device memory: 8-row windows of them (a row
    shard's bytes are, per segment, one contiguous range) are
    compared bit for bit with the CPU oracle run on the same rows."""
    import numpy as np
    import oracle as orc
    import workloads as W
    orc.lib()
    n = R * C
    e = int(exmy.max_exponent(t).item())
    ok = True
    checked = 0
    for r0 in windows:
        rows = W.to_bits(t[r0:r0 + 8])
        for i, (x, y) in enumerate(FORMATS):
            k = 1 + x + y
            ws, offs = exmy.segments(k, n)
            got = torch.cat([packed[i][o + r0 * C * w // 8: o + (r0 + 8) * C * w // 8] for w, o in zip(ws, offs)])
            ref = orc.encode(rows, (x, y), e, orc.ROWS)[0]
            ok = ok and bool(np.array_equal(got.cpu().numpy(), ref))
            checked += ref.size
        x, y = FORMATS[-1]
        q = orc.quantize(rows, (x, y), e)
        ok = ok and bool(np.array_equal(W.to_bits(qout[r0:r0 + 8]), q))
        ok = ok and bool(np.array_equal(W.to_bits(dout[r0:r0 + 8]), q))
    return {"ok": ok, "e_max": e, "windows": [f"rows {r}..{r + 7}" for r in windows],
            "packed_bytes_compared": checked,
            "what": "every format's packed bytes of 8-row windows (row-shard byte ranges) and the last format's "
                    "quantize / decode rows, vs the CPU oracle on the same rows"}


def config1_latency(exmy, dev, reps: int = 30):
    """BASELINE configs[0] ("config 1"): a 65,536-element fp32 tensor (256 x
    256), e3m2 -- L2-resident and launch-bound, so per-call latency (median
    us of CUDA events around one call, L2 flushed by a 256 MB write between
    calls) through the Python binding, histogram -> e_max -> quantize ->
    encode -> decode."""
    import workloads as W
    t = W.f32_wide((256, 256), seed=0).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hist = torch.zeros(256, dtype=torch.int64, device=dev)
    meta = exmy.emax(exmy.histogram(t))
    q = torch.empty_like(t)
    d = torch.empty_like(t)
    pk = torch.empty(65536 * 6 // 8, dtype=torch.uint8, device=dev)
    p = exmy.encode(t, "e3m2", meta, out=pk, strict=False)
    ops = {"histogram": lambda: exmy.histogram(t, out=hist), "emax": lambda: exmy.emax(hist, out=meta),
           "quantize": lambda: exmy.quantize(t, "e3m2", meta, out=q),
           "encode": lambda: exmy.encode(t, "e3m2", meta, out=pk, strict=False),
           "decode": lambda: exmy.decode(p, out=d)}
    res = {}
    for name, fn in ops.items():
        ts = []
        for i in range(reps + 3):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        res[name] = round(ts[len(ts) // 2], 2)
    res["workload"] = "config1: 256x256 fp32 N(0,1)*2^U{-12..12}, e3m2, per-call median, L2 flushed between calls"
    return res


def multi_gpu_report(dist, dev, t, pk, gathered, ev, per_op_ms, ms_total, args, ws, rank, nf, packed_b):
    """Per-rank step times, the all-gather's algbw / busbw (NCCL convention:
    busbw = algbw (G-1)/G), the same all-gather of the bf16 shard (the wire
    the codec saves: 16/k), and how many distinct GPUs the ranks ran on."""
    import torch.distributed as tdist
    mine = torch.tensor([ms_total / args.steps], dtype=torch.float64, device=dev)
    times = [torch.zeros_like(mine) for _ in range(ws)]
    tdist.all_gather(times, mine)
    ag_ms = per_op_ms.get("allgather", 0.0) / nf           # per all-gather (one per format)
    # the uncompressed exchange for comparison: all-gather of the bf16 shard
    full = torch.empty(ws * t.numel(), dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream(dev)
    for _ in range(2):
        tdist.all_gather_into_tensor(full, t.reshape(-1)) if args.dist_backend == "nccl" else None
    reps = max(3, min(args.steps, 10))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    tdist.barrier()
    a.record(st)
    for _ in range(reps):
        if args.dist_backend == "nccl":
            tdist.all_gather_into_tensor(full, t.reshape(-1))
        else:
            parts = [torch.empty_like(t.reshape(-1), device="cpu") for _ in range(ws)]
            tdist.all_gather(parts, t.reshape(-1).cpu())
    b.record(st)
    torch.cuda.synchronize(dev)
    bf_ms = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
    tdist.all_reduce(bf_ms, op=tdist.ReduceOp.MAX)
    bf_ms = float(bf_ms.item())
    del full
    # distinct physical GPUs behind the ranks
    try:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        uuid = f"cuda:{dev.index}"
    uuids = [None] * ws
    tdist.all_gather_object(uuids, uuid)
    ag_bytes = ws * packed_b
    bf_bytes = ws * t.numel() * 2

    def bw(nbytes, ms):
        alg = nbytes / (ms * 1e-3) / 1e9 if ms > 0 else None
        return {"ms": round(ms, 4), "bytes": nbytes, "algbw_gbs": round(alg, 1) if alg else None,
                "busbw_gbs": round(alg * (ws - 1) / ws, 1) if alg else None}
    return {"ranks": ws, "gpus_active": len(set(uuids)), "backend": args.dist_backend,
            "rank_ms_per_step": [round(float(x.item()), 4) for x in times],
            "allgather_packed": bw(ag_bytes, ag_ms), "allgather_bf16": bw(bf_bytes, bf_ms),
            "wire_ratio_bf16_over_packed": round(bf_bytes / ag_bytes, 4),
            "time_ratio_bf16_over_packed": round(bf_ms / ag_ms, 3) if ag_ms > 0 else None}


def bench_blocked(exmy, t, args, peak, st):
    """Per-row metadata (the paper's quality recipe) on the bench
    tensor: block max exponent, quantize, encode, decode (ROWS), e3m3."""
    R_, C_ = t.shape
    n = R_ * C_
    x, y = 3, 3
    k = 7
    meta = torch.empty((R_, 1), dtype=torch.uint8, device=t.device)
    q = torch.empty_like(t)
    d = torch.empty_like(t)
    buf = torch.empty(n * k // 8, dtype=torch.uint8, device=t.device)
    ops = {
        "block_max": (lambda: exmy.block_max_exponent(t, "row", y, "before", out=meta), 2 * n, 2 * n),
        "quantize": (lambda: exmy.quantize_blocked(t, (x, y), meta, "row", out=q), 2 * n, 4 * n),
        "encode": (lambda: exmy.encode_blocked(t, (x, y), meta, "row", out=buf, strict=False), 2 * n,
                   2 * n + n * k // 8),
    }
    res = {}
    reps = max(args.steps, 5)
    for name, (fn, in_b, alg_b) in ops.items():
        for _ in range(3):
            fn()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        res[name] = {"us_per_call": round(ms * 1e3, 2), "hbm_gbs": round(alg_b / ms / 1e6, 1),
                     "frac_of_measured": round(alg_b / ms / 1e6 / peak, 4)}
    p = exmy.encode_blocked(t, (x, y), meta, "row", out=buf, strict=False)
    for _ in range(3):
        exmy.decode(p, out=d)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        exmy.decode(p, out=d)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    alg = n * k // 8 + 2 * n
    res["decode"] = {"us_per_call": round(ms * 1e3, 2), "hbm_gbs": round(alg / ms / 1e6, 1),
                     "frac_of_measured": round(alg / ms / 1e6 / peak, 4)}
    res["config"] = "e3m3, ROWS packing, one metadata byte per row (block 1 x 16384), scheme max-before; " \
                    "timed back-to-back through the Python binding (includes its per-call overhead)"
    return res


# ------------------------------------------------------ the oracle arm
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_step(bits, orc, threads: int = 1):
    """One hot-path pass of the CPU oracle over a (rows, C) bf16 sample:
    histogram -> e_max -> 7 x (quantize, encode, decode).  threads > 1 splits
    the rows into contiguous 8-row-aligned chunks, one per thread (the oracle
    is plain single-threaded C; ctypes releases the GIL), with the histogram
    summed across chunks before e_max.  Returns the codec-call input bytes."""
    from concurrent.futures import ThreadPoolExecutor
    rows = bits.shape[0]
    per = max(8, (rows // threads) // 8 * 8)
    chunks = [bits[r:r + per] for r in range(0, rows, per)]
    nbytes = bits.size * 2
    with ThreadPoolExecutor(max_workers=len(chunks)) as ex:
        hists = list(ex.map(orc.histogram, chunks))
        e = orc.emax(sum(hists))
        in_bytes = nbytes

        def one(ch, x, y):
            orc.quantize(ch, (x, y), e)
            p, idx, sb, ns = orc.encode(ch, (x, y), e, orc.ROWS)
            orc.decode(p, ch.shape, (x, y), e, orc.ROWS, idx, sb, ch.dtype)
            return p.size

        for x, y in FORMATS:
            packed = sum(ex.map(lambda ch: one(ch, x, y), chunks))
            in_bytes += nbytes + nbytes + packed
    return in_bytes


def time_oracle(bits, orc, threads: int, reps: int = 3):
    """median wall time of `reps` oracle passes (GB/s of codec-call input)"""
    vals = []
    for _ in range(reps):
        t0 = time.perf_counter()
        nb = oracle_step(bits, orc, threads)
        vals.append(nb / (time.perf_counter() - t0) / 1e9)
    return statistics.median(vals), vals


def cpu_baseline(sample: torch.Tensor):
    """The oracle as it stands (SURVEY 8(d) "Oracle baseline"): one thread and
    all host cores, median of 3 passes each, on a bounded sample of the bench
    tensor (its first rows)."""
    import oracle as orc
    import workloads as W
    bits = W.to_bits(sample)
    orc.lib()
    cores = host_cores()
    one, one_all = time_oracle(bits, orc, 1)
    many, many_all = time_oracle(bits, orc, cores)
    return {"value": round(many, 5), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "single_thread": {"value": round(one, 5), "runs": [round(v, 5) for v in one_all]},
            "all_cores": {"value": round(many, 5), "threads": cores, "runs": [round(v, 5) for v in many_all]},
            "sample": f"rows 0..{bits.shape[0]} of the same 16384x16384 bf16 tensor ({bits.size} elements, "
                      f"{bits.shape[0] / R * 100:.3g}% of it): histogram + 7 x (quantize, encode, decode), "
                      f"scalar C oracle (gcc -O2 -fno-tree-vectorize), median of 3 passes on 1 thread and on "
                      f"{cores} threads (contiguous 8-row chunks)"}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import oracle as orc
    import workloads as W
    t = W.bf16_weights((R, C), seed=SEED, device="cuda" if torch.cuda.is_available() else "cpu")
    rows = args.cpu_rows
    bits = W.to_bits(t[:rows])
    orc.lib()
    cores = host_cores()
    for _ in range(args.warmup):
        oracle_step(bits, orc, cores)
    t0 = time.perf_counter()
    in_bytes = 0
    for _ in range(args.steps):
        in_bytes += oracle_step(bits, orc, cores)
    dt = time.perf_counter() - t0
    v = in_bytes / dt / 1e9
    print(json.dumps({
        "metric": METRIC, "value": round(v, 5), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "impl": "reference",
        "config": {"workload": "config2 sample: rows of the 16384x16384 bf16 ~N(0,0.02^2) tensor, ROWS, "
                               "7-bit formats; step = histogram, e_max, 7x(quantize, encode, decode)",
                   "rows": rows, "elements": int(bits.size)},
        "cpu_baseline": {"value": round(v, 5), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{rows} of {R} rows per step (bounded sample), scalar C oracle on {cores} threads"},
        "e2e": {"value": round(v, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-blocked", action="store_true", help="skip the per-row metadata section")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
