"""N>1 host logic of the sharded driver (paper_2405_13938_b200.dist) on CPU:
world_size 2 and 4 over gloo, with the oracle standing in for the kernels
(the product path itself has no CPU fallback).  Checks the two properties
the exchange step must give: all-gathered packed bytes == a single encode of
the whole tensor (global e_max via the histogram all-reduce), and
decode of every gathered shard == quantize of the whole tensor."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleCodec:
    """The four codec calls of the binding, computed by the CPU oracle."""

    def __init__(self):
        import oracle
        self.o = oracle
        oracle.lib()

    def segments(self, k, n):
        return self.o.segments(k, n)

    def histogram(self, t):
        import workloads as W
        return torch.from_numpy(self.o.histogram(W.to_bits(t)).astype(np.int64))

    def emax(self, hist):
        return torch.tensor([self.o.emax(hist.numpy().astype(np.uint64))], dtype=torch.uint8)

    CAP = 16

    def encode(self, t, fmt, meta, axis="rows", strict=True):
        import workloads as W
        x, y = self.o.parse_format(fmt)
        bits = W.to_bits(t)
        ax = self.o.ROWS if axis == "rows" else self.o.COLS
        packed, idx, sb, ns = self.o.encode(bits, (x, y), int(meta.item()), ax)
        spi = torch.zeros(self.CAP, dtype=torch.int64)
        spb = torch.zeros(self.CAP, dtype=torch.int32)
        c = min(ns, self.CAP)
        spi[:c] = torch.from_numpy(np.asarray(idx[:c], np.int64))
        spb[:c] = torch.from_numpy(np.asarray(sb[:c]).astype(np.uint32).view(np.int32))
        return types.SimpleNamespace(data=torch.from_numpy(packed), x=x, y=y, sp_index=spi, sp_bits=spb,
                                     sp_count=torch.tensor([ns], dtype=torch.int64), capacity=self.CAP)

    def decode_raw(self, data, rows, cols, fmt, meta, axis="rows", dtype=torch.bfloat16, specials=None):
        import workloads as W
        ax = self.o.ROWS if axis == "rows" else self.o.COLS
        idx = sb = None
        if specials is not None:
            spi, spb, spc, cap = specials
            c = min(int(spc.reshape(-1)[0]), cap)
            idx = spi[:c].numpy().astype(np.int64)
            sb = spb[:c].numpy().view(np.uint32)
        out = self.o.decode(data.numpy(), (rows, cols), fmt, int(meta.item()) if torch.is_tensor(meta) else meta,
                            ax, idx, sb, out_dtype=np.uint16 if dtype == torch.bfloat16 else np.uint32)
        return W.from_bits(out)


class OraclePushCodec(OracleCodec):
    """encode_push on CPU: the shard's oracle bytes copied to their global
    offsets in each destination (shared-memory tensors standing in for the
    NVLink-mapped peer buffers)."""

    def encode_push(self, shard, fmt, meta, row0, total_rows, dsts):
        import workloads as W
        x, y = self.o.parse_format(fmt)
        k = 1 + x + y
        R, C = shard.shape
        packed = self.o.encode(W.to_bits(shard), (x, y), int(meta.item()), self.o.ROWS)[0]
        ws, offs_local = self.o.segments(k, R * C)
        _, offs_glob = self.o.segments(k, total_rows * C)
        for w, ol, og in zip(ws, offs_local, offs_glob):
            n = R * C * w // 8
            start = og + row0 * C * w // 8
            for d in dsts:
                d[start:start + n] = torch.from_numpy(packed[ol:ol + n])
        return None

    def decode_pull(self, srcs, shard_rows, cols, fmt, meta, dtype=torch.bfloat16):
        import workloads as W
        od = np.uint16 if dtype == torch.bfloat16 else np.uint32
        parts = [self.o.decode(s_.numpy(), (shard_rows, cols), fmt, int(meta.item()), self.o.ROWS, out_dtype=od)
                 for s_ in srcs]
        return W.from_bits(np.concatenate(parts))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _specials_tensor():
    """NaN/Inf in every quarter of the rows, so every rank (up to 4) carries a
    list; specials don't disturb the byte layout and decode restores them"""
    import workloads as W
    full = W.bf16_weights((64, 48), seed=11, std=0.05)
    flat = full.view(-1)
    flat[5] = float("inf")
    flat[48 * 20 + 3] = float("-inf")
    flat[48 * 33] = float("nan")
    flat[48 * 63 + 47] = float("nan")
    return full


def _worker(rank, ws, port, fmt, axis, results):
    import sys
    sys.path.insert(0, ROOT)
    import workloads as W
    from paper_2405_13938_b200 import dist as xdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        full = _specials_tensor()
        r0, r1 = xdist.shard_rows(64, ws, rank, axis == "rows")
        codec = OracleCodec()
        glob, dec, (gi, gb) = xdist.sharded_roundtrip(full[r0:r1].contiguous(), fmt, axis=axis, codec=codec,
                                                      return_specials=True)
        results[rank] = (glob.numpy().tobytes(), W.to_bits(dec).tobytes(), gi.numpy().tolist(),
                         gb.numpy().view(np.uint32).tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 4])
@pytest.mark.parametrize("fmt,axis", [("e3m3", "rows"), ("e2m2", "cols"), ("e5m3", "rows"), ("e1m1", "cols")])
def test_sharded_roundtrip_gloo(orc, ws, fmt, axis):
    import workloads as W
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, fmt, axis, results)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    bits = W.to_bits(_specials_tensor())
    e = orc.emax(orc.histogram(bits))
    ax = orc.ROWS if axis == "rows" else orc.COLS
    ref_packed, ref_idx, ref_bits, ref_n = orc.encode(bits, fmt, e, ax)
    assert ref_n == 4
    q = orc.quantize(bits, fmt, e)     # NaN/Inf pass through quantize; decode restores them from the lists
    for r in range(ws):
        glob, dec, gi, gb = results[r]
        assert np.frombuffer(glob, np.uint8).tolist() == ref_packed.tolist()
        np.testing.assert_array_equal(np.frombuffer(dec, np.uint16).reshape(64, 48), q)
        assert gi == list(ref_idx) and gb == [int(b) for b in ref_bits]


def test_shard_rows_validation():
    from paper_2405_13938_b200 import dist as xdist
    assert xdist.shard_rows(64, 4, 1) == (16, 32)
    with pytest.raises(ValueError):
        xdist.shard_rows(60, 8, 0)
    with pytest.raises(ValueError):
        xdist.shard_rows(64, 4, 0, True) if False else xdist.shard_rows(48, 4, 0, True)
    assert xdist.shard_rows(48, 4, 0, False) == (0, 12)


def _push_worker(rank, ws, port, fmt, paths, results):
    import sys
    sys.path.insert(0, ROOT)
    import workloads as W
    from paper_2405_13938_b200 import dist as xdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        full = W.bf16_weights((64, 48), seed=13, std=0.05)
        r0, r1 = xdist.shard_rows(64, ws, rank, True)
        codec = OraclePushCodec()
        x, y = codec.o.parse_format(fmt)
        nb = 64 * 48 * (1 + x + y) // 8
        # every rank maps every rank's buffer (the symmetric-memory picture)
        peers = [torch.from_file(p, shared=True, size=nb, dtype=torch.uint8) for p in paths]
        meta, _ = xdist.pushed_encode(full[r0:r1].contiguous(), fmt, 64, r0, peers, codec=codec)
        results[rank] = (peers[rank].numpy().tobytes(), int(meta.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 4])
@pytest.mark.parametrize("fmt", ["e3m3", "e2m1", "e4m4"])
def test_pushed_encode_gloo(orc, tmp_path, ws, fmt):
    """fused encode + all-gather host wiring: each rank's buffer ends as the
    single encode of the whole tensor, with the all-reduced global e_max"""
    import workloads as W
    x, y = orc.parse_format(fmt)
    nb = 64 * 48 * (1 + x + y) // 8
    paths = []
    for r in range(ws):
        p = tmp_path / f"peer{r}.bin"
        p.write_bytes(bytes(nb))
        paths.append(str(p))
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_push_worker, args=(r, ws, port, fmt, paths, results)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    bits = W.to_bits(W.bf16_weights((64, 48), seed=13, std=0.05))
    e = orc.emax(orc.histogram(bits))
    ref = orc.encode(bits, fmt, e, orc.ROWS)[0]
    for r in range(ws):
        buf, meta = results[r]
        assert meta == e
        assert np.frombuffer(buf, np.uint8).tolist() == ref.tolist()


def _pull_worker(rank, ws, port, fmt, paths, results):
    import sys
    sys.path.insert(0, ROOT)
    import workloads as W
    from paper_2405_13938_b200 import dist as xdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        full = W.bf16_weights((64, 48), seed=17, std=0.05)
        r0, r1 = xdist.shard_rows(64, ws, rank, True)
        codec = OraclePushCodec()
        x, y = codec.o.parse_format(fmt)
        per = 64 // ws
        nb = per * 48 * (1 + x + y) // 8
        hist = codec.histogram(full[r0:r1].contiguous())
        xdist.allreduce_histogram(hist)
        meta = codec.emax(hist)
        # this rank's packed shard into its own shared buffer, then pull everything
        mine = torch.from_file(paths[rank], shared=True, size=nb, dtype=torch.uint8)
        mine.copy_(codec.encode(full[r0:r1].contiguous(), fmt, meta).data)
        peers = [torch.from_file(p_, shared=True, size=nb, dtype=torch.uint8) for p_ in paths]
        out = xdist.pulled_decode(mine, per, 48, fmt, meta, peers, codec=codec)
        results[rank] = W.to_bits(out).tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 4])
def test_pulled_decode_gloo(orc, tmp_path, ws):
    """pull-decode host wiring: every rank decodes the whole tensor from all
    ranks' packed shards == the oracle's quantize of the whole tensor"""
    import workloads as W
    fmt = "e3m3"
    nb = (64 // ws) * 48 * 7 // 8
    paths = []
    for r in range(ws):
        p = tmp_path / f"shard{r}.bin"
        p.write_bytes(bytes(nb))
        paths.append(str(p))
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_pull_worker, args=(r, ws, port, fmt, paths, results)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    bits = W.to_bits(W.bf16_weights((64, 48), seed=17, std=0.05))
    ref = orc.quantize(bits, fmt, orc.emax(orc.histogram(bits)))
    for r in range(ws):
        np.testing.assert_array_equal(np.frombuffer(results[r], np.uint16).reshape(64, 48), ref)
