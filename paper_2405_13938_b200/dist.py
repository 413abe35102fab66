"""Sharded eXmY driver (A8): one process per GPU, torch.distributed (NCCL over
NVLink 5 / NVSwitch on B200; gloo in the CPU tests).

The paper's layout is shard-friendly: "the array can be sharded along rows or
columns, before or after packing, and each shard can be independently
reconstructed".  Rank r owns rows [r*R/G, (r+1)*R/G); a row
shard's packed bytes are, per segment j, the contiguous byte range
off_j + [r0*C*w_j/8, r1*C*w_j/8) of the single-GPU packed buffer.  So:

  1. each rank histograms its shard; one 2 KiB all-reduce (sum) gives the
     global per-tensor histogram -> global e_max (metadata);
  2. encode / decode are embarrassingly parallel (no communication);
  3. the exchange of compressed shards ("network
     communication") is one all-gather of each rank's packed bytes;
     `to_global_layout` re-arranges the gathered shard buffers into exactly
     the bytes a single-GPU encode of the whole tensor produces.

The codec calls go through ``codec`` (default: this package's CUDA binding)
so the host logic can be exercised with any implementation of the same four
calls; the product path has no CPU fallback.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _default_codec():
    import paper_2405_13938_b200 as exmy
    return exmy


def shard_rows(R: int, G: int, r: int, axis_rows: bool = True) -> tuple[int, int]:
    """Row range of rank r (ROWS packing needs multiples of 8)."""
    if R % G:
        raise ValueError(f"rows {R} not divisible by world size {G}")
    per = R // G
    if axis_rows and per % 8:
        raise ValueError("ROWS packing needs R/G to be a multiple of 8 (P:351-353)")
    return r * per, (r + 1) * per


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo (CPU tests / 1-GPU smoke runs) moves device tensors through host."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def allreduce_histogram(hist: torch.Tensor, group=None) -> torch.Tensor:
    """C1: sum of the per-rank exponent histograms (int64[256], in place)."""
    if _host_staged(hist, group):
        h = hist.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        hist.copy_(h)
        return hist
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def allgather_bytes(local: torch.Tensor, out: torch.Tensor, group=None) -> torch.Tensor:
    """C2: all-gather of equal-size packed shards into out[G * nbytes]."""
    if _host_staged(local, group) or dist.get_backend(group) == "gloo":
        G = dist.get_world_size(group)
        parts = [torch.empty_like(local, device="cpu") for _ in range(G)]
        dist.all_gather(parts, local.cpu(), group=group)
        out.copy_(torch.cat(parts))
        return out
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def to_global_layout(gathered: torch.Tensor, G: int, rows_per_rank: int, C: int, k: int, codec=None) -> torch.Tensor:
    """Rearrange G concatenated shard buffers (rank order) into the byte layout
    of a single encode of the full (G*rows_per_rank, C) tensor."""
    codec = codec or _default_codec()
    n_local = rows_per_rank * C
    nb = n_local * k // 8
    ws, offs = codec.segments(k, n_local)
    parts = []
    for w, o in zip(ws, offs):
        seg_len = n_local * w // 8
        for r in range(G):
            parts.append(gathered[r * nb + o: r * nb + o + seg_len])
    return torch.cat(parts)


def sharded_encode(shard: torch.Tensor, fmt, axis="rows", group=None, codec=None):
    """Encode this rank's row shard with the GLOBAL per-tensor e_max.
    Returns (packed, meta); byte-identical to the corresponding ranges of a
    single-GPU encode of the full tensor."""
    codec = codec or _default_codec()
    hist = codec.histogram(shard)
    allreduce_histogram(hist, group)
    meta = codec.emax(hist)
    return codec.encode(shard, fmt, meta, axis=axis, strict=False), meta


def _allgather_stack(t: torch.Tensor, group=None) -> torch.Tensor:
    """[G, *t.shape] of every rank's equal-shape tensor (rank order)."""
    G = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "gloo":
        parts = [torch.empty_like(t, device="cpu") for _ in range(G)]
        dist.all_gather(parts, t.cpu(), group=group)
        return torch.stack(parts).to(t.device)
    out = torch.empty((G,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out


def allgather_specials(p, group=None):
    """Every rank's out-of-band NaN/Inf list (D9): (index[G, cap],
    bits[G, cap], count[G]) with shard-local indices, and the capacity.
    Raises E_CAPACITY (synchronising) if any rank overflowed its list, so no
    NaN/Inf is ever dropped silently."""
    cap = int(p.capacity)
    n = max(cap, 1)
    idx = _allgather_stack(p.sp_index[:n], group)
    bits = _allgather_stack(p.sp_bits[:n], group)
    cnt = _allgather_stack(p.sp_count.reshape(-1)[:1].to(torch.int64), group).reshape(-1)
    worst = int(cnt.max())
    if worst > cap:
        import paper_2405_13938_b200 as exmy
        raise exmy.ExmyError(6, f"sharded encode: a shard holds {worst} NaN/Inf but the specials capacity is {cap}")
    return idx, bits, cnt, cap


def global_specials(idx, bits, cnt, elems_per_rank: int):
    """Concatenate the per-rank lists into the single-GPU list: indices offset
    by r * elems_per_rank (row-major shards), ascending."""
    gi, gb = [], []
    for r in range(idx.shape[0]):
        c = int(cnt[r])
        gi.append(idx[r, :c] + r * elems_per_rank)
        gb.append(bits[r, :c])
    return torch.cat(gi), torch.cat(gb)


def sharded_roundtrip(shard: torch.Tensor, fmt, axis="rows", group=None, codec=None, gather=True,
                      return_specials=False):
    """Encode own shard -> all-gather packed shards and specials lists ->
    decode every shard with its own specials (NaN/Inf restored, D9).
    Returns (global packed bytes in single-GPU layout, decoded full tensor)
    [, (global specials index, bits)]."""
    codec = codec or _default_codec()
    G = dist.get_world_size(group)
    p, meta = sharded_encode(shard, fmt, axis, group, codec)
    R_local, C = (1, shard.shape[0]) if shard.dim() == 1 else (shard.numel() // shard.shape[-1], shard.shape[-1])
    nb = p.data.numel()
    out = torch.empty(G * nb, dtype=torch.uint8, device=p.data.device)
    allgather_bytes(p.data, out, group)
    sidx, sbits, scnt, cap = allgather_specials(p, group)
    k = 1 + p.x + p.y
    glob = to_global_layout(out, G, R_local, C, k, codec)
    dec = None
    if gather:
        dec = torch.cat([codec.decode_raw(out[r * nb:(r + 1) * nb], R_local, C, (p.x, p.y), meta, axis=axis,
                                          dtype=shard.dtype,
                                          specials=(sidx[r], sbits[r], scnt[r:r + 1], cap))
                         for r in range(G)], 0)
    if return_specials:
        return glob, dec, global_specials(sidx, sbits, scnt, R_local * C)
    return glob, dec


# --------------------------------------------- fused encode + all-gather (push)
_SYMM_HANDLES = {}


def symmetric_packed_buffers(nbytes: int, group=None):
    """This rank's gathered packed buffer plus every rank's, mapped into this
    process (NVLink peer memory through torch symmetric memory): the
    destinations of `pushed_encode`.  Needs CUDA peers (NCCL group).  The
    rendezvous handle is kept (multicast_status / multicast pushes)."""
    from torch.distributed import _symmetric_memory as symm_mem
    buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
    h = symm_mem.rendezvous(buf, group=dist.group.WORLD if group is None else group)
    peers = [h.get_buffer(r, (nbytes,), torch.uint8) for r in range(h.world_size)]
    _SYMM_HANDLES[buf.data_ptr()] = h
    return buf, peers


def multicast_ptr(buf) -> int:
    """The NVLS multicast address bound to `buf` (from symmetric_packed_buffers)
    on every rank, or 0 when this node / driver offers no multicast."""
    h = _SYMM_HANDLES.get(buf.data_ptr())
    if h is None:
        return 0
    try:
        return int(getattr(h, "multicast_ptr", 0) or 0)
    except Exception:
        return 0


def multicast_status(buf) -> dict:
    h = _SYMM_HANDLES.get(buf.data_ptr())
    return {"symmetric": h is not None, "world_size": getattr(h, "world_size", None),
            "multicast": multicast_ptr(buf) != 0}


def pushed_encode(shard: torch.Tensor, fmt, total_rows: int, row0: int, peer_buffers, group=None, codec=None,
                  meta=None, multicast: int = 0):
    """Fused encode + all-gather: the global metadata from
    the 2 KiB histogram all-reduce (unless given), then ONE kernel encodes this
    rank's row shard and stores its bytes at their global offsets into every
    rank's buffer (peer_buffers), then a barrier.  Afterwards every rank's
    buffer holds the single-GPU encode of the whole tensor -- no NCCL
    all-gather, no staging copy, the transfer overlaps the conversion.
    multicast: a multicast address of the gathered buffer (multicast_ptr):
    one multimem.st per store reaches every rank (NVLS) instead of one store
    per peer.  Returns (meta, specials of the shard with global indices)."""
    codec = codec or _default_codec()
    if meta is None:
        hist = codec.histogram(shard)
        allreduce_histogram(hist, group)
        meta = codec.emax(hist)
    if multicast:
        sp = codec.encode_push_multicast(shard, fmt, meta, row0, total_rows, multicast)
    else:
        sp = codec.encode_push(shard, fmt, meta, row0, total_rows, peer_buffers)
    if shard.is_cuda:
        torch.cuda.current_stream(shard.device).synchronize()   # the stores have landed before peers read
    dist.barrier(group)
    return meta, sp


def pulled_decode(local_packed: torch.Tensor, shard_rows: int, cols: int, fmt, meta, peer_buffers, group=None,
                  codec=None, dtype=torch.bfloat16):
    """Decode the whole tensor from every rank's packed shard (peer_buffers:
    this process's mappings of each rank's packed shard buffer, symmetric
    memory), the mirror of `pushed_encode`: one kernel, the all-gather happens
    in its loads.  A barrier first makes every rank's shard complete."""
    codec = codec or _default_codec()
    if local_packed.is_cuda:
        torch.cuda.current_stream(local_packed.device).synchronize()
    dist.barrier(group)
    return codec.decode_pull(peer_buffers, shard_rows, cols, fmt, meta, dtype=dtype)
