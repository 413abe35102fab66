"""The EXMY checkpoint container (include/exmy.h "checkpoint container";
SURVEY 8(f) row 4, file layout after S:369-378).  CPU tests: the packed
tensors come from the oracle, so the container is checked without a GPU:
bitwise round trip, lazy reads touch only the requested tensor's bytes,
CRC32 catches corruption, malformed files are rejected, file size = n*k/8 +
metadata + manifest (perfect compression).  The GPU test decodes
loaded tensors with the kernels."""
import os
import struct
import zlib

import numpy as np
import pytest
import torch

import workloads as W


@pytest.fixture(scope="module")
def exmy():
    import paper_2405_13938_b200 as m
    return m


def packed_from_oracle(exmy, orc, shape, fmt, seed, per_row=False, dt="bf16", specials=False):
    t = W.bf16_weights(shape, seed=seed) if dt == "bf16" else W.f32_wide(shape, seed=seed)
    bits = W.to_bits(t).copy()
    if specials:
        bits.reshape(-1)[[3, 17]] = 0x7FC0 if dt == "bf16" else 0x7FC00000
    x, y = orc.parse_format(fmt)
    R, C = shape
    if per_row:
        meta = orc.block_max_exponent(bits, (1, C))
        pk, idx, sb, ns = orc.encode_blocked(bits, fmt, meta, (1, C), orc.ROWS)
        block = (1, C)
        m = torch.from_numpy(meta.copy())
    else:
        e = orc.emax(orc.histogram(bits))
        pk, idx, sb, ns = orc.encode(bits, fmt, e, orc.ROWS)
        block = None
        m = torch.tensor([e], dtype=torch.uint8)
    cap = max(ns, 1)
    spi = torch.zeros(cap, dtype=torch.int64)
    spb = torch.zeros(cap, dtype=torch.int32)
    spi[:ns] = torch.from_numpy(idx)
    spb[:ns] = torch.from_numpy(sb.view(np.int32))
    p = exmy.Packed(torch.from_numpy(pk), m, spi, spb, torch.tensor([ns]), shape, x, y, exmy.ROWS,
                    torch.bfloat16 if dt == "bf16" else torch.float32, block)
    return p, bits


def test_roundtrip_and_lazy_reads(exmy, orc, tmp_path):
    path = str(tmp_path / "m.exmy")
    ps = {
        "emb": packed_from_oracle(exmy, orc, (64, 96), "e3m3", 1)[0],
        "w1": packed_from_oracle(exmy, orc, (128, 64), "e2m2", 2, per_row=True)[0],
        "w2": packed_from_oracle(exmy, orc, (32, 48), "e4m4", 3, dt="f32", specials=True)[0],
    }
    size = exmy.save_checkpoint(path, ps)
    assert size == os.path.getsize(path)
    with exmy.Checkpoint(path) as ck:
        assert ck.names == ["emb", "w1", "w2"]
        assert ck.bytes_read == 0                    # opening reads the manifest only
        q = ck.load("w1", device="cpu")
        want = ps["w1"].data.numel() + ps["w1"].meta.numel()
        assert ck.bytes_read == want                 # lazy: only w1's sections
        assert torch.equal(q.data, ps["w1"].data) and torch.equal(q.meta.reshape(-1), ps["w1"].meta.reshape(-1))
        assert q.block == (1, 64) and q.shape == (128, 64) and (q.x, q.y) == (2, 2)
        r = ck.load("w2", device="cpu")
        a, b, c = r.specials()
        a0, b0, c0 = ps["w2"].specials()
        assert c == c0 == 2 and torch.equal(a, a0) and torch.equal(b, b0)
        assert r.dtype == torch.float32
        assert all(ck.verify(n) for n in ck.names)


def test_crc_catches_corruption(exmy, orc, tmp_path):
    path = str(tmp_path / "c.exmy")
    p, _ = packed_from_oracle(exmy, orc, (64, 64), "e3m2", 5)
    exmy.save_checkpoint(path, {"a": p, "b": p})
    raw = bytearray(open(path, "rb").read())
    raw[-10] ^= 0x40                                  # a byte inside tensor b's payload
    open(path, "wb").write(bytes(raw))
    with exmy.Checkpoint(path) as ck:
        assert ck.verify("a") and not ck.verify("b")


def test_crc_is_zlib_crc32(exmy, orc, tmp_path):
    """the stored CRC is the IEEE CRC32 of the payload sections (zlib's)"""
    path = str(tmp_path / "z.exmy")
    p, _ = packed_from_oracle(exmy, orc, (16, 32), "e2m1", 6)
    exmy.save_checkpoint(path, {"t": p})
    raw = open(path, "rb").read()
    payload = p.meta.numpy().tobytes() + p.data.numpy().tobytes()
    crc = struct.unpack("<I", raw[len(raw) - len(payload) - 4:len(raw) - len(payload)])[0]
    assert crc == zlib.crc32(payload)
    assert raw[:4] == b"EXMY" and raw[4] == 2 and struct.unpack("<I", raw[5:9])[0] == 1


def test_file_size_is_perfect_compression(exmy, orc, tmp_path):
    """S:353-ish example: (1024, 4096) e3m2 per row = n*6/8 + 1024 metadata
    bytes + header/manifest (compression vs fp32 ~ 5.33x)"""
    path = str(tmp_path / "s.exmy")
    R, C = 1024, 4096
    p = exmy.Packed(torch.zeros(R * C * 6 // 8, dtype=torch.uint8), torch.zeros((R, 1), dtype=torch.uint8),
                    torch.zeros(1, dtype=torch.int64), torch.zeros(1, dtype=torch.int32), torch.tensor([0]),
                    (R, C), 3, 2, exmy.ROWS, torch.float32, (1, C))
    size = exmy.save_checkpoint(path, {"x": p})
    name_len = 1
    manifest = 2 + name_len + 1 + 2 * 4 + 4 + 1 + 16 * (1 + 2 + 2) + 4   # e3m2: k=6 -> 4+2
    assert size == 9 + manifest + R * C * 6 // 8 + R
    assert 4 * R * C / size > 5.3


def test_empty_and_malformed(exmy, tmp_path):
    path = str(tmp_path / "e.exmy")
    assert exmy.save_checkpoint(path, {}) == 9
    with exmy.Checkpoint(path) as ck:
        assert ck.names == []
    bad = str(tmp_path / "bad.exmy")
    open(bad, "wb").write(b"EXMZ\x01\x00\x00\x00\x00")
    with pytest.raises(exmy.ExmyError) as ei:
        exmy.Checkpoint(bad)
    assert ei.value.status == 10
    open(bad, "wb").write(b"EXMY\x03\x00\x00\x00\x00")     # version 3 (unknown)
    with pytest.raises(exmy.ExmyError):
        exmy.Checkpoint(bad)
    open(bad, "wb").write(b"EXMY\x01\x05\x00\x00\x00abc")  # 5 entries, truncated manifest
    with pytest.raises(exmy.ExmyError):
        exmy.Checkpoint(bad)
    with pytest.raises(exmy.ExmyError) as ei:
        exmy.Checkpoint(str(tmp_path / "missing.exmy"))
    assert ei.value.status == 9


@pytest.mark.gpu
def test_gpu_decode_of_loaded(exmy, orc, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = "cuda"
    t1 = W.bf16_weights((256, 512), seed=7, device=dev)
    t2 = W.bf16_weights((128, 1024), seed=8, device=dev) * 30
    ps = {"a": exmy.encode(t1, "e3m3"), "b": exmy.encode_blocked(t2, "e2m3", None, "row"),
          "c": exmy.encode_fs(t2, "e2m1", None, "row")}
    g = exmy.GroupCodec([t1, torch.ones(4096, dtype=torch.bfloat16, device=dev)], "e4m3")
    for i, p in enumerate(g.encode()):
        ps[f"g{i}"] = p
    path = str(tmp_path / "gpu.exmy")
    exmy.save_checkpoint(path, ps)
    with exmy.Checkpoint(path) as ck:
        for name, p in ps.items():
            q = ck.load(name, device=dev)
            assert torch.equal(q.data, p.data), name
            assert torch.equal(exmy.decode(q).reshape(-1), exmy.decode(p).reshape(-1)), name
            assert ck.verify(name)


def _one_tensor_file(exmy, orc, tmp_path, specials=True):
    path = str(tmp_path / "v.exmy")
    p, _ = packed_from_oracle(exmy, orc, (32, 48), "e4m4", 3, dt="f32", specials=specials)
    exmy.save_checkpoint(path, {"w": p})
    return path, p


def _manifest_fields(raw):
    """offsets of the single entry's fields: (name 'w', rank 2, e4m4: k = 9 ->
    segments w8, w1) -> dict of byte positions"""
    pos = 9 + 2 + 1 + 1 + 8 + 4 + 1            # header, name_len, name, rank, dims, x y scheme kind, flags
    secs = {}
    for name in ("meta", "seg8", "seg1", "scale", "specials"):
        secs[name] = pos
        pos += 16
    return secs


def test_specials_are_interleaved_records(exmy, orc, tmp_path):
    """version 2 stores (u64 index, u32 bits) pairs, as SPEC's container says"""
    path, p = _one_tensor_file(exmy, orc, tmp_path)
    raw = open(path, "rb").read()
    f = _manifest_fields(raw)
    off, ln = struct.unpack("<QQ", raw[f["specials"]:f["specials"] + 16])
    assert ln == 24
    recs = [struct.unpack("<QI", raw[off + 12 * j: off + 12 * j + 12]) for j in range(2)]
    idx, bits, cnt = p.specials()
    assert recs == [(int(idx[j]), int(bits[j]) & 0xFFFFFFFF) for j in range(cnt)]


def test_version1_layout_still_reads(exmy, orc, tmp_path):
    """a version-1 file (indices then bits) loads to the same specials"""
    path, p = _one_tensor_file(exmy, orc, tmp_path)
    raw = bytearray(open(path, "rb").read())
    f = _manifest_fields(raw)
    off, ln = struct.unpack("<QQ", raw[f["specials"]:f["specials"] + 16])
    recs = [struct.unpack("<QI", raw[off + 12 * j: off + 12 * j + 12]) for j in range(ln // 12)]
    v1 = b"".join(struct.pack("<Q", i) for i, _ in recs) + b"".join(struct.pack("<I", b) for _, b in recs)
    raw[off:off + ln] = v1
    raw[4] = 1
    open(path, "wb").write(bytes(raw))
    with exmy.Checkpoint(path) as ck:
        q = ck.load("w", device="cpu")
    a, b, c = q.specials()
    a0, b0, c0 = p.specials()
    assert c == c0 and torch.equal(a, a0) and torch.equal(b, b0)


@pytest.mark.parametrize("field,value", [
    ("seg8", "len+8"),            # segment length != prod(dims) * w / 8
    ("meta", "len+1"),            # metadata length != block count
    ("specials", "len+5"),        # not a whole number of 12-byte records
    ("specials", "wrap"),         # offset + length wraps around 2^64
    ("seg1", "off-1"),            # sections not contiguous
])
def test_malformed_manifest_rejected(exmy, orc, tmp_path, field, value):
    path, _ = _one_tensor_file(exmy, orc, tmp_path)
    raw = bytearray(open(path, "rb").read())
    at = _manifest_fields(raw)[field]
    off, ln = struct.unpack("<QQ", raw[at:at + 16])
    if value == "len+8":
        ln += 8
    elif value == "len+1":
        ln += 1
    elif value == "len+5":
        ln += 5
    elif value == "wrap":
        off, ln = 2 ** 64 - 8, 16
    elif value == "off-1":
        off -= 1
    raw[at:at + 16] = struct.pack("<QQ", off, ln)
    open(path, "wb").write(bytes(raw))
    with pytest.raises(exmy.ExmyError) as ei:
        exmy.Checkpoint(path)
    assert ei.value.status == 10


def test_specials_index_out_of_range_rejected(exmy, orc, tmp_path):
    """a crafted index past the tensor would make the GPU scatter write out of
    bounds: the reader refuses it"""
    path, _ = _one_tensor_file(exmy, orc, tmp_path)
    raw = bytearray(open(path, "rb").read())
    at = _manifest_fields(raw)["specials"]
    off, ln = struct.unpack("<QQ", raw[at:at + 16])
    raw[off:off + 8] = struct.pack("<Q", 32 * 48)     # == numel: one past the end
    open(path, "wb").write(bytes(raw))
    with exmy.Checkpoint(path) as ck:                  # the manifest is fine ...
        with pytest.raises(exmy.ExmyError) as ei:      # ... the read is not
            ck.load("w", device="cpu")
        assert ei.value.status == 10
        assert not ck.verify("w")                     # and the CRC disagrees too


def test_huge_entry_count_rejected(exmy, tmp_path):
    """an entry count the file cannot hold is E_CONTAINER, not an allocation"""
    bad = str(tmp_path / "n.exmy")
    open(bad, "wb").write(b"EXMY\x02\xff\xff\xff\xff" + bytes(64))
    with pytest.raises(exmy.ExmyError) as ei:
        exmy.Checkpoint(bad)
    assert ei.value.status == 10


def test_scheme_is_recorded(exmy, orc, tmp_path):
    """the block scheme (max-before 0 / max-after 1) travels with the tensor"""
    path = str(tmp_path / "s.exmy")
    p, _ = packed_from_oracle(exmy, orc, (16, 32), "e2m1", 6, per_row=True)
    p.scheme = 1
    exmy.save_checkpoint(path, {"t": p})
    with exmy.Checkpoint(path) as ck:
        assert ck.info("t").scheme == 1
        assert ck.load("t", device="cpu").scheme == 1


def test_capacity_zero_packed_writes_no_specials(exmy, orc, tmp_path):
    """a Packed whose encode had capacity 0 but counted NaN/Inf stores no
    (garbage) specials records"""
    path = str(tmp_path / "z.exmy")
    p, _ = packed_from_oracle(exmy, orc, (32, 48), "e4m4", 3, dt="f32", specials=True)
    p.sp_capacity = 0
    exmy.save_checkpoint(path, {"w": p})
    with exmy.Checkpoint(path) as ck:
        assert ck.info("w").specials_count == 0
