"""CPU oracle for the eXmY codec -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2405_13938_b200`` never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around the plain C
oracle in ``exmy_oracle.c``; the arithmetic and its paper citations live there.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "exmy_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_exmy.so")

F32, BF16 = 0, 1
ROWS, COLS = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2, no auto-vectorisation)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "exmy_oracle.h")))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-tree-vectorize", "-ffp-contract=off", "-std=c11", "-Wall", "-Wextra",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        i64, i32, u32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p
        L.oracle_format_valid.argtypes = [i32, i32, i32]
        L.oracle_bias.argtypes = [i32, i32]
        L.oracle_code_magnitude.argtypes = [u32, i32, i32, i32]
        L.oracle_code_magnitude.restype = dbl
        L.oracle_code_value.argtypes = [u32, i32, i32, i32]
        L.oracle_code_value.restype = dbl
        L.oracle_round_f32.argtypes = [dbl]
        L.oracle_round_f32.restype = u32
        L.oracle_round_bf16.argtypes = [dbl]
        L.oracle_round_bf16.restype = ctypes.c_uint16
        L.oracle_encode_codes.argtypes = [vp, i32, i64, i32, i32, i32, vp, vp]
        L.oracle_encode_element.argtypes = [u32, i32, i32, i32, ctypes.POINTER(u32)]
        L.oracle_histogram.argtypes = [vp, i32, i64, vp]
        L.oracle_histogram.restype = None
        L.oracle_emax.argtypes = [vp]
        L.oracle_choose_x.argtypes = [vp, dbl]
        L.oracle_quantize.argtypes = [vp, vp, i32, i64, i32, i32, i32]
        L.oracle_segments.argtypes = [i32, vp, i64, vp]
        L.oracle_shape_ok.argtypes = [i64, i64, i32]
        L.oracle_pack.argtypes = [vp, i64, i64, i32, i32, vp]
        L.oracle_unpack.argtypes = [vp, i64, i64, i32, i32, vp]
        L.oracle_encode.argtypes = [vp, i32, i64, i64, i32, i32, i32, i32, vp, vp, vp, i64]
        L.oracle_encode.restype = i64
        L.oracle_decode.argtypes = [vp, i64, i64, i32, i32, i32, i32, vp, vp, i64, vp, i32]
        L.oracle_block_shape_ok.argtypes = [i64, i64, i64, i64]
        L.oracle_block_max_exponent.argtypes = [vp, i32, i64, i64, i64, i64, i32, i32, vp]
        L.oracle_quantize_blocked.argtypes = [vp, vp, i32, i64, i64, i64, i64, i32, i32, vp]
        L.oracle_encode_blocked.argtypes = [vp, i32, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, i64]
        L.oracle_encode_blocked.restype = i64
        L.oracle_decode_blocked.argtypes = [vp, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, i64, vp, i32]
        L.oracle_fs_grid_top.argtypes = [i32, i32]
        L.oracle_fs_grid_top.restype = dbl
        L.oracle_block_float_scale.argtypes = [vp, i32, i64, i64, i64, i64, vp]
        L.oracle_fs_factor.argtypes = [u32, i32, i32]
        L.oracle_fs_factor.restype = u32
        L.oracle_fs_scale_in.argtypes = [u32, u32, i32, i32]
        L.oracle_fs_scale_in.restype = u32
        L.oracle_fs_scale_out.argtypes = [u32, u32, i32, i32]
        L.oracle_fs_scale_out.restype = u32
        L.oracle_quantize_fs.argtypes = [vp, vp, i32, i64, i64, i64, i64, i32, i32, vp]
        L.oracle_encode_fs.argtypes = [vp, i32, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, i64]
        L.oracle_encode_fs.restype = i64
        L.oracle_decode_fs.argtypes = [vp, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, i64, vp, i32]
        L.oracle_embedding_bag.argtypes = [vp, i64, i64, i32, i32, vp, i32, vp, vp, i64, vp, i32, vp]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return BF16
    if a.dtype == np.uint32:
        return F32
    raise TypeError("oracle takes raw bit patterns: uint32 (fp32) or uint16 (bf16)")


def parse_format(fmt) -> tuple[int, int]:
    if isinstance(fmt, str):
        f = fmt.strip().lower()
        if not f.startswith("e") or "m" not in f:
            raise ValueError(fmt)
        x, y = f[1:].split("m")
        return int(x), int(y)
    return int(fmt[0]), int(fmt[1])


# ------------------------------------------------------------------ scalars
def bias(x: int, e_max: int) -> int:
    return lib().oracle_bias(x, e_max)


def code_value(code: int, fmt, e_max: int) -> float:
    x, y = parse_format(fmt)
    return lib().oracle_code_value(code, x, y, e_max)


def grid(fmt, e_max: int) -> np.ndarray:
    """All 2^k code values (float64), indexed by code."""
    x, y = parse_format(fmt)
    k = 1 + x + y
    return np.array([lib().oracle_code_value(c, x, y, e_max) for c in range(1 << k)])


def round_f32(v: float) -> int:
    return lib().oracle_round_f32(v)


def round_bf16(v: float) -> int:
    return lib().oracle_round_bf16(v)


# ------------------------------------------------------------------- arrays
def histogram(bits: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(bits)
    h = np.zeros(256, dtype=np.uint64)
    lib().oracle_histogram(_p(bits), _dtype_code(bits), bits.size, _p(h))
    return h


def emax(hist: np.ndarray) -> int:
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    return lib().oracle_emax(_p(h))


def choose_x(hist: np.ndarray, budget: float) -> int:
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    return lib().oracle_choose_x(_p(h), budget)


def quantize(bits: np.ndarray, fmt, e_max: int) -> np.ndarray:
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    out = np.empty_like(bits)
    rc = lib().oracle_quantize(_p(bits), _p(out), _dtype_code(bits), bits.size, x, y, e_max)
    if rc:
        raise ValueError("invalid format/e_max")
    return out


def encode_codes(bits: np.ndarray, fmt, e_max: int) -> np.ndarray:
    """Per-element k-bit codes (no packing; specials -> code 0) as uint16."""
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits).reshape(-1)
    codes = np.empty(bits.size, np.uint16)
    special = np.empty(bits.size, np.uint8)
    if lib().oracle_encode_codes(_p(bits), _dtype_code(bits), bits.size, x, y, e_max, _p(codes), _p(special)):
        raise ValueError("invalid format/e_max")
    return codes


def segments(k: int, n: int):
    w = np.zeros(4, np.int32)
    o = np.zeros(4, np.int64)
    ns = lib().oracle_segments(k, _p(w), n, _p(o))
    return [int(v) for v in w[:ns]], [int(v) for v in o[:ns]]


def pack(codes: np.ndarray, shape, axis: int, k: int) -> np.ndarray:
    rows, cols = shape
    codes = np.ascontiguousarray(codes, dtype=np.uint16).reshape(-1)
    out = np.empty(rows * cols * k // 8, np.uint8)
    if lib().oracle_pack(_p(codes), rows, cols, axis, k, _p(out)):
        raise ValueError("bad shape/k")
    return out


def unpack(packed: np.ndarray, shape, axis: int, k: int) -> np.ndarray:
    rows, cols = shape
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.empty(rows * cols, np.uint16)
    if lib().oracle_unpack(_p(packed), rows, cols, axis, k, _p(out)):
        raise ValueError("bad shape/k")
    return out.reshape(rows, cols)


def encode(bits: np.ndarray, fmt, e_max: int, axis: int = ROWS, capacity: int | None = None):
    """Returns (packed uint8, sp_index int64, sp_bits uint32, total_specials)."""
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    k = 1 + x + y
    packed = np.empty(rows * cols * k // 8, np.uint8)
    cap = rows * cols if capacity is None else capacity
    idx = np.empty(max(cap, 1), np.int64)
    sb = np.empty(max(cap, 1), np.uint32)
    ns = lib().oracle_encode(_p(bits), _dtype_code(bits), rows, cols, axis, x, y, e_max, _p(packed), _p(idx), _p(sb), cap)
    if ns < 0:
        raise ValueError("invalid format/e_max/shape")
    kept = min(ns, cap)
    return packed, idx[:kept].copy(), sb[:kept].copy(), int(ns)


def decode(packed: np.ndarray, shape, fmt, e_max: int, axis: int = ROWS,
           sp_index=None, sp_bits=None, out_dtype=np.uint16) -> np.ndarray:
    x, y = parse_format(fmt)
    rows, cols = shape
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    if sp_index is None:
        sp_index = np.zeros(1, np.int64)
        sp_bits = np.zeros(1, np.uint32)
        cnt = 0
    else:
        sp_index = np.ascontiguousarray(sp_index, np.int64)
        sp_bits = np.ascontiguousarray(sp_bits, np.uint32)
        cnt = sp_index.size
    out = np.empty((rows, cols), dtype=out_dtype)
    odt = BF16 if out.dtype == np.uint16 else F32
    rc = lib().oracle_decode(_p(packed), rows, cols, axis, x, y, e_max, _p(sp_index), _p(sp_bits), cnt, _p(out), odt)
    if rc:
        raise ValueError("invalid format/e_max/shape")
    return out


# ------------------------------------------------------------ block metadata
SCHEME_MAX_BEFORE, SCHEME_MAX_AFTER = 0, 1


def block_max_exponent(bits: np.ndarray, block, y: int = 0, scheme: int = SCHEME_MAX_BEFORE) -> np.ndarray:
    """Per-block metadata; bits (rows, cols); block = (br, bc)."""
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    br, bc = block
    meta = np.zeros((rows // br) * (cols // bc), np.uint8)
    if lib().oracle_block_max_exponent(_p(bits), _dtype_code(bits), rows, cols, br, bc, y, scheme, _p(meta)):
        raise ValueError("bad block shape / scheme")
    return meta.reshape(rows // br, cols // bc)


def quantize_blocked(bits: np.ndarray, fmt, meta: np.ndarray, block) -> np.ndarray:
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    m = np.ascontiguousarray(meta, np.uint8)
    out = np.empty_like(bits)
    if lib().oracle_quantize_blocked(_p(bits), _p(out), _dtype_code(bits), rows, cols, block[0], block[1], x, y, _p(m)):
        raise ValueError("invalid arguments")
    return out


def encode_blocked(bits: np.ndarray, fmt, meta: np.ndarray, block, axis: int = ROWS):
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    m = np.ascontiguousarray(meta, np.uint8)
    k = 1 + x + y
    packed = np.empty(rows * cols * k // 8, np.uint8)
    cap = rows * cols
    idx = np.empty(max(cap, 1), np.int64)
    sb = np.empty(max(cap, 1), np.uint32)
    ns = lib().oracle_encode_blocked(_p(bits), _dtype_code(bits), rows, cols, axis, block[0], block[1], x, y, _p(m),
                                     _p(packed), _p(idx), _p(sb), cap)
    if ns < 0:
        raise ValueError("invalid arguments")
    return packed, idx[:ns].copy(), sb[:ns].copy(), int(ns)


def decode_blocked(packed, shape, fmt, meta, block, axis: int = ROWS, sp_index=None, sp_bits=None,
                   out_dtype=np.uint16) -> np.ndarray:
    x, y = parse_format(fmt)
    rows, cols = shape
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    m = np.ascontiguousarray(meta, np.uint8)
    if sp_index is None:
        sp_index, sp_bits, cnt = np.zeros(1, np.int64), np.zeros(1, np.uint32), 0
    else:
        sp_index = np.ascontiguousarray(sp_index, np.int64)
        sp_bits = np.ascontiguousarray(sp_bits, np.uint32)
        cnt = sp_index.size
    out = np.empty((rows, cols), dtype=out_dtype)
    odt = BF16 if out.dtype == np.uint16 else F32
    if lib().oracle_decode_blocked(_p(packed), rows, cols, axis, block[0], block[1], x, y, _p(m), _p(sp_index),
                                   _p(sp_bits), cnt, _p(out), odt):
        raise ValueError("invalid arguments")
    return out


# ------------------------------------------------------------ float scaling
# reading D23: per-block fp32 metadata = largest finite |v|, e_max fixed 127
def fs_grid_top(fmt) -> float:
    x, y = parse_format(fmt)
    return lib().oracle_fs_grid_top(x, y)


def block_float_scale(bits: np.ndarray, block) -> np.ndarray:
    """fp32 bit patterns (uint32) of each block's largest finite magnitude."""
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    br, bc = block
    amax = np.zeros((rows // br) * (cols // bc), np.uint32)
    if lib().oracle_block_float_scale(_p(bits), _dtype_code(bits), rows, cols, br, bc, _p(amax)):
        raise ValueError("bad block shape")
    return amax.reshape(rows // br, cols // bc)


def fs_factor(amax_bits: int, fmt) -> int:
    """fp32 bits of the block's encode factor RN32(G / A1) (amax != 0)"""
    x, y = parse_format(fmt)
    return lib().oracle_fs_factor(amax_bits, x, y)


def fs_scale_in(v_bits: int, amax_bits: int, fmt) -> int:
    x, y = parse_format(fmt)
    return lib().oracle_fs_scale_in(v_bits, amax_bits, x, y)


def fs_scale_out(code: int, amax_bits: int, fmt) -> int:
    x, y = parse_format(fmt)
    return lib().oracle_fs_scale_out(code, amax_bits, x, y)


def quantize_fs(bits: np.ndarray, fmt, amax: np.ndarray, block) -> np.ndarray:
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    a = np.ascontiguousarray(amax, np.uint32)
    out = np.empty_like(bits)
    if lib().oracle_quantize_fs(_p(bits), _p(out), _dtype_code(bits), rows, cols, block[0], block[1], x, y, _p(a)):
        raise ValueError("invalid arguments")
    return out


def encode_fs(bits: np.ndarray, fmt, amax: np.ndarray, block, axis: int = ROWS):
    x, y = parse_format(fmt)
    bits = np.ascontiguousarray(bits)
    rows, cols = bits.shape
    a = np.ascontiguousarray(amax, np.uint32)
    k = 1 + x + y
    packed = np.empty(rows * cols * k // 8, np.uint8)
    cap = rows * cols
    idx = np.empty(max(cap, 1), np.int64)
    sb = np.empty(max(cap, 1), np.uint32)
    ns = lib().oracle_encode_fs(_p(bits), _dtype_code(bits), rows, cols, axis, block[0], block[1], x, y, _p(a),
                                _p(packed), _p(idx), _p(sb), cap)
    if ns < 0:
        raise ValueError("invalid arguments")
    return packed, idx[:ns].copy(), sb[:ns].copy(), int(ns)


def decode_fs(packed, shape, fmt, amax, block, axis: int = ROWS, sp_index=None, sp_bits=None,
              out_dtype=np.uint16) -> np.ndarray:
    x, y = parse_format(fmt)
    rows, cols = shape
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    a = np.ascontiguousarray(amax, np.uint32)
    if sp_index is None:
        sp_index, sp_bits, cnt = np.zeros(1, np.int64), np.zeros(1, np.uint32), 0
    else:
        sp_index = np.ascontiguousarray(sp_index, np.int64)
        sp_bits = np.ascontiguousarray(sp_bits, np.uint32)
        cnt = sp_index.size
    out = np.empty((rows, cols), dtype=out_dtype)
    odt = BF16 if out.dtype == np.uint16 else F32
    if lib().oracle_decode_fs(_p(packed), rows, cols, axis, block[0], block[1], x, y, _p(a), _p(sp_index),
                              _p(sp_bits), cnt, _p(out), odt):
        raise ValueError("invalid arguments")
    return out


# ------------------------------------------------------------ embedding bag
def embedding_bag(packed, shape, fmt, meta, indices, offsets, weights=None, mode="sum") -> np.ndarray:
    """Pooled decode of rows of a COLS-packed table (reading D25): fp32
    (nbags, cols); meta: one byte (per tensor) or one per row."""
    x, y = parse_format(fmt)
    rows, cols = shape
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    m = np.ascontiguousarray(np.asarray(meta, dtype=np.uint8).reshape(-1))
    per_row = 1 if m.size == rows and rows != 1 else 0
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    nb = off.size - 1
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
    out = np.zeros((nb, cols), np.float32)
    if lib().oracle_embedding_bag(_p(packed), rows, cols, x, y, _p(m), per_row, _p(idx), _p(off), nb,
                                  None if w is None else _p(w), 0 if mode == "sum" else 1, _p(out)):
        raise ValueError("invalid arguments")
    return out
