"""eXmY tensor codec on B200 (arXiv 2405.13938) -- thin Python binding.

Argument marshalling only: every step of the codec runs in the sm_100a
kernels of ``libexmy.so`` through its C ABI (``include/exmy.h``).  PyTorch is
used for device memory, streams and process groups.  There is no CPU
fallback: importing without the built library raises.

    import paper_2405_13938_b200 as exmy
    h = exmy.histogram(t)                  # uint64[256] on t.device
    meta = exmy.emax(h)                    # uint8[1] device metadata
    q = exmy.quantize(t, "e3m2", meta)     # emulation
    p = exmy.encode(t, "e3m3", axis="rows")  # Packed
    t2 = exmy.decode(p)                    # == quantize(t, "e3m3", p.meta)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# EXMY_LIB_PATH: A/B experiments with an alternative build of the same ABI
_LIB_PATH = os.environ.get("EXMY_LIB_PATH") or os.path.join(_PKG, "libexmy.so")

F32, BF16 = 0, 1
ROWS, COLS = 0, 1
_AXES = {"rows": ROWS, "cols": COLS, ROWS: ROWS, COLS: COLS}

STATUS = {0: "ok", 1: "E_FORMAT", 2: "E_META", 3: "E_SHAPE", 4: "E_DTYPE", 5: "E_ALIGN",
          6: "E_CAPACITY", 7: "E_CUDA", 8: "E_ARG", 9: "E_IO", 10: "E_CONTAINER", 11: "E_CHECKSUM"}


class ExmyError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {STATUS.get(status, status)} ({_lib.exmy_status_string(status).decode()})")


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the codec has no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
    sig = {
        "exmy_version": ([], ctypes.c_char_p),
        "exmy_specials_words": ([], i32),
        "exmy_status_string": ([i32], ctypes.c_char_p),
        "exmy_format_valid": ([i32, i32], i32),
        "exmy_packed_bytes": ([i64, i32, i32], i64),
        "exmy_segments": ([i32, i64, vp, vp], i32),
        "exmy_bias_from_emax": ([i32, i32, vp], i32),
        "exmy_emax_from_bias": ([i32, i32, vp], i32),
        "exmy_emax_from_histogram_host": ([vp], i32),
        "exmy_choose_x": ([vp, dbl, vp], i32),
        "exmy_debug_force_generic": ([i32], i32),
        "exmy_debug_hist_mode": ([i32], i32),
        "exmy_debug_hist_blocks": ([i32], i32),
        "exmy_debug_enc_tma": ([i32], i32),
        "exmy_debug_rowwise_cluster": ([i32], i32),
        "exmy_debug_probe": ([vp, i64, vp, i64, vp], i32),
        "exmy_exponent_histogram": ([vp, i32, i64, vp, vp], i32),
        "exmy_emax_from_histogram": ([vp, vp, vp], i32),
        "exmy_max_exponent": ([vp, i32, i64, vp, vp], i32),
        "exmy_quantize": ([vp, vp, i32, i64, i32, i32, vp, vp], i32),
        "exmy_encode": ([vp, i32, i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "exmy_decode": ([vp, i64, i64, i32, i32, i32, vp, vp, vp, vp, i64, vp, i32, vp], i32),
        "exmy_block_max_exponent": ([vp, i32, i64, i64, i64, i64, i32, i32, vp, vp], i32),
        "exmy_quantize_blocked": ([vp, vp, i32, i64, i64, i64, i64, i32, i32, vp, vp], i32),
        "exmy_encode_blocked": ([vp, i32, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "exmy_decode_blocked": ([vp, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, i64, vp, i32, vp], i32),
        "exmy_encode_rowwise": ([vp, i32, i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "exmy_decode_rows": ([vp, i64, i64, i32, i32, vp, i32, vp, i64, vp, i32, vp], i32),
        "exmy_encode_host": ([vp, i32, i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp], i32),
        "exmy_decode_host": ([vp, i64, i64, i32, i32, i32, vp, vp, vp, vp, i64, vp, vp, i32, vp, vp], i32),
        "exmy_block_float_scale": ([vp, i32, i64, i64, i64, i64, vp, vp], i32),
        "exmy_quantize_fs": ([vp, vp, i32, i64, i64, i64, i64, i32, i32, vp, vp], i32),
        "exmy_encode_fs": ([vp, i32, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "exmy_decode_fs": ([vp, i64, i64, i32, i64, i64, i32, i32, vp, vp, vp, vp, i64, vp, i32, vp], i32),
        "exmy_encode_push": ([vp, i32, i64, i64, i64, i64, i32, i32, vp, vp, i32, vp, vp, vp, i64, vp], i32),
        "exmy_encode_push_multicast": ([vp, i32, i64, i64, i64, i64, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "exmy_embedding_bag": ([vp, i64, i64, i32, i32, vp, i32, vp, vp, i64, vp, i32, vp, vp], i32),
        "exmy_gemv": ([vp, i64, i64, i32, i32, vp, i32, vp, vp, vp, i64, vp, i64, vp, vp], i32),
        "exmy_debug_gemv_bulk": ([i32], i32),
        "exmy_decode_pull": ([vp, i32, i64, i64, i32, i32, vp, vp, i32, vp], i32),
        "exmy_ckpt_write": ([ctypes.c_char_p, vp, i32], i64),
        "exmy_ckpt_open": ([ctypes.c_char_p, vp], i32),
        "exmy_ckpt_count": ([vp], i32),
        "exmy_ckpt_info": ([vp, i32, vp], i32),
        "exmy_ckpt_find": ([vp, ctypes.c_char_p], i32),
        "exmy_ckpt_read": ([vp, i32, vp, vp, vp, vp, vp], i32),
        "exmy_ckpt_verify": ([vp, i32], i32),
        "exmy_ckpt_bytes_read": ([vp], i64),
        "exmy_ckpt_close": ([vp], None),
        "exmy_group_plan_bytes": ([i32], ctypes.c_size_t),
        "exmy_group_plan": ([vp, i32, i32, i32, i32, i32, vp, ctypes.c_size_t], i32),
        "exmy_group_plan_rows": ([vp, i32, i32, i32, i32, i32, vp, ctypes.c_size_t], i32),
        "exmy_group_max_exponent": ([vp, vp, vp], i32),
        "exmy_group_encode": ([vp, vp, vp], i32),
        "exmy_group_encode_rowwise": ([vp, vp, vp], i32),
        "exmy_group_decode": ([vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib = _load()
LIB_PATH = _LIB_PATH
EXPORTED = ["exmy_version", "exmy_specials_words", "exmy_status_string", "exmy_format_valid", "exmy_packed_bytes", "exmy_segments",
            "exmy_bias_from_emax", "exmy_emax_from_bias", "exmy_emax_from_histogram_host", "exmy_choose_x",
            "exmy_debug_force_generic", "exmy_debug_hist_mode", "exmy_debug_hist_blocks", "exmy_debug_enc_tma", "exmy_debug_rowwise_cluster", "exmy_debug_gemv_bulk", "exmy_debug_probe",
            "exmy_exponent_histogram",
            "exmy_emax_from_histogram", "exmy_quantize", "exmy_encode", "exmy_decode", "exmy_encode_host",
            "exmy_decode_host", "exmy_block_max_exponent", "exmy_quantize_blocked", "exmy_encode_blocked",
            "exmy_decode_blocked", "exmy_decode_rows", "exmy_max_exponent", "exmy_encode_rowwise",
            "exmy_group_plan_bytes", "exmy_group_plan", "exmy_group_plan_rows", "exmy_group_max_exponent", "exmy_group_encode", "exmy_group_encode_rowwise",
            "exmy_group_decode", "exmy_block_float_scale", "exmy_quantize_fs", "exmy_encode_fs", "exmy_decode_fs",
            "exmy_encode_push", "exmy_encode_push_multicast", "exmy_decode_pull", "exmy_embedding_bag", "exmy_gemv", "exmy_ckpt_write", "exmy_ckpt_open", "exmy_ckpt_count", "exmy_ckpt_info",
            "exmy_ckpt_find", "exmy_ckpt_read", "exmy_ckpt_verify", "exmy_ckpt_bytes_read", "exmy_ckpt_close"]


def lib():
    return _lib


SPECIALS_WORDS = _lib.exmy_specials_words()   # the sp_count workspace (include/exmy.h)


def specials_workspace(device) -> torch.Tensor:
    """device int64[SPECIALS_WORDS]: word 0 = the specials count (uint64)"""
    return torch.zeros(SPECIALS_WORDS, dtype=torch.int64, device=device)


def version() -> str:
    return _lib.exmy_version().decode()


# ----------------------------------------------------------------- helpers
def parse_format(fmt) -> tuple[int, int]:
    """'e3m2' -> (3, 2); case-insensitive."""
    if isinstance(fmt, str):
        f = fmt.strip().lower()
        if not f.startswith("e") or "m" not in f:
            raise ValueError(f"bad format {fmt!r}")
        x, y = f[1:].split("m")
        x, y = int(x), int(y)
    else:
        x, y = int(fmt[0]), int(fmt[1])
    if not _lib.exmy_format_valid(x, y):
        raise ValueError(f"unsupported format e{x}m{y} (x in [0,8], 3 <= 1+x+y <= 9)")
    return x, y


def format_name(x: int, y: int) -> str:
    return f"e{x}m{y}"


def all_formats(kmin: int = 3, kmax: int = 9):
    """Every GPU format of total width kmin..kmax (42 formats for 3..9)."""
    return [(x, k - 1 - x) for k in range(kmin, kmax + 1) for x in range(0, min(8, k - 1) + 1)]


def packed_bytes(n: int, fmt) -> int:
    x, y = parse_format(fmt)
    r = _lib.exmy_packed_bytes(n, x, y)
    if r < 0:
        raise ValueError("n must be a non-negative multiple of 8")
    return r


def segments(k: int, n: int):
    w = (ctypes.c_int * 4)()
    o = (ctypes.c_int64 * 4)()
    ns = _lib.exmy_segments(k, n, w, o)
    if ns < 0:
        raise ValueError("bad k or n")
    return list(w)[:ns], list(o)[:ns]


def bias_from_emax(x: int, e_max: int) -> int:
    b = ctypes.c_int()
    _check(_lib.exmy_bias_from_emax(x, e_max, ctypes.byref(b)), "bias_from_emax")
    return b.value


def emax_from_bias(x: int, bias: int) -> int:
    e = ctypes.c_int()
    _check(_lib.exmy_emax_from_bias(x, bias, ctypes.byref(e)), "emax_from_bias")
    return e.value


def choose_x(hist, flush_budget: float = 0.0011) -> int:
    """X from a histogram; hist: 256 counts (any device)."""
    h = torch.as_tensor(hist).detach().to("cpu", torch.int64).contiguous()
    xo = ctypes.c_int()
    _check(_lib.exmy_choose_x(ctypes.c_void_p(h.data_ptr()), float(flush_budget), ctypes.byref(xo)), "choose_x")
    return xo.value


def force_generic(on: bool | None = None) -> bool:
    """Test knob: route everything through the integer generic paths."""
    return bool(_lib.exmy_debug_force_generic(-1 if on is None else int(on)))


def hist_mode(mode: int | None = None) -> int:
    return _lib.exmy_debug_hist_mode(-1 if mode is None else int(mode))


def roofline_probe(src: torch.Tensor, out_bytes: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """diagnostic (exmy_debug_probe): stream src's bytes in and out_bytes out
    with the codec's access shape; time it for a read:write mix's HBM limit"""
    _require_cuda(src)
    if out is None:
        out = torch.empty(max(int(out_bytes), 16), dtype=torch.uint8, device=src.device)
    _check(_lib.exmy_debug_probe(_ptr(src), src.numel() * src.element_size(), _ptr(out), int(out_bytes),
                                 _stream(src.device)), "roofline_probe")
    return out


def enc_tma(on: bool | None = None) -> int:
    """knob: ROWS encode through the TMA-staged kernel (1) or the register
    pipeline (0); returns the previous setting"""
    return _lib.exmy_debug_enc_tma(-1 if on is None else int(on))


def gemv_bulk(on: bool | None = None) -> int:
    """knob: gemv with bulk-staged packed bytes (1, cols % 16 == 0) or the
    register-pipelined kernel (0); returns the previous setting"""
    return _lib.exmy_debug_gemv_bulk(-1 if on is None else int(on))


def rowwise_cluster(on: bool | None = None) -> int:
    """knob: wide-row encode_rowwise on thread-block clusters (1) or the
    two-pass paths (0); returns the previous setting"""
    return _lib.exmy_debug_rowwise_cluster(-1 if on is None else int(on))


def hist_blocks(blocks: int | None = None) -> int:
    """test knob: cap the histogram grid (0 = auto); returns the previous cap"""
    return _lib.exmy_debug_hist_blocks(-1 if blocks is None else int(blocks))


def _check(status: int, what: str):
    if status != 0:
        raise ExmyError(status, what)


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _dtype_code(dt) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.bfloat16:
        return BF16
    raise TypeError(f"eXmY codec takes float32 or bfloat16 tensors, got {dt}")


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tensor must live on a CUDA device (no CPU fallback)")


def _meta_tensor(meta, device) -> torch.Tensor:
    if isinstance(meta, torch.Tensor):
        if meta.dtype != torch.uint8 or meta.numel() != 1:
            raise TypeError("meta must be a uint8 tensor with one element")
        return meta.to(device) if meta.device != torch.device(device) else meta
    e = int(meta)
    if not 0 <= e <= 254:
        raise ValueError("e_max must be in [0, 254] (D4)")
    return torch.tensor([e], dtype=torch.uint8, device=device)


def _as_2d(t: torch.Tensor):
    if t.dim() == 0:
        raise ValueError("scalar tensor")
    if t.dim() == 1:
        return 1, t.shape[0]
    return t.numel() // t.shape[-1], t.shape[-1]


# ---------------------------------------------------------------- device ops
def histogram(t: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exponent histogram: int64[256] (uint64 semantics) on t.device.
    ``out`` is accumulated into when given."""
    _require_cuda(t)
    t = t.contiguous()
    if out is None:
        out = torch.zeros(256, dtype=torch.int64, device=t.device)
    _check(_lib.exmy_exponent_histogram(_ptr(t), _dtype_code(t.dtype), t.numel(), _ptr(out), _stream(t.device)),
           "exponent_histogram")
    return out


def emax(hist: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device metadata byte: top populated histogram bin in [0,254]."""
    _require_cuda(hist)
    if out is None:
        out = torch.empty(1, dtype=torch.uint8, device=hist.device)
    _check(_lib.exmy_emax_from_histogram(_ptr(hist), _ptr(out), _stream(hist.device)), "emax_from_histogram")
    return out


def max_exponent(t: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-tensor metadata of t (max biased exponent): one
    read-only reduction (falls back to histogram + e_max for unaligned t)."""
    _require_cuda(t)
    t = t.contiguous()
    if out is None:
        out = torch.empty(1, dtype=torch.uint8, device=t.device)
    s = _lib.exmy_max_exponent(_ptr(t), _dtype_code(t.dtype), t.numel(), _ptr(out), _stream(t.device))
    if s == 5:   # E_ALIGN
        return emax(histogram(t), out=out)
    _check(s, "max_exponent")
    return out


def quantize(t: torch.Tensor, fmt, meta=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Emulation: nearest eXmY grid value in t's dtype; NaN/Inf kept."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    t = t.contiguous()
    m = max_exponent(t) if meta is None else _meta_tensor(meta, t.device)
    if out is None:
        out = torch.empty_like(t)
    _check(_lib.exmy_quantize(_ptr(t), _ptr(out), _dtype_code(t.dtype), t.numel(), x, y, _ptr(m), _stream(t.device)),
           "quantize")
    return out


@dataclass
class Packed:
    """Packed eXmY tensor: segments of the power-of-2 decomposition."""
    data: torch.Tensor        # uint8[n*k/8]
    meta: torch.Tensor        # uint8[1] device: max biased exponent
    sp_index: torch.Tensor    # int64[capacity]
    sp_bits: torch.Tensor     # int32[capacity] (fp32 bit patterns)
    sp_count: torch.Tensor    # int64[1] device (uint64 semantics)
    shape: tuple
    x: int
    y: int
    axis: int
    dtype: torch.dtype        # source dtype
    block: tuple | None = None   # (block_rows, block_cols) when meta is per block
    layout: tuple | None = None  # (rows, cols) packed when not the 2-D view of shape (grouped 1-D tensors)
    scale: torch.Tensor | None = None   # float-scaling metadata: per-block fp32 amax (reading D23)
    sp_capacity: int | None = None   # specials capacity the encode ran with (entries written); None: sp_index.numel()
    scheme: int = 0              # block metadata scheme: 0 max-before, 1 max-after, 2 float scaling

    @property
    def capacity(self) -> int:
        """entries the encode could write: decode scatters min(count, capacity)"""
        return self.sp_index.numel() if self.sp_capacity is None else int(self.sp_capacity)

    @property
    def k(self) -> int:
        return 1 + self.x + self.y

    @property
    def rows(self) -> int:
        return (self.layout or _as_2d_shape(self.shape))[0]

    @property
    def cols(self) -> int:
        return (self.layout or _as_2d_shape(self.shape))[1]

    def segments(self):
        """[(width, uint8 view)] in decomposition order."""
        n = self.rows * self.cols
        ws, offs = segments(self.k, n)
        return [(w, self.data[o:o + n * w // 8]) for w, o in zip(ws, offs)]

    def specials(self):
        """(index, bits, total count) of the out-of-band NaN/Inf (D9); the lists
        hold min(count, capacity) entries."""
        cnt = int(self.sp_count[0].item()) if self.sp_count is not None else 0
        c = min(cnt, self.capacity)
        return self.sp_index[:c], self.sp_bits[:c], cnt

    def check_specials(self):
        """Raise E_CAPACITY if the encode saw more NaN/Inf than its specials
        capacity (the extra ones would decode as their in-band code 0).
        Synchronises the stream."""
        cnt = int(self.sp_count[0].item()) if self.sp_count is not None else 0
        if cnt > self.capacity:
            raise ExmyError(6, f"encode: {cnt} NaN/Inf elements but specials capacity {self.capacity}; "
                               f"re-encode with specials_capacity >= {cnt}")
        return self


def _as_2d_shape(shape):
    if len(shape) == 1:
        return 1, shape[0]
    r = 1
    for s in shape[:-1]:
        r *= s
    return r, shape[-1]


def encode(t: torch.Tensor, fmt, meta=None, axis="rows", specials_capacity: int = 4096,
           out: torch.Tensor | None = None, strict: bool = True) -> Packed:
    """Type conversion + power-of-2 bit packing.  meta=None derives
    the per-tensor max biased exponent.  strict: synchronise and
    raise E_CAPACITY when the tensor holds more NaN/Inf than
    specials_capacity (strict=False keeps the call asynchronous; check later
    with Packed.check_specials())."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    ax = _AXES[axis]
    t = t.contiguous()
    R, C = _as_2d(t)
    dev = t.device
    m = max_exponent(t) if meta is None else _meta_tensor(meta, dev)
    n = R * C
    k = 1 + x + y
    if out is None:
        out = torch.empty(n * k // 8 if n % 8 == 0 else 0, dtype=torch.uint8, device=dev)
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode(_ptr(t), _dtype_code(t.dtype), R, C, ax, x, y, _ptr(m), _ptr(out), _ptr(spi), _ptr(spb),
                            _ptr(spc), cap, _stream(dev)), "encode")
    return _finish(Packed(out, m, spi, spb, spc, tuple(t.shape), x, y, ax, t.dtype, sp_capacity=cap), strict)


def _finish(p: Packed, strict: bool) -> Packed:
    return p.check_specials() if strict else p


def decode(p: Packed, dtype: torch.dtype | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Unpack + dequantize; RTNE to ``dtype`` (default: source dtype)."""
    dtype = p.dtype if dtype is None else dtype
    dev = p.data.device
    R, C = p.rows, p.cols
    if out is None:
        out = torch.empty(p.shape, dtype=dtype, device=dev)
    cap = p.capacity if p.sp_count is not None else 0
    if p.scale is not None:
        _check(_lib.exmy_decode_fs(_ptr(p.data), R, C, p.axis, p.block[0], p.block[1], p.x, p.y, _ptr(p.scale),
                                   _ptr(p.sp_index), _ptr(p.sp_bits), _ptr(p.sp_count), cap, _ptr(out),
                                   _dtype_code(dtype), _stream(dev)), "decode_fs")
        return out
    if p.block is not None:
        _check(_lib.exmy_decode_blocked(_ptr(p.data), R, C, p.axis, p.block[0], p.block[1], p.x, p.y, _ptr(p.meta),
                                        _ptr(p.sp_index), _ptr(p.sp_bits), _ptr(p.sp_count), cap, _ptr(out),
                                        _dtype_code(dtype), _stream(dev)), "decode_blocked")
        return out
    _check(_lib.exmy_decode(_ptr(p.data), R, C, p.axis, p.x, p.y, _ptr(p.meta), _ptr(p.sp_index), _ptr(p.sp_bits),
                            _ptr(p.sp_count), cap, _ptr(out), _dtype_code(dtype), _stream(dev)), "decode")
    return out


# ------------------------------------------------------------ block metadata
SCHEMES = {"before": 0, "max-before": 0, "after": 1, "max-after": 1, 0: 0, 1: 1}


def block_shape(shape, block):
    """'tensor' | 'row' | 'col' | ('subrow', L) | (br, bc) -> (br, bc)."""
    R, C = _as_2d_shape(tuple(shape))
    if block == "tensor":
        return R, C
    if block == "row":
        return 1, C
    if block in ("col", "column"):
        return R, 1
    if isinstance(block, tuple) and len(block) == 2 and block[0] == "subrow":
        return 1, int(block[1])
    return int(block[0]), int(block[1])


def block_max_exponent(t: torch.Tensor, block, y: int = 0, scheme="before", out: torch.Tensor | None = None):
    """Per-block metadata: max biased exponent before / after rounding to y
    mantissa bits.  Returns uint8 (R/br, C/bc)."""
    _require_cuda(t)
    t = t.contiguous()
    R, C = _as_2d(t)
    br, bc = block_shape(t.shape, block)
    if out is None:
        out = torch.empty((R // br if br else 0, C // bc if bc else 0), dtype=torch.uint8, device=t.device)
    _check(_lib.exmy_block_max_exponent(_ptr(t), _dtype_code(t.dtype), R, C, br, bc, int(y), SCHEMES[scheme],
                                        _ptr(out), _stream(t.device)), "block_max_exponent")
    return out


def quantize_blocked(t: torch.Tensor, fmt, meta: torch.Tensor, block, out: torch.Tensor | None = None):
    _require_cuda(t)
    x, y = parse_format(fmt)
    t = t.contiguous()
    R, C = _as_2d(t)
    br, bc = block_shape(t.shape, block)
    if out is None:
        out = torch.empty_like(t)
    _check(_lib.exmy_quantize_blocked(_ptr(t), _ptr(out), _dtype_code(t.dtype), R, C, br, bc, x, y,
                                      _ptr(meta.contiguous()), _stream(t.device)), "quantize_blocked")
    return out


def encode_blocked(t: torch.Tensor, fmt, meta: torch.Tensor | None, block, axis="rows", scheme="before",
                   specials_capacity: int = 4096, out: torch.Tensor | None = None, strict: bool = True) -> Packed:
    """Encode with one metadata byte per block; meta=None computes it with
    the given scheme."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    ax = _AXES[axis]
    t = t.contiguous()
    R, C = _as_2d(t)
    br, bc = block_shape(t.shape, block)
    dev = t.device
    if meta is None:
        meta = block_max_exponent(t, (br, bc), y, scheme)
    meta = meta.contiguous()
    n = R * C
    k = 1 + x + y
    if out is None:
        out = torch.empty(n * k // 8 if n % 8 == 0 else 0, dtype=torch.uint8, device=dev)
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode_blocked(_ptr(t), _dtype_code(t.dtype), R, C, ax, br, bc, x, y, _ptr(meta), _ptr(out),
                                    _ptr(spi), _ptr(spb), _ptr(spc), cap, _stream(dev)), "encode_blocked")
    return _finish(Packed(out, meta, spi, spb, spc, tuple(t.shape), x, y, ax, t.dtype, (br, bc), sp_capacity=cap,
                          scheme=SCHEMES[scheme]), strict)


def encode_rowwise(t: torch.Tensor, fmt, axis="rows", scheme="before", specials_capacity: int = 4096,
                   out: torch.Tensor | None = None, meta_out: torch.Tensor | None = None,
                   strict: bool = True) -> Packed:
    """Per-row metadata + encode in one call (fused single-pass kernel for ROWS)."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    ax = _AXES[axis]
    t = t.contiguous()
    R, C = _as_2d(t)
    dev = t.device
    n = R * C
    k = 1 + x + y
    if out is None:
        out = torch.empty(n * k // 8 if n % 8 == 0 else 0, dtype=torch.uint8, device=dev)
    meta = meta_out if meta_out is not None else torch.empty((R, 1), dtype=torch.uint8, device=dev)
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode_rowwise(_ptr(t), _dtype_code(t.dtype), R, C, ax, x, y, SCHEMES[scheme], _ptr(meta),
                                    _ptr(out), _ptr(spi), _ptr(spb), _ptr(spc), cap, _stream(dev)), "encode_rowwise")
    return _finish(Packed(out, meta, spi, spb, spc, tuple(t.shape), x, y, ax, t.dtype, (1, C), sp_capacity=cap,
                          scheme=SCHEMES[scheme]), strict)


def _check_indices(idx: torch.Tensor, rows: int, what: str):
    """host-side validation (synchronises): every row index in [0, rows)"""
    if idx.numel():
        lo, hi = torch.aminmax(idx)
        lo, hi = int(lo), int(hi)
        if lo < 0 or hi >= rows:
            raise IndexError(f"{what}: row index out of range [0, {rows}): min {lo}, max {hi}")


def decode_rows(p: Packed, row_index: torch.Tensor, dtype: torch.dtype | None = None,
                out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """Gather-decode rows of a COLS-packed tensor (embedding lookup).
    check: validate the indices first (one host sync; check=False for
    graph capture with trusted indices)."""
    if p.axis != COLS:
        raise ValueError("row gather needs the COLS layout (rows are contiguous byte ranges)")
    dtype = p.dtype if dtype is None else dtype
    idx = row_index.to(device=p.data.device, dtype=torch.int64).contiguous()
    if check:
        _check_indices(idx, p.rows, "decode_rows")
    if out is None:
        out = torch.empty((idx.numel(), p.cols), dtype=dtype, device=p.data.device)
    per_row = 0
    if p.block is not None:
        if p.block != (1, p.cols):
            raise ValueError("gather supports per-tensor or per-row metadata")
        per_row = 1
    _check(_lib.exmy_decode_rows(_ptr(p.data), p.rows, p.cols, p.x, p.y, _ptr(p.meta), per_row, _ptr(idx), idx.numel(),
                                 _ptr(out), _dtype_code(dtype), _stream(p.data.device)), "decode_rows")
    return out


def gemv(p: Packed, act: torch.Tensor, out: torch.Tensor | None = None, specials: bool = True) -> torch.Tensor:
    """Decode fused into a matrix-vector product (reading D26): fp32
    act (m, cols) @ W.T for the ROWS-packed W (rows, cols) -> fp32 (m, rows);
    the decoded weights never reach HBM.  specials: apply the encode's
    NaN/Inf list (the placeholder codes decode to 0)."""
    if p.axis != ROWS:
        raise ValueError("gemv needs the ROWS layout")
    dev = p.data.device
    a = act.to(device=dev, dtype=torch.float32)
    if a.dim() == 1:
        a = a.unsqueeze(0)
    a = a.contiguous()
    if a.dim() != 2 or a.shape[1] != p.cols:
        raise ValueError(f"gemv: act must be (m, {p.cols})")
    per_row = 0
    if p.block is not None:
        if p.block != (1, p.cols) or p.scheme == 2:
            raise ValueError("gemv supports per-tensor or per-row exponent metadata")
        per_row = 1
    if out is None:
        out = torch.empty((a.shape[0], p.rows), dtype=torch.float32, device=dev)
    cap = p.capacity if specials else 0
    _check(_lib.exmy_gemv(_ptr(p.data), p.rows, p.cols, p.x, p.y, _ptr(p.meta), per_row, _ptr(p.sp_index),
                          _ptr(p.sp_bits), _ptr(p.sp_count), cap, _ptr(a), a.shape[0], _ptr(out), _stream(dev)), "gemv")
    return out


def embedding_bag(p: Packed, indices: torch.Tensor, offsets: torch.Tensor, per_sample_weights=None, mode="sum",
                  out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """Pooled decode of rows of a COLS-packed table (reading D25): fp32
    (nbags, cols), like torch.nn.functional.embedding_bag with offsets of
    length nbags + 1; the decoded rows never reach HBM."""
    if p.axis != COLS:
        raise ValueError("embedding_bag needs the COLS layout (rows are contiguous byte ranges)")
    dev = p.data.device
    idx = indices.to(device=dev, dtype=torch.int64).contiguous()
    off = offsets.to(device=dev, dtype=torch.int64).contiguous()
    nb = off.numel() - 1
    if nb < 0:
        raise ValueError("offsets needs nbags + 1 entries")
    if check:
        _check_indices(idx, p.rows, "embedding_bag")
        if nb > 0:
            o = off.cpu()
            if int(o[0]) != 0 or int(o[-1]) != idx.numel() or bool((o[1:] < o[:-1]).any()):
                raise ValueError("embedding_bag offsets must start at 0, be non-decreasing and end at len(indices)")
    w = None if per_sample_weights is None else per_sample_weights.to(device=dev, dtype=torch.float32).contiguous()
    per_row = 0
    if p.block is not None:
        if p.block != (1, p.cols):
            raise ValueError("embedding_bag supports per-tensor or per-row metadata")
        per_row = 1
    if out is None:
        out = torch.empty((nb, p.cols), dtype=torch.float32, device=dev)
    _check(_lib.exmy_embedding_bag(_ptr(p.data), p.rows, p.cols, p.x, p.y, _ptr(p.meta), per_row, _ptr(idx), _ptr(off),
                                   nb, _ptr(w), {"sum": 0, "mean": 1}[mode], _ptr(out), _stream(dev)), "embedding_bag")
    return out


def decode_raw(data: torch.Tensor, rows: int, cols: int, fmt, meta, axis="rows", dtype=torch.bfloat16,
               out: torch.Tensor | None = None, specials=None) -> torch.Tensor:
    """Decode bare packed bytes (e.g. one row shard).  specials:
    optional (sp_index, sp_bits, sp_count, capacity) of this (rows, cols)
    tensor, restored after the decode (D9)."""
    x, y = parse_format(fmt)
    dev = data.device
    m = _meta_tensor(meta, dev)
    if out is None:
        out = torch.empty((rows, cols), dtype=dtype, device=dev)
    spi = spb = spc = None
    cap = 0
    if specials is not None:
        spi, spb, spc, cap = specials
    _check(_lib.exmy_decode(_ptr(data), rows, cols, _AXES[axis], x, y, _ptr(m), _ptr(spi), _ptr(spb), _ptr(spc),
                            int(cap), _ptr(out), _dtype_code(dtype), _stream(dev)), "decode")
    return out


# ----------------------------------------------- fused encode + all-gather
def encode_push(shard: torch.Tensor, fmt, meta: torch.Tensor, row0: int, total_rows: int, dsts,
                specials_capacity: int = 4096):
    """Encode the row shard [row0, row0+rows) of a (total_rows, cols) tensor and
    store its packed bytes, at their global offsets, into every buffer of
    ``dsts`` (device uint8 tensors or raw device pointers of
    total_rows*cols*k/8 bytes; peers' buffers on a multi-GPU node).  Returns
    (sp_index, sp_bits, sp_count) of the shard's specials (global indices)."""
    _require_cuda(shard)
    x, y = parse_format(fmt)
    shard = shard.contiguous()
    R, C = _as_2d(shard)
    ptrs = (ctypes.c_void_p * len(dsts))(*[d.data_ptr() if isinstance(d, torch.Tensor) else int(d) for d in dsts])
    dev = shard.device
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode_push(_ptr(shard), _dtype_code(shard.dtype), R, C, int(row0), int(total_rows), x, y,
                                 _ptr(_meta_tensor(meta, dev)), ptrs, len(dsts), _ptr(spi), _ptr(spb), _ptr(spc), cap,
                                 _stream(dev)), "encode_push")
    return spi, spb, spc


def encode_push_multicast(shard: torch.Tensor, fmt, meta: torch.Tensor, row0: int, total_rows: int, mc_ptr: int,
                          specials_capacity: int = 4096):
    """encode_push with ONE destination: a multicast address (NVLS,
    multimem.st) of the gathered buffer bound on every GPU -- each store
    reaches all of them.  Returns the shard's (sp_index, sp_bits, sp_count)."""
    _require_cuda(shard)
    x, y = parse_format(fmt)
    shard = shard.contiguous()
    R, C = _as_2d(shard)
    dev = shard.device
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode_push_multicast(_ptr(shard), _dtype_code(shard.dtype), R, C, int(row0), int(total_rows), x,
                                           y, _ptr(_meta_tensor(meta, dev)), ctypes.c_void_p(int(mc_ptr)), _ptr(spi),
                                           _ptr(spb), _ptr(spc), cap, _stream(dev)), "encode_push_multicast")
    return spi, spb, spc


def decode_pull(srcs, shard_rows: int, cols: int, fmt, meta, dtype=torch.bfloat16, out: torch.Tensor | None = None,
                device=None):
    """Decode the (len(srcs) * shard_rows, cols) tensor whose row shard s is the
    packed tensor at srcs[s] (device uint8 tensors or raw device pointers, e.g.
    peers' buffers mapped over NVLink): the all-gather happens in the loads."""
    x, y = parse_format(fmt)
    first = next((s_ for s_ in srcs if isinstance(s_, torch.Tensor)), None)
    dev = torch.device(device) if device is not None else (first.device if first is not None else torch.device("cuda"))
    ptrs = (ctypes.c_void_p * len(srcs))(*[s_.data_ptr() if isinstance(s_, torch.Tensor) else int(s_) for s_ in srcs])
    if out is None:
        out = torch.empty((len(srcs) * shard_rows, cols), dtype=dtype, device=dev)
    _check(_lib.exmy_decode_pull(ptrs, len(srcs), shard_rows, cols, x, y, _ptr(_meta_tensor(meta, dev)), _ptr(out),
                                 _dtype_code(out.dtype), _stream(dev)), "decode_pull")
    return out


# ------------------------------------------------------------ float scaling
def block_float_scale(t: torch.Tensor, block, out: torch.Tensor | None = None) -> torch.Tensor:
    """Float-scaling metadata (Fig. 2's third scheme, reading D23): per block
    the largest finite magnitude, fp32, shape (R/br, C/bc)."""
    _require_cuda(t)
    t = t.contiguous()
    R, C = _as_2d(t)
    br, bc = block_shape((R, C), block)
    if out is None:
        out = torch.empty((R // br, C // bc), dtype=torch.float32, device=t.device)
    _check(_lib.exmy_block_float_scale(_ptr(t), _dtype_code(t.dtype), R, C, br, bc, _ptr(out), _stream(t.device)),
           "block_float_scale")
    return out


def quantize_fs(t: torch.Tensor, fmt, scale: torch.Tensor | None, block, out: torch.Tensor | None = None):
    """Float-scaled emulation: decode(encode(t)) in t's dtype (scale=None:
    derived with block_float_scale)."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    t = t.contiguous()
    R, C = _as_2d(t)
    br, bc = block_shape((R, C), block)
    if scale is None:
        scale = block_float_scale(t, (br, bc))
    if out is None:
        out = torch.empty_like(t)
    _check(_lib.exmy_quantize_fs(_ptr(t), _ptr(out), _dtype_code(t.dtype), R, C, br, bc, x, y, _ptr(scale),
                                 _stream(t.device)), "quantize_fs")
    return out


def encode_fs(t: torch.Tensor, fmt, scale: torch.Tensor | None, block, axis="rows", specials_capacity: int = 4096,
              out: torch.Tensor | None = None, strict: bool = True) -> Packed:
    """Encode with float-scaling metadata (reading D23); Packed.scale holds it."""
    _require_cuda(t)
    x, y = parse_format(fmt)
    ax = _AXES[axis]
    t = t.contiguous()
    R, C = _as_2d(t)
    dev = t.device
    br, bc = block_shape((R, C), block)
    if scale is None:
        scale = block_float_scale(t, (br, bc))
    n = R * C
    if out is None:
        out = torch.empty(n * (1 + x + y) // 8 if n % 8 == 0 else 0, dtype=torch.uint8, device=dev)
    cap = int(specials_capacity)
    spi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    spb = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    spc = specials_workspace(dev)
    _check(_lib.exmy_encode_fs(_ptr(t), _dtype_code(t.dtype), R, C, ax, br, bc, x, y, _ptr(scale), _ptr(out),
                               _ptr(spi), _ptr(spb), _ptr(spc), cap, _stream(dev)), "encode_fs")
    meta = torch.full((1,), 127, dtype=torch.uint8, device=dev)
    return _finish(Packed(out, meta, spi, spb, spc, tuple(t.shape), x, y, ax, t.dtype, (br, bc), None, scale,
                          sp_capacity=cap, scheme=2), strict)


# ------------------------------------------------------- host-buffer path
class HostCodec:
    """End-to-end codec for host tensors (pinned): H2D -> histogram -> e_max ->
    encode -> D2H, all inside the C ABI (exmy_encode_host / exmy_decode_host).
    Device scratch is allocated once here (the library itself never allocates)."""

    def __init__(self, shape, dtype, fmt, axis="rows", device="cuda", specials_capacity: int = 4096):
        self.x, self.y = parse_format(fmt)
        self.R, self.C = _as_2d_shape(tuple(shape))
        self.shape = tuple(shape)
        self.dtype = dtype
        self.axis = _AXES[axis]
        self.device = torch.device(device)
        n = self.R * self.C
        self.nbytes_packed = n * (1 + self.x + self.y) // 8
        self.dev_in = torch.empty(self.shape, dtype=dtype, device=device)
        self.dev_hist = torch.zeros(256, dtype=torch.int64, device=device)
        self.dev_meta = torch.zeros(1, dtype=torch.uint8, device=device)
        self.dev_packed = torch.empty(self.nbytes_packed, dtype=torch.uint8, device=device)
        self.dev_out = torch.empty(self.shape, dtype=dtype, device=device)
        self.cap = specials_capacity
        self.spi = torch.empty(max(self.cap, 1), dtype=torch.int64, device=device)
        self.spb = torch.empty(max(self.cap, 1), dtype=torch.int32, device=device)
        self.spc = specials_workspace(device)

    def encode(self, host_in: torch.Tensor, host_packed: torch.Tensor, host_meta: torch.Tensor | None = None):
        _check(_lib.exmy_encode_host(_ptr(host_in), _dtype_code(self.dtype), self.R, self.C, self.axis, self.x,
                                     self.y, _ptr(self.dev_in), _ptr(self.dev_hist), _ptr(self.dev_meta),
                                     _ptr(self.dev_packed), _ptr(self.spi), _ptr(self.spb), _ptr(self.spc), self.cap,
                                     _ptr(host_packed), _ptr(host_meta), _stream(self.device)), "encode_host")

    def decode(self, host_packed: torch.Tensor, host_out: torch.Tensor):
        _check(_lib.exmy_decode_host(_ptr(host_packed), self.R, self.C, self.axis, self.x, self.y, _ptr(self.dev_meta),
                                     _ptr(self.spi), _ptr(self.spb), _ptr(self.spc), self.cap, _ptr(self.dev_packed),
                                     _ptr(self.dev_out), _dtype_code(self.dtype), _ptr(host_out),
                                     _stream(self.device)), "decode_host")


# ------------------------------------------------- grouped launch (tensor table)
class _GroupEntry(ctypes.Structure):
    """exmy_group_entry (include/exmy.h)"""
    _fields_ = [("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("packed", ctypes.c_void_p),
                ("meta", ctypes.c_void_p), ("sp_index", ctypes.c_void_p), ("sp_bits", ctypes.c_void_p),
                ("sp_count", ctypes.c_void_p), ("sp_capacity", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64)]


def group_layout(shape) -> tuple[int, int]:
    """(rows, cols) a tensor is packed as in a group (ROWS layout): the 2-D view
    of its shape; a 1-D tensor of n elements (a norm / bias vector, no rows of
    its own) is packed as (8, n/8).  Needs rows % 8 == 0 and cols % 4 == 0."""
    shape = tuple(shape)
    if len(shape) == 1:
        return (8, shape[0] // 8) if shape[0] % 32 == 0 else (-1, -1)
    return _as_2d_shape(shape)


def group_plan(entries, dtype, fmt, out_dtype=None, per_row: bool = False) -> bytes:
    """Host plan bytes for a list of dicts with keys of exmy_group_entry
    (pointers as ints / tensors); per_row: exmy_group_plan_rows (one
    metadata byte per row).  Low-level: see GroupCodec."""
    x, y = parse_format(fmt)
    n = len(entries)
    arr = (_GroupEntry * max(n, 1))()
    for i, e in enumerate(entries):
        for f, _ in _GroupEntry._fields_:
            v = e.get(f[:-1] if f == "in_" else f, 0)
            if isinstance(v, torch.Tensor):
                v = v.data_ptr()
            setattr(arr[i], f, v or 0)
    nb = _lib.exmy_group_plan_bytes(n)
    buf = (ctypes.c_uint64 * max(1, (nb + 7) // 8))()
    fn = _lib.exmy_group_plan_rows if per_row else _lib.exmy_group_plan
    _check(fn(arr if n else None, n, _dtype_code(dtype), x, y,
              _dtype_code(out_dtype if out_dtype is not None else dtype), buf, nb), "group_plan")
    return bytes(buf)[:nb]


class GroupCodec:
    """Whole-model codec over a table of tensors: per-tensor
    metadata (max biased exponent), ROWS encode and decode of every
    tensor in a constant number of launches (exmy_group_*), bit-identical to
    exmy.encode / exmy.decode of each tensor in its group_layout.

        g = GroupCodec(weights, "e3m3")
        packed = g.encode()          # list[Packed]
        outs = g.decode()            # list[Tensor] (out_dtype, default: input dtype)

    per_row=True: one metadata byte per row of each tensor's group_layout
    (the paper's Llama recipe), bit-identical to encode_blocked /
    decode with block "row" per tensor; self.meta is then every tensor's
    row bytes back to back (self.meta_offsets[i] = tensor i's first).

    The device buffers (packed bytes, metadata, specials, outputs) are owned
    here and reused by every call; the plan is copied to the device once, so
    the calls can be captured in a CUDA graph."""

    def __init__(self, tensors, fmt, out_dtype=None, specials_capacity: int = 0, decode_outputs: bool = True,
                 per_row: bool = False):
        tensors = [t.contiguous() for t in tensors]
        if not tensors:
            raise ValueError("empty tensor table")
        _require_cuda(*tensors)
        self.x, self.y = parse_format(fmt)
        self.k = 1 + self.x + self.y
        self.dtype = tensors[0].dtype
        if any(t.dtype != self.dtype for t in tensors):
            raise TypeError("all tensors of a group share one dtype")
        self.out_dtype = self.dtype if out_dtype is None else out_dtype
        self.device = tensors[0].device
        dev = self.device
        self.tensors = tensors
        self.layouts = [group_layout(t.shape) for t in tensors]
        n = len(tensors)
        self.per_row = bool(per_row)
        offs = [0]
        for (R, C) in self.layouts:
            offs.append(offs[-1] + (max(R, 0) if self.per_row else 1))
        self.meta_offsets = offs[:-1]
        self.meta = torch.zeros(max(offs[-1], 1), dtype=torch.uint8, device=dev)
        self.packed = [torch.empty(max(R * C, 0) * self.k // 8, dtype=torch.uint8, device=dev)
                       for R, C in self.layouts]
        cap = int(specials_capacity)
        self.cap = cap
        self.spi = torch.empty((n, max(cap, 1)), dtype=torch.int64, device=dev)
        self.spb = torch.empty((n, max(cap, 1)), dtype=torch.int32, device=dev)
        self.spc = torch.zeros(n, dtype=torch.int64, device=dev)
        self.outs = [torch.empty(t.shape, dtype=self.out_dtype, device=dev) for t in tensors] if decode_outputs \
            else None
        ents = []
        for i, (t, (R, C)) in enumerate(zip(tensors, self.layouts)):
            if R < 0 or C < 0:
                raise ValueError(f"tensor {i} of shape {tuple(t.shape)}: a 1-D group member needs n % 32 == 0")
            ents.append({"in": t.data_ptr(), "out": self.outs[i].data_ptr() if self.outs else 0,
                         "packed": self.packed[i].data_ptr(), "meta": self.meta.data_ptr() + self.meta_offsets[i],
                         "sp_index": self.spi[i].data_ptr() if cap else 0,
                         "sp_bits": self.spb[i].data_ptr() if cap else 0,
                         "sp_count": self.spc[i].data_ptr(), "sp_capacity": cap, "rows": R, "cols": C})
        self.plan_host = torch.frombuffer(bytearray(group_plan(ents, self.dtype, (self.x, self.y), self.out_dtype,
                                                               self.per_row)),
                                          dtype=torch.uint8).clone()   # torch allocation: 64-byte aligned
        self.plan_dev = self.plan_host.to(dev)
        self._ph = ctypes.c_void_p(self.plan_host.data_ptr())

    def _call(self, fn, what):
        _check(fn(self._ph, _ptr(self.plan_dev), _stream(self.device)), what)

    def max_exponent(self) -> torch.Tensor:
        """meta[i] := max biased exponent of tensor i (2 launches); per-row
        plans: every row's byte (1 launch)."""
        self._call(_lib.exmy_group_max_exponent, "group_max_exponent")
        return self.meta

    def encode(self, meta: torch.Tensor | None = None) -> list:
        """Encode every tensor; meta=None derives the metadata first (per-row
        plans: in the same pass, exmy_group_encode_rowwise)."""
        if meta is None:
            if self.per_row:
                self._call(_lib.exmy_group_encode_rowwise, "group_encode_rowwise")
                return self.packed_list()
            self.max_exponent()
        else:
            self.meta.copy_(meta)
        self._call(_lib.exmy_group_encode, "group_encode")
        return self.packed_list()

    def packed_list(self) -> list:
        res = []
        for i, (t, lay) in enumerate(zip(self.tensors, self.layouts)):
            o = self.meta_offsets[i]
            if self.per_row:
                meta, block = self.meta[o:o + lay[0]].view(lay[0], 1), (1, lay[1])
            else:
                meta, block = self.meta[o:o + 1], None
            res.append(Packed(self.packed[i], meta, self.spi[i], self.spb[i], self.spc[i:i + 1],
                              tuple(t.shape), self.x, self.y, ROWS, self.dtype, block,
                              lay if t.dim() == 1 else None, sp_capacity=self.cap))
        return res

    def decode(self) -> list:
        """Decode every tensor's packed bytes into self.outs (+ specials)."""
        if self.outs is None:
            raise ValueError("GroupCodec built with decode_outputs=False")
        self._call(_lib.exmy_group_decode, "group_decode")
        return self.outs


# ------------------------------------------------------ checkpoint container
class _CkptTensor(ctypes.Structure):
    """exmy_ckpt_tensor (include/exmy.h)"""
    _fields_ = [("name", ctypes.c_char_p), ("rank", ctypes.c_int), ("dims", ctypes.c_int64 * 8),
                ("x", ctypes.c_int), ("y", ctypes.c_int), ("scheme", ctypes.c_int), ("block_kind", ctypes.c_int),
                ("block_p0", ctypes.c_int64), ("block_p1", ctypes.c_int64), ("axis", ctypes.c_int),
                ("src_dtype", ctypes.c_int), ("meta", ctypes.c_void_p), ("meta_bytes", ctypes.c_int64),
                ("packed", ctypes.c_void_p), ("packed_bytes", ctypes.c_int64), ("scale", ctypes.c_void_p),
                ("scale_bytes", ctypes.c_int64), ("sp_index", ctypes.c_void_p), ("sp_bits", ctypes.c_void_p),
                ("specials_count", ctypes.c_int64)]


def _block_kind(p: Packed):
    """(block_kind, p0, p1) of S:375 for a Packed's metadata granularity"""
    if p.block is None:
        return 0, 0, 0
    R, C = p.rows, p.cols
    br, bc = p.block
    if (br, bc) == (R, C):
        return 0, 0, 0
    if (br, bc) == (1, C):
        return 1, 0, 0
    if (br, bc) == (R, 1):
        return 2, 0, 0
    if br == 1:
        return 3, bc, 0
    return 4, br, bc


def save_checkpoint(path: str, tensors: dict) -> int:
    """Write {name: Packed} to an EXMY container (host copies of the device
    buffers); returns the file size.  Layout in include/exmy.h."""
    keep = []
    arr = (_CkptTensor * max(len(tensors), 1))()
    for i, (name, p) in enumerate(tensors.items()):
        dims = list(p.layout) if p.layout is not None else list(p.shape)
        data = p.data.detach().cpu().contiguous()
        meta = p.meta.detach().cpu().contiguous()
        scale = p.scale.detach().cpu().contiguous() if p.scale is not None else None
        cnt = int(p.sp_count[0].item()) if p.sp_count is not None else 0
        cnt = min(cnt, p.capacity) if cnt else 0
        spi = p.sp_index[:cnt].detach().cpu().contiguous() if cnt else None
        spb = p.sp_bits[:cnt].detach().cpu().contiguous() if cnt else None
        nm = name.encode()
        keep += [data, meta, scale, spi, spb, nm]
        e = arr[i]
        e.name = nm
        e.rank = len(dims)
        for d, v in enumerate(dims):
            e.dims[d] = int(v)
        e.x, e.y = p.x, p.y
        e.scheme = 2 if p.scale is not None else int(p.scheme)
        e.block_kind, e.block_p0, e.block_p1 = _block_kind(p)
        e.axis = p.axis
        e.src_dtype = _dtype_code(p.dtype)
        e.meta, e.meta_bytes = meta.data_ptr(), meta.numel()
        e.packed, e.packed_bytes = data.data_ptr(), data.numel()
        if scale is not None:
            e.scale, e.scale_bytes = scale.data_ptr(), scale.numel() * 4
        if cnt:
            e.sp_index, e.sp_bits, e.specials_count = spi.data_ptr(), spb.data_ptr(), cnt
    n = _lib.exmy_ckpt_write(path.encode(), arr, len(tensors))
    if n < 0:
        raise ExmyError(int(-n), "ckpt_write")
    return int(n)


class Checkpoint:
    """Lazy reader of an EXMY container: opening reads the manifest only;
    ``load(name)`` reads that tensor's byte ranges (pread) and moves them to
    the device; ``verify(name)`` checks its CRC32."""

    def __init__(self, path: str):
        h = ctypes.c_void_p()
        _check(_lib.exmy_ckpt_open(path.encode(), ctypes.byref(h)), "ckpt_open")
        self._h = h
        self.names = []
        for i in range(_lib.exmy_ckpt_count(h)):
            self.names.append(self.info(i).name.decode())

    def close(self):
        if self._h:
            _lib.exmy_ckpt_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _index(self, name) -> int:
        i = name if isinstance(name, int) else _lib.exmy_ckpt_find(self._h, name.encode())
        if i < 0:
            raise KeyError(name)
        return i

    def info(self, name) -> _CkptTensor:
        e = _CkptTensor()
        _check(_lib.exmy_ckpt_info(self._h, self._index(name), ctypes.byref(e)), "ckpt_info")
        return e

    @property
    def bytes_read(self) -> int:
        return int(_lib.exmy_ckpt_bytes_read(self._h))

    def verify(self, name) -> bool:
        s = _lib.exmy_ckpt_verify(self._h, self._index(name))
        if s == 11:
            return False
        _check(s, "ckpt_verify")
        return True

    def load(self, name, device="cuda") -> Packed:
        i = self._index(name)
        e = self.info(i)
        pin = torch.cuda.is_available()
        meta = torch.empty(e.meta_bytes, dtype=torch.uint8, pin_memory=pin)
        data = torch.empty(e.packed_bytes, dtype=torch.uint8, pin_memory=pin)
        scale = torch.empty(e.scale_bytes // 4, dtype=torch.float32, pin_memory=pin) if e.scale_bytes else None
        cnt = e.specials_count
        spi = torch.empty(max(cnt, 1), dtype=torch.int64)
        spb = torch.empty(max(cnt, 1), dtype=torch.int32)
        _check(_lib.exmy_ckpt_read(self._h, i, _ptr(meta), _ptr(data), _ptr(scale), _ptr(spi) if cnt else None,
                                   _ptr(spb) if cnt else None), "ckpt_read")
        dims = tuple(int(e.dims[d]) for d in range(e.rank))
        R, C = _as_2d_shape(dims)
        kind = e.block_kind
        block = {0: None, 1: (1, C), 2: (R, 1), 3: (1, int(e.block_p0)), 4: (int(e.block_p0), int(e.block_p1))}[kind]
        if scale is not None and block is None:
            block = (R, C)
        if block is not None and scale is None:
            meta = meta.reshape(R // block[0], C // block[1])
        dev = torch.device(device)
        to = (lambda t: t.to(dev, non_blocking=True) if t is not None else None)
        spc = torch.tensor([cnt], dtype=torch.int64)
        dt = torch.bfloat16 if e.src_dtype == BF16 else torch.float32
        return Packed(to(data), to(meta), to(spi), to(spb), to(spc), dims, int(e.x), int(e.y), int(e.axis), dt,
                      block, None, to(scale.reshape(R // block[0], C // block[1])) if scale is not None else None,
                      sp_capacity=cnt, scheme=int(e.scheme))
