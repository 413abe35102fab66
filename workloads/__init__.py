"""Seeded synthetic inputs shared by the tests, the oracle runs and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
tensors with the shapes and value distributions of the paper's workloads
 and lists raw IEEE bit patterns
(NaN payloads, infinities, signed zeros, fp32 subnormals).  Both the CUDA
path and the oracle consume exactly the same tensors from here.

Distributions (P:450-471 exponent-histogram observations):
  * LLM weights  : N(0, 0.02^2) bf16 (HF initializer_range), peaked exponent
                   histogram, no exact zeros.
  * wide fp32    : N(0,1) * 2^U{-12..12} (config 1 bulk).
  * gradients    : N(0,1) * 1e-3 with 0.1 % outliers x100 (config 4).
  * Adam m / v   : N(0,1) * 1e-4 ; (N(0,1) * 1e-3)^2 with 1 % exact zeros
                   (zero-initialised state).
  * embeddings   : U(-1e-4, 1e-4) fp32 (DLRM-style init; an assumption).
"""
from __future__ import annotations

import numpy as np
import torch

# raw fp32 bit patterns of the special values the codec must carry (D9-D11)
SPECIAL_F32_BITS = [
    0x7FC00000,  # quiet NaN
    0x7F800001,  # signalling NaN, payload 1
    0xFFC12345,  # negative NaN with payload
    0x7F800000,  # +Inf
    0xFF800000,  # -Inf
    0x00000000,  # +0
    0x80000000,  # -0
    0x00000001,  # smallest fp32 subnormal
    0x807FFFFF,  # largest negative fp32 subnormal
    0x007FFFFF,  # largest fp32 subnormal
    0x7F7FFFFF,  # FLT_MAX
    0xFF7FFFFF,  # -FLT_MAX
]
SPECIAL_BF16_BITS = [0x7FC0, 0x7F81, 0xFFC1, 0x7F80, 0xFF80, 0x0000, 0x8000, 0x0001,
                     0x807F, 0x007F, 0x7F7F, 0xFF7F]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def bf16_weights(shape, seed: int = 1, std: float = 0.02, device="cpu") -> torch.Tensor:
    """LLM-weight-like bf16 tensor ~ N(0, std^2) (config 2/3)."""
    g = _gen(seed, device)
    t = torch.empty(shape, dtype=torch.bfloat16, device=device)
    t.normal_(0.0, std, generator=g)
    return t


def f32_wide(shape, seed: int = 0, device="cpu") -> torch.Tensor:
    """N(0,1) * 2^U{-12..12} fp32 (config 1 bulk)."""
    g = _gen(seed, device)
    v = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    e = torch.randint(-12, 13, shape, generator=g, device=device).to(torch.float32)
    return v * torch.exp2(e)


def f32_gradients(n: int, seed: int = 2, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    v = torch.randn(n, generator=g, device=device) * 1e-3
    mask = torch.rand(n, generator=g, device=device) < 1e-3
    return torch.where(mask, v * 100.0, v)


def f32_adam_m(n: int, seed: int = 3, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return torch.randn(n, generator=g, device=device) * 1e-4


def f32_adam_v(n: int, seed: int = 4, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    v = (torch.randn(n, generator=g, device=device) * 1e-3) ** 2
    zero = torch.rand(n, generator=g, device=device) < 1e-2
    return torch.where(zero, torch.zeros_like(v), v)


def f32_embedding(rows: int, cols: int = 128, seed: int = 5, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return (torch.rand((rows, cols), generator=g, device=device) * 2.0 - 1.0) * 1e-4


def random_bits_f32(n: int, seed: int = 7) -> np.ndarray:
    """Uniformly random fp32 bit patterns (every class incl. NaN/Inf/subnormal)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)


def random_bits_bf16(n: int, seed: int = 7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << 16, size=n, dtype=np.uint32).astype(np.uint16)


def all_bf16_bits() -> np.ndarray:
    return np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)


# Llama-3-8B parameter shapes (config 3): 291 tensors, 8,030,261,248 params.
def llama3_8b_shapes():
    shapes = [("embed_tokens", (128256, 4096))]
    for l in range(32):
        p = f"layers.{l}."
        shapes += [
            (p + "q_proj", (4096, 4096)), (p + "k_proj", (1024, 4096)),
            (p + "v_proj", (1024, 4096)), (p + "o_proj", (4096, 4096)),
            (p + "gate_proj", (14336, 4096)), (p + "up_proj", (14336, 4096)),
            (p + "down_proj", (4096, 14336)),
            (p + "input_layernorm", (4096,)), (p + "post_attention_layernorm", (4096,)),
        ]
    shapes += [("norm", (4096,)), ("lm_head", (128256, 4096))]
    return shapes


def to_bits(t: torch.Tensor) -> np.ndarray:
    """Raw bit patterns of a CPU/GPU fp32 or bf16 tensor as numpy uint32/uint16."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy().view(np.uint32)
    raise TypeError(t.dtype)


def from_bits(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32).copy()).view(torch.float32)
    raise TypeError(a.dtype)
