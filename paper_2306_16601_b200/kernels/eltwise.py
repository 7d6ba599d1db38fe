"""Dense f32 auxiliary operators on the GPU (mirror of the reference's
``sparseinfer.kernels.eltwise``, eltwise.py:1-160, plus per-tensor
``quantize`` from tensor.py:140-151).

Each op is one native kernel (csrc/eltwise.cu) reached through the C ABI;
the summation orders and expression trees are the reference's, so results
match its numba kernels element for element.  Inputs and outputs are CUDA
float32 tensors; there is no CPU path.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .. import _lib
from ..tensor import DType, QuantParams


def _cuda_f32(x, name: str) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32:
        raise ValueError(f"{name} must be a CUDA float32 tensor")
    return x if x.is_contiguous() else x.contiguous()


def _stream(t: torch.Tensor):
    return torch.cuda.current_stream(t.device).cuda_stream


def softmax_f32(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Numerically-stable softmax over the last axis (eltwise.py:34-59)."""
    x = _cuda_f32(x, "x")
    if out is None:
        out = torch.empty_like(x)
    n = x.shape[-1]
    _lib.check(_lib.lib().si_softmax_rows_f32(x.data_ptr(), out.data_ptr(), x.numel() // n, n, _stream(x)),
               "softmax_f32")
    return out


def layer_norm_f32(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """Layer normalization over the last axis with affine gamma/beta
    (eltwise.py:62-99)."""
    x = _cuda_f32(x, "x")
    n = x.shape[-1]
    gamma = _cuda_f32(gamma, "gamma")
    beta = _cuda_f32(beta, "beta")
    if tuple(gamma.shape) != (n,) or tuple(beta.shape) != (n,):
        raise ValueError("gamma/beta must match the normalized axis")
    if out is None:
        out = torch.empty_like(x)
    _lib.check(_lib.lib().si_layer_norm_f32(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), float(eps),
                                            out.data_ptr(), x.numel() // n, n, _stream(x)), "layer_norm_f32")
    return out


def batch_matmul_f32(a: torch.Tensor, b: torch.Tensor, transpose_b: bool = False, alpha: float = 1.0,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched f32 matmul with a fixed accumulation order (eltwise.py:102-160).

    a: [B, M, K]; b: [B, K, N] (or [B, N, K] with transpose_b)."""
    a = _cuda_f32(a, "a")
    b = _cuda_f32(b, "b")
    if a.ndim != 3 or b.ndim != 3 or a.shape[0] != b.shape[0]:
        raise ValueError(f"bad batch matmul shapes {tuple(a.shape)} x {tuple(b.shape)}")
    bs, m, k = a.shape
    if transpose_b:
        if b.shape[2] != k:
            raise ValueError(f"inner dims differ: {tuple(a.shape)} x {tuple(b.shape)}^T")
        n = b.shape[1]
    else:
        if b.shape[1] != k:
            raise ValueError(f"inner dims differ: {tuple(a.shape)} x {tuple(b.shape)}")
        n = b.shape[2]
    if out is None:
        out = torch.empty((bs, m, n), dtype=torch.float32, device=a.device)
    bmm_strided(a, b, out, bs, 1, m, k, n, (m * k, 0, k), (b.shape[1] * b.shape[2], 0, b.shape[2]),
                (m * n, 0, n), transpose_b, alpha)
    return out


def bmm_strided(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, nb0: int, nb1: int, m: int, k: int, n: int,
                sa, sb, so, transpose_b: bool, alpha: float) -> torch.Tensor:
    """The two-level strided form of batch_matmul_f32 (si_bmm_f32): element
    strides (batch0, batch1, row) for a, b and out.  Used by the attention
    block to address (sequence, head) slices of token-major [N, H] tensors."""
    _lib.check(_lib.lib().si_bmm_f32(a.data_ptr(), b.data_ptr(), out.data_ptr(), nb0, nb1, m, k, n, *sa, *sb, *so,
                                     1 if transpose_b else 0, float(np.float32(alpha)), _stream(a)),
               "batch_matmul_f32")
    return out


def quantize_f32(x: torch.Tensor, q: QuantParams, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-tensor quantize (tensor.py:140-151): clamp(rint(f64 x / f64 scale)
    + zero_point) as u8 / s8."""
    x = _cuda_f32(x, "x")
    if q.per_channel:
        raise ValueError("quantize_f32: per-tensor params only")
    lo, hi = q.dtype.bounds
    dt = torch.int8 if q.dtype is DType.S8 else torch.uint8
    if q.dtype not in (DType.S8, DType.U8):
        raise ValueError("quantize_f32: 8-bit targets only")
    if out is None:
        out = torch.empty(x.shape, dtype=dt, device=x.device)
    _lib.check(_lib.lib().si_quantize_f32(x.data_ptr(), x.numel(), float(np.float32(q.scale)), int(q.zero_point),
                                          int(lo), int(hi), out.data_ptr(), _stream(x)), "quantize")
    return out


def attention_fused(qkv: torch.Tensor, ctx: torch.Tensor, batch: int, seq: int, heads: int, head_dim: int,
                    alpha: float) -> bool:
    """scores -> softmax -> context for every (sequence, head) in one kernel
    (si_attention_f32), bit-equal to bmm_strided(nt) + softmax_f32 +
    bmm_strided(nn).  Returns False (nothing launched) when the shape is
    outside the fused kernel's smem budget (seq > 128 or head_dim > 64)."""
    rc = _lib.lib().si_attention_f32(qkv.data_ptr(), ctx.data_ptr(), batch, seq, heads, head_dim, qkv.stride(0),
                                     ctx.stride(0), float(np.float32(alpha)), _stream(qkv))
    if rc == _lib.SI_EUNSUPPORTED:
        return False
    _lib.check(rc, "attention")
    return True


def attention_scale(head_dim: int) -> np.float32:
    """1/sqrt(d) as the f32 alpha of the scores product."""
    return np.float32(1.0 / math.sqrt(float(head_dim)))
