"""Dense INT8 GEMM baseline on the GPU (mirror of the reference's
``sparseinfer.kernels.dense``, dense.py:1-207).

Same math and epilogue as the sparse path but reading every weight, so
sparse-vs-dense timings compare like for like.  On the GPU the dense weight
runs through the same tcgen05 kernel (K2): its plan image holds the dense
W^T tiles the sparse path also multiplies, so a dense plan is the sparse
plan of the weight with every 4x1 block present.  Results equal
``dense_gemm_s8`` of the reference bit for bit (integer MACs, int32 wrap,
the same compiled epilogue programs).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ..sparse import encode_sparse
from .epilogue import EpilogueProgram, build_program
from .spmm import DEFAULT_BN, ActivationLayout, SpmmPlan, plan_spmm, relayout_activation, spmm_exec


@dataclass(frozen=True)
class DenseGemmPlan:
    """dense.py:22-37; ``sparse_plan`` is the device plan of the dense weight."""

    m: int
    k: int
    n: int
    bn: int
    num_bn: int
    threads: int
    program: EpilogueProgram
    sparse_plan: SpmmPlan

    @property
    def groups(self) -> int:
        return -(-self.m // 4)


def plan_dense_gemm(w: np.ndarray, n: int, threads: int = 1, program: EpilogueProgram | None = None,
                    bias: np.ndarray | None = None, bn: int = DEFAULT_BN, device=None) -> DenseGemmPlan:
    """dense.py:40-70 (same validation and defaults)."""
    w = np.ascontiguousarray(w, dtype=np.int8)
    if w.ndim != 2:
        raise ValueError("weight must be 2-D")
    if n <= 0:
        raise ValueError("N must be positive")
    m, k = w.shape
    if program is None:
        program = build_program(np.ones(m, np.float32), 1.0, 0, None)
    if bias is None:
        bias = np.zeros(m, dtype=np.int32)
    bias = np.ascontiguousarray(bias, dtype=np.int32)
    sw = encode_sparse(w, np.asarray(program.scale_in, np.float32))
    plan = plan_spmm(sw, n, threads=threads, program=program, bias=bias, bn=bn, device=device)
    return DenseGemmPlan(m=m, k=k, n=n, bn=bn, num_bn=-(-n // bn), threads=threads, program=program,
                         sparse_plan=plan)


def dense_gemm_exec(plan: DenseGemmPlan, act: ActivationLayout, pool=None, sides=None, out=None,
                    kernel: str = "auto") -> torch.Tensor:
    """dense.py:156-190: run the planned dense baseline; [N, M] CUDA tensor."""
    if act.k != plan.k or act.n != plan.n or act.bn != plan.bn:
        raise ValueError("activation layout does not match the plan")
    return spmm_exec(plan.sparse_plan, act, pool=pool, sides=sides, out=out, kernel=kernel)


def dense_gemm_s8(w: np.ndarray, a, program: EpilogueProgram | None = None, bias: np.ndarray | None = None,
                  threads: int = 1, pool=None, bn: int = DEFAULT_BN, device=None) -> torch.Tensor:
    """dense.py:193-207: one-shot dense baseline over a logical [K, N] u8 activation."""
    n = a.shape[1]
    plan = plan_dense_gemm(w, n, threads, program, bias, bn, device=device)
    act = relayout_activation(a, bn, device=device)
    return dense_gemm_exec(plan, act, pool)
