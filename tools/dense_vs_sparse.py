"""Sparse-vs-dense INT8 table on the GPU (the paper's Table 5 analogue,
PAPER.md:388-393) over BASELINE config 2 / config 5 shapes and N = 32..8192.

    python tools/dense_vs_sparse.py > gpurun_out/dense_vs_sparse.md

Columns (CUDA-event means over 20 back-to-back calls replayed from one CUDA
graph after 3 warm-ups; the inputs stay L2-warm across calls):
  * cuBLASLt: the vendor dense INT8 GEMM, torch._int_mm(X s8 [N, K], W^T s8
    [K, M]) -> s32 [N, M] -- a comparator only (never on the product path),
    its epilogue-free s32 output already as many bytes as our f32 output;
  * own dense: kernels/dense.py (every 4x1 block present, the same K2
    tcgen05 kernel with the dequant epilogue);
  * sparse: the product at 90% 4x1-block sparsity (AUTO, [K, N] activations,
    f32 dequant epilogue), and its speed-up over each dense column.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P  # noqa: E402
from paper_2306_16601_b200 import kernels as K, workloads as W  # noqa: E402
from paper_2306_16601_b200.kernels.dense import dense_gemm_exec, plan_dense_gemm  # noqa: E402

SHAPES = [(768, 768), (3072, 768), (768, 3072), (1024, 1024), (4096, 1024), (1024, 4096)]
NS = [32, 128, 512, 2048, 8192]


def time_ms(fn, reps=20):
    """Mean device time per call: `reps` calls captured in one CUDA graph and
    replayed (host launch cost excluded; inputs are L2-warm across calls)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    print("| M x K | N | cuBLASLt int8 us | own dense us | sparse 90% us | vs cuBLASLt | vs own dense |")
    print("|---|---|---|---|---|---|---|")
    for (m, k) in SHAPES:
        rng = np.random.default_rng(m * 7 + k)
        bias = rng.integers(-1000, 1001, m).astype(np.int32)
        scales = rng.uniform(1e-4, 1e-3, m).astype(np.float32)
        prog = W.program("deq_f32", scales)
        wd = rng.integers(-127, 128, (m, k)).astype(np.int8)
        wt = torch.from_numpy(np.ascontiguousarray(wd.T)).cuda()          # [K, M] s8
        w90 = P.generate_pattern_weight(m, k, 0.9, 5)
        sw = P.encode_sparse(w90, scales)
        for n in NS:
            x = rng.integers(0, 256, (k, n)).astype(np.uint8)
            xs8 = torch.from_numpy((x.astype(np.int16) - 128).astype(np.int8).T.copy()).cuda()   # [N, K] s8
            o32 = torch.empty((n, m), dtype=torch.int32, device="cuda")
            tv = time_ms(lambda: torch._int_mm(xs8, wt, out=o32))
            act = K.relayout_activation(x)
            dp = plan_dense_gemm(wd, n, program=prog, bias=bias)
            out = torch.empty((n, m), dtype=torch.float32, device="cuda")
            td = time_ms(lambda: dense_gemm_exec(dp, act, out=out))
            sp = K.plan_spmm(sw, n, program=prog, bias=bias)
            ts = time_ms(lambda: K.spmm_exec(sp, act, out=out))
            print(f"| {m}x{k} | {n} | {tv * 1e3:.1f} | {td * 1e3:.1f} | {ts * 1e3:.1f} | {tv / ts:.2f} | "
                  f"{td / ts:.2f} |", flush=True)


if __name__ == "__main__":
    main()
