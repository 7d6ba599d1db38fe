"""Sparse-vs-dense INT8 table on the GPU (the paper's Table 5 analogue) over
BASELINE config 2's shapes (f32 dequant epilogue).

    python tools/dense_vs_sparse.py [N] > gpurun_out/dense_vs_sparse.md

Dense: kernels/dense.py (every weight read; same tcgen05 kernel family).
Sparse: the default AUTO path at 70/80/90% 4x1-block sparsity.  Times are
CUDA-event means over 20 back-to-back calls after 3 warm-ups.
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


def time_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    print(f"| M x K | N | dense us | dense TOPS (2MKN) | 70% us | x | 80% us | x | 90% us | x |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for (m, k) in SHAPES:
        rng = np.random.default_rng(m * 7 + k)
        x = rng.integers(0, 256, (k, n)).astype(np.uint8)
        bias = rng.integers(-1000, 1001, m).astype(np.int32)
        scales = rng.uniform(1e-4, 1e-3, m).astype(np.float32)
        prog = W.program("deq_f32", scales)
        act = K.relayout_activation(x)
        wd = rng.integers(-127, 128, (m, k)).astype(np.int8)
        dp = plan_dense_gemm(wd, n, program=prog, bias=bias)
        out = torch.empty((n, m), dtype=torch.float32, device="cuda")
        td = time_ms(lambda: dense_gemm_exec(dp, act, out=out))
        row = [f"{m}x{k}", str(n), f"{td * 1e3:.1f}", f"{2.0 * m * k * n / td / 1e9:.0f}"]
        for r in (0.7, 0.8, 0.9):
            w = P.generate_pattern_weight(m, k, r, 5)
            sp = K.plan_spmm(P.encode_sparse(w, scales), n, program=prog, bias=bias)
            ts = time_ms(lambda: K.spmm_exec(sp, act, out=out))
            row += [f"{ts * 1e3:.1f}", f"{td / ts:.2f}"]
        print("| " + " | ".join(row) + " |", flush=True)


if __name__ == "__main__":
    main()
