"""BASELINE config 2 on the GPU: every (M, K) x N x sparsity cell with the f32
dequant epilogue; effective TOPS (2*nnz*N/s) and the cell's HBM-roofline
fraction (algorithmic bytes / measured HBM bandwidth).

    python tools/config2_sweep.py [auto|gather|tc] [N,N,...] > gpurun_out/config2.md

Times are CUDA-event means over back-to-back calls replayed from one CUDA
graph after warm-up; the activation and the output stay resident (cells
below ~64 MB are L2-warm).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P  # noqa: E402
from paper_2306_16601_b200 import kernels as K, workloads as W  # noqa: E402


def main():
    kernel = sys.argv[1] if len(sys.argv) > 1 else "auto"
    ns = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else W.CONFIG2_N
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        hbm = 6650.0
    print(f"kernel={kernel}; HBM peak used for the roofline fraction: {hbm:.0f} GB/s\n")
    print("| M x K | sparsity | " + " | ".join(f"N={n} us (TOPS)" for n in ns) + " | roofline frac @max N |")
    print("|---|---|" + "---|" * (len(ns) + 1))
    cells = W.config2_cells()
    by = {}
    for c in cells:
        by.setdefault((c.m, c.k, c.ratio), []).append(c)
    for (m, k, r), cs in by.items():
        w, _, bias, scales = W.baseline_inputs(m, k, 1, r, cs[0].seed, with_x=False)
        sw = P.encode_sparse(w, scales)
        prog = W.program("deq_f32", scales)
        row = [f"{m}x{k}", f"{int(r * 100)}%"]
        frac = ""
        for c in cs:
            if c.n not in ns:
                continue
            x = np.random.default_rng(c.seed + 1).integers(0, 256, (k, c.n), dtype=np.uint8)
            plan = K.plan_spmm(sw, c.n, program=prog, bias=bias)
            act = K.relayout_activation(x)
            out = K.spmm_exec(plan, act, kernel=kernel)
            reps = 50 if c.n <= 2048 else 20
            for _ in range(3):
                K.spmm_exec(plan, act, out=out, kernel=kernel)
            torch.cuda.synchronize()
            # the calls are captured into one CUDA graph: the host's per-call
            # Python/ctypes cost (~13 us) would otherwise floor every small cell
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(reps):
                    K.spmm_exec(plan, act, out=out, kernel=kernel)
            g.replay()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / reps
            row.append(f"{ms * 1e3:.1f} ({c.ops() / ms / 1e9:.0f})")
            if c.n == max(ns):
                frac = f"{c.hbm_bytes() / (ms / 1e3) / 1e9 / hbm:.2f}"
        row.append(frac)
        print("| " + " | ".join(row) + " |", flush=True)


if __name__ == "__main__":
    main()
