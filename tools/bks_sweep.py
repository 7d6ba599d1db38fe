"""Experiment: K2 pair kernel with 128-k vs 256-k stages on small and medium
token counts (experiment library, SI_K2_BKS=128|256), CUDA-graph replay."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

def timeit(plan, act, reps=20):
    out = K.spmm_exec(plan, act, kernel="tc")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            K.spmm_exec(plan, act, out=out, kernel="tc")
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

shapes = [(3072, 768, 4096, 0.8, "gelu_erf_u8"), (768, 768, 128, 0.9, "deq_f32"), (768, 768, 512, 0.9, "deq_f32"),
          (3072, 768, 512, 0.9, "deq_f32"), (768, 3072, 2048, 0.9, "deq_f32"), (1024, 1024, 2048, 0.9, "deq_f32"),
          (4096, 1024, 2048, 0.9, "deq_f32"), (4096, 1024, 8192, 0.9, "deq_f32"), (1024, 4096, 8192, 0.9, "deq_f32"),
          (1024, 1024, 8192, 0.9, "requant_u8"), (4096, 1024, 16384, 0.9, "requant_u8"), (4096, 1024, 65536, 0.9, "requant_u8")]
for m, k, n, ratio, kind in shapes:
    w, x, bias, scales = workloads.baseline_inputs(m, k, n, ratio, 11)
    sw = P.encode_sparse(w, scales)
    plan = K.plan_spmm(sw, n, program=workloads.program(kind, scales), bias=bias)
    act = K.relayout_tokens(np.ascontiguousarray(x.T))
    res = []
    for b in ("256", "128"):
        os.environ["SI_K2_BKS"] = b
        res.append(timeit(plan, act))
    print(f"{m}x{k} N={n} {kind}: 256-k {res[0]:.1f} us, 128-k {res[1]:.1f} us", flush=True)
