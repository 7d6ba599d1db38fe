"""Experiment: one weight shape under different epilogue programs (K2, graph replay)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

def timeit(plan, act, reps=20, **kw):
    out = K.spmm_exec(plan, act, kernel="tc", **kw)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            K.spmm_exec(plan, act, out=out, kernel="tc", **kw)
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for m, k, n in ((2304, 768, 8192), (768, 768, 8192), (768, 3072, 8192)):
    w, x, bias, scales = workloads.baseline_inputs(m, k, n, 0.85, 11)
    sw = P.encode_sparse(w, scales)
    act = K.relayout_tokens(np.ascontiguousarray(x.T))
    res = []
    for kind in ("s32", "deq_f32", "requant_u8"):
        plan = K.plan_spmm(sw, n, program=workloads.program(kind, scales), bias=bias)
        res.append(f"{kind} {timeit(plan, act):.1f} us")
    print(f"{m}x{k} N={n}: " + ", ".join(res), flush=True)
