"""Run one config cell a few times (profiling driver; used under ncu on the GPU box).

    python tests/prof_one.py <cell> [kernel] [reps] [layout kn|nk]
cell: c5a | c5b | c5c | c3 | c1
"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c5a"
kernel = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
layout = sys.argv[4] if len(sys.argv) > 4 else "kn"
cells = {"c5a": workloads.CONFIG5[0], "c5b": workloads.CONFIG5[1], "c5c": workloads.CONFIG5[2],
         "c3": workloads.CONFIG3, "c1": workloads.CONFIG1[1]}
c = cells[name]
w, x, bias, scales = workloads.baseline_inputs(c.m, c.k, c.n, c.ratio, c.seed)
sw = P.encode_sparse(w, scales)
plan = K.plan_spmm(sw, c.n, program=workloads.program(c.program, scales), bias=bias)
act = K.relayout_activation(x) if layout == "kn" else K.relayout_tokens(np.ascontiguousarray(x.T))
out = None
for i in range(reps):
    out = K.spmm_exec(plan, act, out=out, kernel=kernel)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if os.environ.get("SI_PROF_GRAPH"):
    # the reps replayed from one CUDA graph (no host launch cost between them)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            K.spmm_exec(plan, act, out=out, kernel=kernel)
    g.replay()
    torch.cuda.synchronize()
    s.record()
    g.replay()
    e.record()
else:
    s.record()
    for i in range(reps):
        K.spmm_exec(plan, act, out=out, kernel=kernel)
    e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"{name} kernel={kernel} {ms*1e3:.1f} us  {c.ops()/ms/1e9:.1f} TOPS  {c.hbm_bytes()/ms/1e6:.1f} GB/s")
