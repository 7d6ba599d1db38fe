"""Experiment: run K4 once on a 1024x1024 @90% requant cell at the given token
count and compare with the tensor-core kernel (K2)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads
n = int(sys.argv[1]); m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w, x, bias, scales = workloads.baseline_inputs(m, 1024, n, 0.9, 77)
sw = P.encode_sparse(w, scales)
plan = K.plan_spmm(sw, n, program=workloads.program("requant_u8", scales), bias=bias)
act = K.relayout_tokens(np.ascontiguousarray(x.T))
ref = K.spmm_exec(plan, act, kernel="tc")
torch.cuda.synchronize()
for _ in range(reps):
    out = K.spmm_exec(plan, act, kernel="ws")
torch.cuda.synchronize()
print(f"n={n} m={m} reps={reps}: mismatches {(out != ref).sum().item()}")
