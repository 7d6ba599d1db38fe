"""Quick K2 sanity run (used under `timeout` on the GPU box)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads
for (m, k, n, kind, lay) in [(128, 128, 256, "s32", "kn"), (128, 128, 256, "s32", "nk"), (256, 384, 1024, "s32", "kn"),
                             (1024, 1024, 4096, "requant_u8", "kn"), (300, 200, 1000, "deq_f32", "nk"),
                             (1024, 1024, 4096, "requant_u8", "nk")]:
    w, x, bias, scales = workloads.baseline_inputs(m, k, n, 0.8, 5)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    act = K.relayout_activation(x) if lay == "kn" else K.relayout_tokens(np.ascontiguousarray(x.T))
    got = K.spmm_exec(plan, act, kernel="tc").cpu().numpy()
    want = oracle.spmm_exec(sw, x, prog, bias)
    bad = np.argwhere(got != want)
    print(m, k, n, kind, lay, "mismatches", len(bad), bad[:3].tolist(), flush=True)
    if len(bad):
        i = tuple(bad[0]); print("  got", got[i], "want", want[i], flush=True)
