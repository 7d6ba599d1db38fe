"""Quick K2s (2:4 sparse tensor-core) sanity run on the GPU box:

    SI_K2_VARIANT=sparse python tests/k2s_quick.py
"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

cases = [(256, 128, 192, 0.9, "s32"), (256, 128, 192, 0.5, "s32"), (200, 300, 1008, 0.8, "s32"),
         (384, 256, 2048, 0.9, "requant_u8"), (1024, 1024, 4096, 0.9, "requant_u8"),
         (300, 200, 1008, 0.8, "deq_f32"), (512, 768, 1504, 0.8, "gelu_erf_u8"), (1024, 4096, 1024, 0.9, "s32")]
for (m, k, n, ratio, kind) in cases:
    w, x, bias, scales = workloads.baseline_inputs(m, k, n, ratio, 5)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    act = K.relayout_activation(x)
    try:
        got = K.spmm_exec(plan, act, kernel="tc").cpu().numpy()
    except Exception as ex:  # noqa: BLE001
        print(m, k, n, ratio, kind, "ERROR", ex, flush=True)
        break
    want = oracle.spmm_exec(sw, x, prog, bias)
    bad = np.argwhere(got.view(np.uint8) != want.view(np.uint8)) if got.dtype == np.float32 else np.argwhere(got != want)
    print(m, k, n, ratio, kind, "mismatches", len(bad), bad[:3].tolist(), flush=True)
    if len(bad):
        i = tuple(bad[0]); print("  got", got[i], "want", want[i], flush=True)
