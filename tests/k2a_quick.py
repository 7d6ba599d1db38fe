"""Quick K2a (W-in-TMEM kernel, spmm_tca.cu) parity + timing on the GPU box:

    SI_K2_VARIANT=tmemw python tests/k2a_quick.py [parity|time]

Parity: [K, N] and token-major [N, K] activations through kernel="tc"
against the C oracle, bit for bit (cases K2a applies to: K <= 1024, >= 2
row tiles)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
import paper_2306_16601_b200 as P  # noqa: E402
from paper_2306_16601_b200 import kernels as K, workloads  # noqa: E402

CASES = [(256, 128, 128, 0.9, "s32"), (512, 256, 100, 0.9, "s32"), (300, 208, 1000, 0.85, "s32"),
         (1024, 1024, 4096, 0.9, "requant_u8"), (768, 768, 2000, 0.9, "requant_u8"),
         (520, 272, 1500, 0.8, "deq_f32"), (768, 768, 1504, 0.8, "gelu_erf_u8"), (4096, 1024, 2240, 0.9, "s32"),
         (384, 512, 3000, 0.7, "requant_u8")]


def parity():
    nbad = 0
    for layout in ("kn", "nk"):
        for (m, k, n, ratio, kind) in CASES:
            if layout == "kn" and n % 16:
                continue   # TMA rows of [K, N] need 16-byte multiples
            w, x, bias, scales = workloads.baseline_inputs(m, k, n, ratio, 5)
            sw = P.encode_sparse(w, scales)
            prog = workloads.program(kind, scales)
            plan = K.plan_spmm(sw, n, program=prog, bias=bias)
            act = K.relayout_activation(x) if layout == "kn" else K.relayout_tokens(np.ascontiguousarray(x.T))
            try:
                got = K.spmm_exec(plan, act, kernel="tc").cpu().numpy()
            except Exception as ex:  # noqa: BLE001
                print(layout, m, k, n, ratio, kind, "ERROR", ex, flush=True)
                nbad += 1
                continue
            want = oracle.spmm_exec(sw, x, prog, bias)
            g = got.view(np.uint32) if got.dtype == np.float32 else got
            wv = want.view(np.uint32) if want.dtype == np.float32 else want
            bad = np.argwhere(g != wv)
            print(layout, m, k, n, ratio, kind, "mismatches", len(bad), bad[:3].tolist(), flush=True)
            nbad += bool(len(bad))
    return nbad


def timing(reps=20):
    for layout in ("kn", "nk"):
        for c in workloads.CONFIG5[:2]:
            w, x, bias, scales = workloads.baseline_inputs(c.m, c.k, c.n, c.ratio, c.seed)
            plan = K.plan_spmm(P.encode_sparse(w, scales), c.n, program=workloads.program(c.program, scales),
                               bias=bias)
            act = K.relayout_activation(x) if layout == "kn" else K.relayout_tokens(np.ascontiguousarray(x.T))
            out = K.spmm_exec(plan, act, kernel="tc")
            for _ in range(3):
                K.spmm_exec(plan, act, out=out, kernel="tc")
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps):
                K.spmm_exec(plan, act, out=out, kernel="tc")
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / reps
            print(f"{layout} {c.name} {ms * 1e3:.1f} us {c.ops() / ms / 1e9:.1f} TOPS", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "parity"
    rc = parity() if what == "parity" else 0
    if what == "time":
        timing()
    sys.exit(1 if rc else 0)
