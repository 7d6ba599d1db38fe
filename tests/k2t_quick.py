"""Quick K2t (X-stationary 2:4 kernel) parity + timing run on the GPU box:

    python tests/k2t_quick.py [parity|time|all]

Parity: token-major activations through kernel="tc" (K2t whenever it
applies) against the C oracle, bit for bit.  Timing: config-5 linears with
token-major X, K2t vs the dense pair kernel (SI_K2_VARIANT is read once per
process, so the pair timing runs in a subprocess).
"""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import oracle  # noqa: E402
import paper_2306_16601_b200 as P  # noqa: E402
from paper_2306_16601_b200 import kernels as K, workloads  # noqa: E402

# (M, K, N, sparsity, program): ragged M / K / N against the 256-row pair
# tiles, 128-k chunks and 224-token tiles, every epilogue form K2t compiles
CASES = [(512, 128, 224, 0.9, "s32"), (512, 256, 100, 0.9, "s32"), (300, 208, 1000, 0.85, "s32"),
         (1024, 1024, 4096, 0.9, "requant_u8"), (768, 768, 2000, 0.9, "requant_u8"),
         (520, 272, 1500, 0.8, "deq_f32"), (768, 768, 1504, 0.9, "gelu_erf_u8"), (4096, 1024, 2240, 0.9, "s32"),
         (1024, 1024, 4480, 0.9, "requant_u8"), (2048, 1024, 1792, 0.7, "requant_u8")]


def k2t_applies(plan) -> bool:
    """K2t's own conditions (spmm_tcx.cu k2t_supported) read off the plan header."""
    from helpers import image_header
    h = image_header(np.asarray(plan.image))
    return h.tr_ok == 1 and h.tc_kpad <= 1024 and h.tc_mtiles >= 2 and h.K % 16 == 0


def parity():
    nbad = 0
    forced = os.environ.get("SI_K2_VARIANT") == "xsparse"
    for (m, k, n, ratio, kind) in CASES:
        w, x, bias, scales = workloads.baseline_inputs(m, k, n, ratio, 5)
        sw = P.encode_sparse(w, scales)
        prog = workloads.program(kind, scales)
        plan = K.plan_spmm(sw, n, program=prog, bias=bias)
        if forced and not k2t_applies(plan):
            print(m, k, n, ratio, kind, "K2t does not apply (skipped)", flush=True)
            continue
        act = K.relayout_tokens(np.ascontiguousarray(x.T))
        try:
            got = K.spmm_exec(plan, act, kernel="tc").cpu().numpy()
        except Exception as ex:  # noqa: BLE001
            print(m, k, n, ratio, kind, "ERROR", ex, flush=True)
            nbad += 1
            continue
        want = oracle.spmm_exec(sw, x, prog, bias)
        g = got.view(np.uint32) if got.dtype == np.float32 else got
        wv = want.view(np.uint32) if want.dtype == np.float32 else want
        bad = np.argwhere(g != wv)
        print(m, k, n, ratio, kind, "mismatches", len(bad), bad[:3].tolist(), flush=True)
        if len(bad):
            i = tuple(bad[0])
            print("  got", got[i], "want", want[i], flush=True)
            nbad += 1
    return nbad


def timing(reps=20):
    for c in workloads.CONFIG5:
        w, x, bias, scales = workloads.baseline_inputs(c.m, c.k, c.n, c.ratio, c.seed)
        sw = P.encode_sparse(w, scales)
        plan = K.plan_spmm(sw, c.n, program=workloads.program(c.program, scales), bias=bias)
        act = K.relayout_tokens(np.ascontiguousarray(x.T))
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
        print(f"{c.name} variant={os.environ.get('SI_K2_VARIANT', 'auto')} {ms * 1e3:.1f} us "
              f"{c.ops() / ms / 1e9:.1f} TOPS {c.hbm_bytes() / ms / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    rc = 0
    if what in ("parity", "all"):
        rc = parity()
    if what in ("time", "all"):
        timing()
        if "SI_K2_VARIANT" not in os.environ:
            subprocess.run([sys.executable, __file__, "time"], env=dict(os.environ, SI_K2_VARIANT="pair"))
    sys.exit(1 if rc else 0)
