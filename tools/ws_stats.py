"""Experiment: where K4's roles wait.  Runs one cell from the experiment
library (SI_LIB=.../libsi_exp.so) with per-(CTA, warp) wait-cycle counters in
mapped host memory and prints each role's share of the kernel time.

    SI_LIB=.../libsi_exp.so python tools/ws_stats.py c5b
"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
stats = torch.zeros(296 * 20 * 5, dtype=torch.int64).pin_memory()
os.environ["SI_WS_STATS"] = str(stats.data_ptr())
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c5b"
cells = {"c5a": workloads.CONFIG5[0], "c5b": workloads.CONFIG5[1]}
c = cells[name]
w, x, bias, scales = workloads.baseline_inputs(c.m, c.k, c.n, c.ratio, c.seed)
sw = P.encode_sparse(w, scales)
plan = K.plan_spmm(sw, c.n, program=workloads.program(c.program, scales), bias=bias)
act = K.relayout_tokens(np.ascontiguousarray(x.T))
for _ in range(2):
    out = K.spmm_exec(plan, act, kernel="ws")
torch.cuda.synchronize()
s = stats.numpy().reshape(296, 20, 5).astype(np.float64)
tot = s[:, :, 4]
roles = {"prod0 (w0)": ([0], ["empty", "-", "-", "-"]), "prod1 (w14)": ([14], ["empty", "-", "-", "-"]),
         "mma0 (w1, leader)": ([1], ["xfull", "tempty", "kc-loop", "issue"]), "mma1-3 (w16,18,19)": ([16, 18, 19], ["xfull", "tempty", "kc-loop", "issue"]),
         "gather (w15,17)": ([15, 17], ["landed", "rempty", "copy", "-"]),
         "epilogue (w2-13)": (list(range(2, 14)), ["tfull", "tile", "wait_read", "tmem ld"])}
for r, (warps, names) in roles.items():
    ctas = slice(0, 148, 2) if r.startswith("mma") else slice(0, 148)
    sel = s[ctas][:, warps, :]
    t = sel[:, :, 4].mean()
    print(f"{r:24s} kernel {t:9.0f} clk: " + "  ".join(f"{n} {100 * sel[:, :, i].mean() / t:5.1f}%" for i, n in enumerate(names) if n != "-"))
