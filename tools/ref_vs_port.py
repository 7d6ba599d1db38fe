"""The reference's own CPU path (numba ``spmm_exec`` of /root/reference, with a
thread pool) timed beside its C restatement (``oracle/si_oracle.c
orc_spmm_exec``, the bench's reference arm), on the same config-5 sample and
the same host, with the outputs compared byte for byte.  Runs only where the
reference exists (the build container); the GPU box cannot import it.

    python tools/ref_vs_port.py [tokens] > profiles/r02_ref_vs_port.md
"""
import concurrent.futures as cf
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import sparseinfer as R  # noqa: E402  (the reference, read-only)
from sparseinfer import kernels as RK  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2306_16601_b200 import workloads  # noqa: E402


class Pool:
    """The injected pool spmm_exec expects (spmm.py:328-332): run(fn, tasks)."""

    def __init__(self, n):
        self.ex = cf.ThreadPoolExecutor(n)

    def run(self, fn, tasks):
        list(self.ex.map(fn, tasks))


def best_of(fn, reps=3):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return min(t)


def main():
    tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    threads = len(os.sched_getaffinity(0))
    pool = Pool(threads)
    print(f"# r02: the reference's numba spmm_exec vs the C port (oracle) on config 5, {tokens} tokens, "
          f"{threads} host threads\n")
    print("| linear | reference numba, T=1 | reference numba, T=all | C port, T=1 | C port, T=all | outputs equal |")
    print("|---|---|---|---|---|---|")
    from paper_2306_16601_b200 import encode_sparse
    for c in workloads.CONFIG5:
        w, x, bias, scales = workloads.baseline_inputs(c.m, c.k, tokens, c.ratio, c.seed)
        sw_r = R.encode_sparse(w, scales)
        prog_r = RK.build_program(scales, 1.0, 0, R.QuantParams(np.float32(2.0), 128, R.DType.U8))
        ops = c.ops(tokens)

        def ref(t):
            plan = RK.plan_spmm(sw_r, tokens, threads=t, program=prog_r, bias=bias)
            act = RK.relayout_activation(x, plan.bn)
            return RK.spmm_exec(plan, act, pool if t > 1 else None)

        sw = encode_sparse(w, scales)
        prog = workloads.program(c.program, scales)

        def port(t):
            return oracle.spmm_exec(sw, x, prog, bias, threads=t)

        same = np.array_equal(ref(threads), port(threads))
        times = [best_of(lambda: ref(1)), best_of(lambda: ref(threads)), best_of(lambda: port(1)),
                 best_of(lambda: port(threads))]
        print(f"| {c.name} | " + " | ".join(f"{t * 1e3:.0f} ms ({ops / t / 1e9:.1f} GOPS)" for t in times)
              + f" | {same} |", flush=True)


if __name__ == "__main__":
    main()
