"""Generate golden vectors by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``sparseinfer`` from
/root/reference/pkg/src (pure Python + numba; nothing is copied) and writes

  golden_cases.npz   small SpMM cases: inputs, encoded weight, program
                     arrays, and spmm_ref / spmm_exec outputs
  golden_pins.json   SPEC known-answer examples evaluated by the reference,
                     generate_pattern_weight digests, and sha256 digests of
                     spmm_ref outputs for BASELINE config 1 and a config-3
                     token slice (inputs regenerated from the seeds)

The GPU box never runs this script (the reference is not there); the tests
only read the committed outputs.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import sparseinfer as si  # noqa: E402
import sparseinfer.kernels as sk  # noqa: E402
from sparseinfer.tensor import DType, Granularity, QuantParams  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


class Pool:
    """The injected pool interface spmm_exec expects (spmm.py:292, 332)."""

    def __init__(self, n):
        self.ex = cf.ThreadPoolExecutor(n)

    def run(self, fn, tasks):
        list(self.ex.map(fn, tasks))


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def baseline_inputs(m, k, n, ratio, seed):
    """BASELINE.json value distributions from one seed."""
    w = si.generate_pattern_weight(m, k, ratio, seed)
    x = np.random.default_rng(seed + 1).integers(0, 256, (k, n), dtype=np.uint8)
    rng = np.random.default_rng(seed + 2)
    bias = rng.integers(-1000, 1001, m).astype(np.int32)
    scales = rng.uniform(1e-4, 1e-3, m).astype(np.float32)
    return w, x, bias, scales


def program_for(kind, scales, m, n, a_zp, rng):
    """Reference programs exercised by the golden cases."""
    side = None
    if kind == "raw":
        prog = sk.build_program(scales, 1.0, a_zp, None)
    elif kind == "deq":
        prog = sk.build_program(scales, 1.0, a_zp, None, [("dequantize_acc",)])
    elif kind == "requant_u8":
        prog = sk.build_program(scales, 1.0, a_zp, QuantParams(np.float32(2.0), 128, DType.U8))
    elif kind == "requant_s8":
        prog = sk.build_program(scales, 0.75, a_zp, QuantParams(np.float32(0.5), 0, DType.S8))
    elif kind == "gelu_u8":
        prog = sk.build_program(scales, 1.0, a_zp, None,
                                [("dequantize_acc",), ("gelu",),
                                 ("quantize", QuantParams(np.float32(0.05), 0, DType.U8))])
    elif kind == "gelu_f32":
        prog = sk.build_program(scales, 1.0, a_zp, None, [("dequantize_acc",), ("gelu",)])
    elif kind == "lut_s8":
        table = rng.integers(0, 256, 256).astype(np.uint8)
        prog = sk.build_program(scales, 1.0, a_zp, QuantParams(np.float32(1.5), 100, DType.U8),
                                [("lut", table, DType.U8, DType.S8)])
    elif kind == "side_chan_s8":
        chan = rng.normal(0, 2, m).astype(np.float32)
        side = rng.normal(0, 3, (1, n, m)).astype(np.float32)
        prog = sk.build_program(scales, 1.0, a_zp, None,
                                [("dequantize_acc",), ("add_side", 0), ("add_channel", chan),
                                 ("quantize", QuantParams(np.float32(0.1), 3, DType.S8))])
    elif kind == "requant_chain":
        prog = sk.build_program(scales, 1.0, a_zp, QuantParams(np.float32(0.5), 10, DType.U8),
                                [("dequantize", QuantParams(np.float32(0.5), 10, DType.U8)),
                                 ("gelu",),
                                 ("quantize", QuantParams(np.float32(0.02), 128, DType.U8))])
    else:
        raise KeyError(kind)
    return prog, side


PROGRAM_KINDS = ["raw", "deq", "requant_u8", "requant_s8", "gelu_u8", "gelu_f32", "lut_s8",
                 "side_chan_s8", "requant_chain"]


def make_cases():
    cases = []
    # SPEC.md:566 edge grid (M, K, N) plus mid-size shapes and degenerate weights
    shapes = [(m, k, n, 0.5) for m in (1, 3, 5, 7) for k in (1, 4, 5, 63) for n in (1, 15, 50)]
    shapes += [(16, 32, 8, 0.75), (64, 96, 70, 0.9), (33, 130, 129, 0.5), (128, 64, 200, 0.7),
               (12, 40, 33, 1.0), (12, 40, 33, 0.0), (256, 256, 64, 0.8)]
    rng = np.random.default_rng(2024)
    for ci, (m, k, n, ratio) in enumerate(shapes):
        kind = PROGRAM_KINDS[ci % len(PROGRAM_KINDS)]
        a_zp = int(rng.integers(0, 20)) if ci % 3 == 0 else 0
        cases.append(dict(m=m, k=k, n=n, ratio=ratio, seed=100 + ci, kind=kind, a_zp=a_zp))
    # every program kind on one mid-size shape, a_zp != 0
    for kind in PROGRAM_KINDS:
        cases.append(dict(m=36, k=72, n=67, ratio=0.8, seed=500, kind=kind, a_zp=5))
    return cases


def run_case(c, pool):
    rng = np.random.default_rng(c["seed"] + 7)
    w, x, bias, scales = baseline_inputs(c["m"], c["k"], c["n"], c["ratio"], c["seed"])
    sw = si.encode_sparse(w, scales)
    prog, side = program_for(c["kind"], scales, c["m"], c["n"], c["a_zp"], rng)
    ref = sk.spmm_ref(sw, x, prog, bias, side)
    out = {}
    for threads in (1, 4):
        plan = sk.plan_spmm(sw, c["n"], threads=threads, program=prog, bias=bias)
        act = sk.relayout_activation(x)
        out[threads] = sk.spmm_exec(plan, act, pool if threads > 1 else None, side)
    return w, x, bias, scales, sw, prog, side, ref, out


def extreme_case():
    """255 activations against -128 weights: the dot4 extreme."""
    m, k, n = 8, 64, 16
    w = np.full((m, k), -128, np.int8)
    w[:, ::3] = 127
    x = np.full((k, n), 255, np.uint8)
    bias = np.array([2**31 - 1 - 10**6, -(2**31) + 10**6] * 4, np.int32)
    scales = np.full(m, 1e-3, np.float32)
    return w, x, bias, scales


def main():
    pool = Pool(4)
    arrays = {}
    meta = []
    for ci, c in enumerate(make_cases()):
        w, x, bias, scales, sw, prog, side, ref, out = run_case(c, pool)
        assert np.array_equal(ref, out[1]) and np.array_equal(ref, out[4]), c
        pre = f"c{ci}_"
        arrays[pre + "w"] = w
        arrays[pre + "x"] = x
        arrays[pre + "bias"] = bias
        arrays[pre + "scales"] = scales
        for f in ("group_ptr", "idx", "vals", "nnz"):
            arrays[pre + f] = getattr(sw, f)
        arrays[pre + "comp"] = sw.row_sums()
        for f in ("scale_in", "ops", "fparams", "iparams", "luts", "chans"):
            arrays[pre + "p_" + f] = getattr(prog, f)
        if side is not None:
            arrays[pre + "side"] = side
        arrays[pre + "ref"] = ref
        meta.append(dict(c, rows=sw.rows, out_dtype=prog.out_dtype.value, a_zp=prog.a_zp,
                         n_sides=prog.n_sides, has_side=side is not None))
    # extreme-value case, raw s32 (the only output comparable near int32 limits)
    w, x, bias, scales = extreme_case()
    sw = si.encode_sparse(w, scales)
    prog = sk.raw_program(sw)
    arrays["extreme_w"] = w
    arrays["extreme_x"] = x
    arrays["extreme_bias"] = bias
    arrays["extreme_ref"] = sk.spmm_ref(sw, x, prog, bias)
    np.savez_compressed(os.path.join(HERE, "golden_cases.npz"), **arrays)
    with open(os.path.join(HERE, "golden_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)

    pins = {}
    # SPEC known-answer examples
    pins["dot4"] = [sk.dot4_accum([1, 2, 3, 4], [1, 1, 1, 1], 0),
                    sk.dot4_accum([255] * 4, [-128] * 4, 0)]
    q = si.compute_quant_params(np.array([-1.0, 3.0], np.float32), Granularity.PER_TENSOR, DType.U8)
    pins["calib_u8"] = [float(q.scale), q.zero_point]
    q2 = si.compute_quant_params(np.array([0, 0, 0, 0], np.float32), Granularity.PER_TENSOR, DType.S8)
    pins["calib_zero_s8"] = [float(q2.scale), q2.zero_point]
    q3 = si.compute_quant_params(np.linspace(-63.5, 63.5, 11).astype(np.float32),
                                 Granularity.PER_TENSOR, DType.S8)
    pins["calib_sym_s8"] = [float(q3.scale), q3.zero_point]
    pins["quantize"] = [
        int(si.quantize(np.float32(0.0), QuantParams(np.float32(0.5), 64, DType.U8))),
        int(si.quantize(np.float32(1.0), QuantParams(np.float32(0.5), 0, DType.S8))),
        int(si.quantize(np.float32(1000.0), QuantParams(np.float32(0.5), 0, DType.S8))),
    ]
    pins["dequantize"] = [
        float(si.dequantize(np.array([64], np.uint8), QuantParams(np.float32(0.5), 64, DType.U8))[0]),
        float(si.dequantize(np.array([-127], np.int8), QuantParams(np.float32(0.5), 0, DType.S8))[0]),
    ]
    pins["requantize"] = int(si.requantize(123456, 2e-4, QuantParams(np.float32(0.1), 10, DType.U8)))
    w1 = np.zeros((4, 8), np.int8)
    w1[:, 3] = [1, 2, 3, 4]
    s1 = si.encode_sparse(w1)
    pins["encode_single"] = dict(group_ptr=s1.group_ptr.tolist(), idx=s1.idx.tolist(),
                                 vals=s1.vals.tolist(), nnz=s1.nnz.tolist())
    pins["partition"] = {str(n): [list(t) for t in sk.plan_spmm(
        si.encode_sparse(si.generate_pattern_weight(64, 64, 0.5, 0)), n, threads=4).tasks]
        for n in (64, 256, 384)}
    gen = {}
    for (m, k, r, s) in [(8, 16, 0.5, 0), (7, 33, 0.75, 3), (768, 768, 0.9, 11),
                         (3072, 768, 0.8, 13), (1024, 1024, 0.9, 15)]:
        w = si.generate_pattern_weight(m, k, r, s)
        gen[f"{m}x{k}@{r}#{s}"] = digest(w)
    pins["generate_pattern_weight"] = gen
    pins["sparsity_ratio_768"] = si.sparsity_ratio(si.encode_sparse(
        si.generate_pattern_weight(768, 768, 0.9, 11)))

    # BASELINE config 1 (768^2 @90%, N=128): s32 and f32 outputs
    w, x, bias, scales = baseline_inputs(768, 768, 128, 0.9, 11)
    sw = si.encode_sparse(w, scales)
    p_raw = sk.raw_program(sw)
    p_deq = sk.build_program(scales, 1.0, 0, None, [("dequantize_acc",)])
    pins["config1"] = dict(seed=11, s32=digest(sk.spmm_ref(sw, x, p_raw, bias)),
                           f32=digest(sk.spmm_ref(sw, x, p_deq, bias)))
    # BASELINE config 3 slice (3072x768 @80%, first 256 tokens of the seed-13 batch),
    # tanh-GELU (the reference's own GELU) -> quant(0.05, 0, u8)
    w, x, bias, scales = baseline_inputs(3072, 768, 4096, 0.8, 13)
    sw = si.encode_sparse(w, scales)
    p_g = sk.build_program(scales, 1.0, 0, None,
                           [("dequantize_acc",), ("gelu",),
                            ("quantize", QuantParams(np.float32(0.05), 0, DType.U8))])
    xs = np.ascontiguousarray(x[:, :256])
    pins["config3_slice256"] = dict(seed=13, u8_tanh=digest(sk.spmm_ref(sw, xs, p_g, bias)))
    with open(os.path.join(HERE, "golden_pins.json"), "w") as f:
        json.dump(pins, f, indent=1)
    print("wrote", len(meta), "cases")


if __name__ == "__main__":
    main()
