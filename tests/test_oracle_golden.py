"""Pin the C oracle (oracle/si_oracle.c) against the reference's own outputs.

The golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py).  If these pass, the oracle is a trustworthy
checker for the GPU parity tests."""

import numpy as np
import pytest

from helpers import baseline_inputs, digest, golden_case
from oracle import oracle
from paper_2306_16601_b200 import encode_sparse, workloads


def test_oracle_builds():
    oracle.build()
    assert oracle.max_threads() >= 1


def test_golden_cases_ref_and_exec(golden):
    d, meta = golden
    for i in range(len(meta)):
        c = golden_case(d, meta, i)
        got_ref = oracle.spmm_ref(c.sw, c.x, c.prog, c.bias, c.side)
        got_exec = oracle.spmm_exec(c.sw, c.x, c.prog, c.bias, c.side, threads=2)
        assert got_ref.dtype == c.ref.dtype, (i, c.meta)
        assert np.array_equal(got_ref, c.ref), (i, c.meta)
        assert np.array_equal(got_exec, c.ref), (i, c.meta)


def test_golden_decode_and_row_sums(golden):
    d, meta = golden
    for i in range(len(meta)):
        c = golden_case(d, meta, i)
        assert np.array_equal(oracle.decode(c.sw), c.w)
        assert np.array_equal(oracle.row_sums(c.sw), d[f"c{i}_comp"])


def test_extreme_values(golden):
    d, _ = golden
    from paper_2306_16601_b200.kernels.spmm import raw_program
    sw = encode_sparse(d["extreme_w"], np.full(d["extreme_w"].shape[0], 1e-3, np.float32))
    got = oracle.spmm_ref(sw, d["extreme_x"], raw_program(sw), d["extreme_bias"])
    assert np.array_equal(got, d["extreme_ref"])


def test_config1_pins(pins):
    w, x, bias, scales = baseline_inputs(768, 768, 128, 0.9, 11)
    sw = encode_sparse(w, scales)
    for kind, key in (("s32", "s32"), ("deq_f32", "f32")):
        prog = workloads.program(kind, scales)
        assert digest(oracle.spmm_ref(sw, x, prog, bias)) == pins["config1"][key]
        assert digest(oracle.spmm_exec(sw, x, prog, bias)) == pins["config1"][key]


def test_config3_slice_pin(pins):
    w, x, bias, scales = baseline_inputs(3072, 768, 4096, 0.8, 13)
    sw = encode_sparse(w, scales)
    prog = workloads.program("gelu_tanh_u8", scales)
    xs = np.ascontiguousarray(x[:, :256])
    assert digest(oracle.spmm_exec(sw, xs, prog, bias)) == pins["config3_slice256"]["u8_tanh"]


@pytest.mark.parametrize("erf", [False, True])
def test_gelu_known_values(erf):
    # GELU(0)=0; odd symmetry of x*Phi(x) - x/2 ...; large x -> x
    g = oracle.gelu(np.array([0.0, 20.0, -20.0, 1.0], np.float32), erf=erf)
    assert g[0] == 0.0 and g[1] == np.float32(20.0) and g[2] == 0.0
    assert abs(g[3] - 0.8413) < 2e-3
