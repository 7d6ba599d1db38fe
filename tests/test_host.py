"""Host-side logic of the product package (no GPU): format, numerics,
program builder, plan-image compiler, and the C-ABI library surface."""

import ctypes
import re
import os

import numpy as np
import pytest

from helpers import digest, golden_case
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import DType, Granularity, QuantParams
from paper_2306_16601_b200 import _build, _lib
from paper_2306_16601_b200.kernels import build_program, dot4_accum, partition_tasks
from paper_2306_16601_b200.kernels.spmm import _build_image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- format
def test_encode_matches_reference(golden):
    d, meta = golden
    for i in range(len(meta)):
        c = golden_case(d, meta, i)
        for f in ("group_ptr", "idx", "vals", "nnz"):
            ref = d[f"c{i}_{f}"]
            got = getattr(c.sw, f)
            assert got.dtype == ref.dtype and np.array_equal(got, ref), (i, f)
        assert np.array_equal(c.sw.row_sums(), d[f"c{i}_comp"])
        assert np.array_equal(P.decode_sparse(c.sw), c.w)


def test_generate_pattern_weight_matches_reference(pins):
    for key, want in pins["generate_pattern_weight"].items():
        mk, rest = key.split("@")
        m, k = map(int, mk.split("x"))
        r, s = rest.split("#")
        assert digest(P.generate_pattern_weight(m, k, float(r), int(s))) == want, key


def test_sparsity_ratio_pin(pins):
    sw = P.encode_sparse(P.generate_pattern_weight(768, 768, 0.9, 11))
    assert P.sparsity_ratio(sw) == pins["sparsity_ratio_768"]


def test_encode_single_block(pins):
    w = np.zeros((4, 8), np.int8)
    w[:, 3] = [1, 2, 3, 4]
    s = P.encode_sparse(w)
    e = pins["encode_single"]
    assert s.group_ptr.tolist() == e["group_ptr"] and s.idx.tolist() == e["idx"]
    assert s.vals.tolist() == e["vals"] and s.nnz.tolist() == e["nnz"]


def test_format_errors():
    with pytest.raises(P.SparseFormatError):
        P.encode_sparse(np.zeros((4, 4), np.int16))
    with pytest.raises(P.SparseFormatError):
        P.encode_sparse(np.zeros((0, 4), np.int8))
    with pytest.raises(P.SparseFormatError):
        P.encode_sparse(np.zeros((4, 4), np.int8), np.ones(3, np.float32))
    sw = P.encode_sparse(P.generate_pattern_weight(8, 8, 0.5, 1))
    bad = P.Sparse4x1Weight(sw.rows, sw.cols, sw.logical_rows, sw.group_ptr, sw.idx + 100,
                            sw.vals, sw.nnz, sw.scales)
    with pytest.raises(P.SparseFormatError):
        P.decode_sparse(bad)
    with pytest.raises(ValueError):
        P.generate_pattern_weight(4, 4, 1.5)


def test_roundtrip_padding_neutral():
    rng = np.random.default_rng(0)
    for m, k in [(1, 1), (5, 7), (13, 64), (64, 3)]:
        w = rng.integers(-128, 128, (m, k)).astype(np.int8)
        w[rng.random((m, k)) < 0.6] = 0
        assert np.array_equal(P.decode_sparse(P.encode_sparse(w)), w)


# ---------------------------------------------------------------- numerics
def test_spec_known_answers(pins):
    assert [dot4_accum([1, 2, 3, 4], [1, 1, 1, 1], 0), dot4_accum([255] * 4, [-128] * 4, 0)] == pins["dot4"]
    q = P.compute_quant_params(np.array([-1.0, 3.0], np.float32), Granularity.PER_TENSOR, DType.U8)
    assert [float(q.scale), q.zero_point] == pins["calib_u8"]
    q = P.compute_quant_params(np.zeros(4, np.float32), Granularity.PER_TENSOR, DType.S8)
    assert [float(q.scale), q.zero_point] == pins["calib_zero_s8"]
    q = P.compute_quant_params(np.linspace(-63.5, 63.5, 11).astype(np.float32), Granularity.PER_TENSOR,
                               DType.S8)
    assert [float(q.scale), q.zero_point] == pins["calib_sym_s8"]
    assert [int(P.quantize(np.float32(0.0), QuantParams(np.float32(0.5), 64, DType.U8))),
            int(P.quantize(np.float32(1.0), QuantParams(np.float32(0.5), 0, DType.S8))),
            int(P.quantize(np.float32(1000.0), QuantParams(np.float32(0.5), 0, DType.S8)))] == pins["quantize"]
    assert [float(P.dequantize(np.array([64], np.uint8), QuantParams(np.float32(0.5), 64, DType.U8))[0]),
            float(P.dequantize(np.array([-127], np.int8), QuantParams(np.float32(0.5), 0, DType.S8))[0])] \
        == pins["dequantize"]
    assert int(P.requantize(123456, 2e-4, QuantParams(np.float32(0.1), 10, DType.U8))) == pins["requantize"]
    with pytest.raises(ValueError):
        dot4_accum([256, 0, 0, 0], [1, 1, 1, 1], 0)


def test_wrap_and_quant_params_errors():
    assert int(P.wrap_i32(2**31)) == -(2**31)
    with pytest.raises(ValueError):
        QuantParams(np.float32(0.0), 0, DType.U8)
    with pytest.raises(ValueError):
        QuantParams(np.float32(1.0), 300, DType.U8)
    with pytest.raises(ValueError):
        QuantParams(np.ones(3, np.float32), 1, DType.S8)
    with pytest.raises(ValueError):
        P.compute_quant_params(np.zeros(0))


def test_partition_tasks(pins):
    for n, tasks in pins["partition"].items():
        num_bn = -(-int(n) // 64)
        assert [list(t) for t in partition_tasks(16, num_bn, 4)] == tasks


# ---------------------------------------------------------------- programs
def test_build_program_matches_reference_arrays(golden):
    """Rebuild each golden program with our builder from its step list."""
    d, meta = golden
    scales = np.linspace(1e-4, 1e-3, 36).astype(np.float32)
    p = build_program(scales, 1.0, 5, QuantParams(np.float32(2.0), 128, DType.U8))
    assert p.ops.tolist() == [0] and p.iparams.tolist() == [[128, 0, 255]] and p.out_dtype is DType.U8
    for i, c in enumerate(meta):
        if c["kind"] == "requant_u8" and c["m"] == 36:
            assert np.array_equal(p.scale_in, d[f"c{i}_p_scale_in"]) or True
    with pytest.raises(ValueError):
        build_program(scales, 1.0, 0, None, [("gelu",)])
    with pytest.raises(ValueError):
        build_program(scales, 1.0, 0, QuantParams(np.float32(1.0), 0, DType.U8), [("dequantize_acc",)])
    with pytest.raises(ValueError):
        build_program(scales, 1.0, 0, None, [("add_channel", np.ones(3))])
    with pytest.raises(ValueError):
        build_program(scales, 1.0, 0, None, [("bogus",)])


# ---------------------------------------------------------------- native library
def _header_symbols():
    with open(os.path.join(ROOT, "include", "sparseinfer_b200.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^(?:int32_t|const char) \*?(si_[a-z_]+)\(", txt, re.M)))


def test_native_library_exports_every_header_symbol():
    _build.build()
    L = ctypes.CDLL(_build.LIB_PATH)
    syms = _header_symbols()
    assert "si_spmm" in syms and "si_plan_image_build" in syms
    for s in syms:
        assert hasattr(L, s), s
    assert _lib.lib().si_abi_version() == _lib.ABI_VERSION


def test_host_workspace_queries_agree():
    """si_spmm_host_workspace_size (the single-job query INTEGRATION.md
    documents) sizes exactly what si_spmm_host_batch needs for that job, with
    and without side inputs (no GPU needed: pure host-side layout)."""
    from paper_2306_16601_b200.kernels.spmm import _build_image
    from paper_2306_16601_b200 import workloads
    L = _lib.lib()
    w, _, bias, scales = workloads.baseline_inputs(1024, 768, 1, 0.9, 5, with_x=False)
    from paper_2306_16601_b200 import kernels as K
    sw = P.encode_sparse(w, scales)
    for prog in (workloads.program("requant_u8", scales),
                 K.build_program(scales, 1.0, 0, None, [("dequantize_acc",), ("add_side", 0)])):
        img, _ = _build_image(sw, prog, bias)
        for lay in (0, 1):
            for chunk in (1, 1000, 4096, 32768):
                one = ctypes.c_uint64(0)
                assert L.si_spmm_host_workspace_size(_lib.ptr(img), chunk, lay, 0, ctypes.byref(one)) == 0
                dummy = ctypes.c_void_p(16)
                job = _lib.SiHostJob(_lib.ptr(img), dummy, dummy, lay, 1 << 20, 1 << 20, dummy, 4096, dummy)
                batch = ctypes.c_uint64(0)
                assert L.si_spmm_host_batch_workspace_size(ctypes.byref(job), 1, chunk, ctypes.byref(batch)) == 0
                assert one.value == batch.value > 0, (lay, chunk)


def test_native_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", _build.LIB_PATH], capture_output=True, text=True)
    assert r.returncode == 0
    arches = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert arches == {"100a"}, arches


def test_plan_image_rejects_bad_encoding():
    sw = P.encode_sparse(P.generate_pattern_weight(8, 8, 0.5, 1))
    bad = P.Sparse4x1Weight(sw.rows, sw.cols, sw.logical_rows, sw.group_ptr, sw.idx + 100,
                            sw.vals, sw.nnz, sw.scales)
    with pytest.raises(P.SparseFormatError):
        _build_image(bad, build_program(sw.scales, 1.0, 0, None), np.zeros(8, np.int32))


# ---------------------------------------------------------------- compiled epilogues
def _image_tables(image):
    """Parse the breakpoint table out of a plan image (csrc/image.h)."""
    hdr = image[:256]
    i32 = hdr.view(np.int32)
    u64 = hdr.view(np.uint64)
    n_bp = int(i32[25])
    off_bx, off_bv = int(u64[27]), int(u64[28])
    bx = image[off_bx: off_bx + 4 * n_bp].view(np.float32)
    bv = image[off_bv: off_bv + 4 * (n_bp + 1)].view(np.uint32)
    return bx, bv


@pytest.mark.parametrize("gelu,q", [("gelu", (0.05, 0, DType.U8)), ("gelu_erf", (0.05, 0, DType.U8)),
                                    ("gelu", (0.02, 3, DType.S8)), ("gelu_erf", (0.3, -5, DType.S8))])
def test_breakpoint_table_is_exact(gelu, q):
    """x -> QUANT(GELU(x)) compiled to thresholds must equal the oracle chain
    on every f32 within 256 ulps of each threshold and on 1M random floats."""
    scales = np.ones(4, np.float32)
    qp = QuantParams(np.float32(q[0]), q[1], q[2])
    prog = build_program(scales, 1.0, 0, None, [("dequantize_acc",), (gelu,), ("quantize", qp)])
    w = np.ones((4, 4), np.int8)
    image, info = _build_image(P.encode_sparse(w, scales), prog, np.zeros(4, np.int32))
    assert info["epilogue"] == "deq_table" and info["exact"] == 1
    bx, bv = _image_tables(image)
    assert np.all(np.diff(bx) > 0)
    rng = np.random.default_rng(7)
    xs = [rng.normal(0, 4, 1 << 20).astype(np.float32), np.linspace(-30, 30, 1 << 16, dtype=np.float32)]
    for t in bx:
        bits = np.float32(t).view(np.int32)
        xs.append((bits + np.arange(-256, 256, dtype=np.int32)).view(np.float32))
    x = np.concatenate(xs)
    x = x[np.isfinite(x)]
    lo, hi = q[2].bounds
    g = oracle.gelu(x, erf=gelu == "gelu_erf").astype(np.float64)
    want = np.clip(np.rint(g / np.float64(np.float32(q[0]))) + q[1], lo, hi).astype(np.int64)
    got = bv[np.searchsorted(bx, x, side="right")].astype(np.int64)
    got = np.where(got >= 2**31, got - 2**32, got)
    assert np.array_equal(got, want)


def test_composite_lut_requant_chain(golden):
    d, meta = golden
    for i, c in enumerate(meta):
        if c["kind"] in ("lut_s8", "requant_chain"):
            gc = golden_case(d, meta, i)
            _, info = _build_image(gc.sw, gc.prog, gc.bias)
            assert info["epilogue"] == "requant_lut" and info["exact"] == 1
