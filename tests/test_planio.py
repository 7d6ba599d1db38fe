"""Plan container (planio.py) round trips and format errors; the dense INT8
comparator (kernels/dense.py) on the GPU against the oracle."""

import os

import numpy as np
import pytest

from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import workloads as W
from paper_2306_16601_b200.kernels import plan_spmm
from paper_2306_16601_b200.planio import MAGIC, PlanFormatError, load_plan, save_plan


def _plan(m=300, k=200, n=64, ratio=0.8, kind="requant_u8", device="cpu"):
    w, x, bias, scales = W.baseline_inputs(m, k, n, ratio, 3)
    sw = P.encode_sparse(w, scales)
    prog = W.program(kind, scales)
    return plan_spmm(sw, n, program=prog, bias=bias, device=device), w, x, bias, prog


def test_round_trip_is_bit_exact_and_deterministic(tmp_path):
    plan, *_ = _plan()
    a, b = tmp_path / "a.si4p", tmp_path / "b.si4p"
    save_plan(plan, str(a))
    save_plan(plan, str(b))
    assert a.read_bytes() == b.read_bytes()
    q = load_plan(str(a), device="cpu")
    np.testing.assert_array_equal(q.image, plan.image)
    for f in ("group_ptr", "idx", "vals", "nnz", "scales"):
        np.testing.assert_array_equal(getattr(q.weight, f), getattr(plan.weight, f))
    for f in ("scale_in", "ops", "fparams", "iparams", "luts", "chans"):
        np.testing.assert_array_equal(getattr(q.program, f), getattr(plan.program, f))
    assert q.program.out_dtype == plan.program.out_dtype and q.program.a_zp == plan.program.a_zp
    np.testing.assert_array_equal(q.bias, plan.bias)
    assert (q.n, q.bn, q.threads) == (plan.n, plan.bn, plan.threads)
    assert q.info == plan.info


@pytest.mark.parametrize("corrupt,msg", [
    (lambda d: b"XXXX" + d[4:], "magic"),
    (lambda d: d[:4] + (7).to_bytes(4, "little") + d[8:], "version"),
    (lambda d: d[:len(d) // 2], "bounds"),
    (lambda d: d[:16] + b"!" + d[17:], "metadata"),
])
def test_format_errors_are_detected(tmp_path, corrupt, msg):
    plan, *_ = _plan()
    p = tmp_path / "p.si4p"
    save_plan(plan, str(p))
    d = p.read_bytes()
    assert d[:4] == MAGIC
    bad = tmp_path / "bad.si4p"
    bad.write_bytes(corrupt(d))
    with pytest.raises(PlanFormatError):
        load_plan(str(bad), device="cpu")


def test_corrupt_image_header_is_rejected(tmp_path):
    plan, *_ = _plan()
    p = tmp_path / "p.si4p"
    save_plan(plan, str(p))
    d = bytearray(p.read_bytes())
    i = bytes(d).rfind(plan.image[:8].tobytes())   # the image's magic + version
    d[i] ^= 0xFF
    p.write_bytes(bytes(d))
    with pytest.raises(ValueError):
        load_plan(str(p), device="cpu")


def _with_image(plan, image):
    import dataclasses
    return dataclasses.replace(plan, image=np.ascontiguousarray(image, dtype=np.uint8))


@pytest.mark.parametrize("edit", ["short", "section", "total", "m_field"])
def test_malformed_image_is_rejected_natively(tmp_path, edit):
    """si_plan_image_validate: a container whose image blob is
    short, has a section outside the image, claims more bytes than it has,
    or disagrees with the packed weight fails with PlanFormatError before
    any kernel could read out of bounds."""
    from helpers import SiImageHeader
    import ctypes
    plan, *_ = _plan()
    img = plan.image.copy()
    hdr = SiImageHeader.from_buffer_copy(img[:ctypes.sizeof(SiImageHeader)].tobytes())
    if edit == "short":
        img = img[:300]
    elif edit == "section":
        off = SiImageHeader.off_tc_wt.offset
        img[off:off + 8] = np.frombuffer(np.uint64(hdr.total_bytes - 64).tobytes(), np.uint8)
    elif edit == "total":
        off = SiImageHeader.total_bytes.offset
        img[off:off + 8] = np.frombuffer(np.uint64(hdr.total_bytes + 4096).tobytes(), np.uint8)
    else:
        off = SiImageHeader.M.offset
        img[off:off + 4] = np.frombuffer(np.int32(hdr.M - 4).tobytes(), np.uint8)
    p = tmp_path / "m.si4p"
    save_plan(_with_image(plan, img), str(p))
    with pytest.raises(PlanFormatError):
        load_plan(str(p), device="cpu")


def test_built_images_validate():
    from paper_2306_16601_b200 import _lib
    for m, k, ratio in ((300, 200, 0.8), (4096, 1024, 0.9), (1, 1, 0.0), (64, 4096, 1.0)):
        plan, *_ = _plan(m, k, 16, ratio)
        assert _lib.lib().si_plan_image_validate(_lib.ptr(plan.image), plan.image.nbytes) == 0


@pytest.mark.gpu
def test_loaded_plan_runs_bit_exact(tmp_path):
    from paper_2306_16601_b200 import kernels as K
    plan, w, x, bias, prog = _plan(1024, 512, 2048, 0.9, "requant_u8", device="cuda")
    p = tmp_path / "p.si4p"
    save_plan(plan, str(p))
    q = load_plan(str(p), device="cuda")
    act = K.relayout_activation(x)
    a = K.spmm_exec(plan, act).cpu().numpy()
    b = K.spmm_exec(q, act).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(b, oracle.spmm_exec(plan.weight, x, prog, bias))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["s32", "deq_f32", "requant_u8"])
def test_dense_comparator_matches_oracle(kind):
    from paper_2306_16601_b200.kernels.dense import dense_gemm_s8
    rng = np.random.default_rng(9)
    m, k, n = 512, 384, 2048
    w = rng.integers(-127, 128, (m, k)).astype(np.int8)
    x = rng.integers(0, 256, (k, n)).astype(np.uint8)
    bias = rng.integers(-1000, 1001, m).astype(np.int32)
    scales = rng.uniform(1e-4, 1e-3, m).astype(np.float32)
    prog = W.program(kind, scales)
    got = dense_gemm_s8(w, x, prog, bias).cpu().numpy()
    want = oracle.spmm_ref(P.encode_sparse(w, scales), x, prog, bias)
    g = got.view(np.uint32) if got.dtype == np.float32 else got
    wv = want.view(np.uint32) if want.dtype == np.float32 else want
    np.testing.assert_array_equal(g, wv)
