"""GPU parity of the 2:4-sparse tensor-core kernels -- K3, X-stationary
(csrc/spmm_xs.cu, kernel="sp"), and K4, W-stationary (csrc/spmm_ws.cu,
kernel="ws") -- against the C oracle -- bit-exact for every
epilogue form it compiles, on shapes ragged against its 256-row pair tiles,
128-k chunks and 224-token tiles, with residual operands (windows holding
more than two nonzero columns of a group) of zero, one and two MMAs."""

import numpy as np
import pytest
import torch

from helpers import baseline_inputs, image_header
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

pytestmark = pytest.mark.gpu

# (M, K, N, sparsity, program)
CASES = [(512, 128, 224, 0.9, "s32"), (512, 256, 100, 0.9, "s32"), (300, 208, 1000, 0.85, "s32"),
         (1024, 1024, 4096, 0.9, "requant_u8"), (768, 768, 2000, 0.9, "requant_u8"),
         (520, 272, 1500, 0.8, "deq_f32"), (768, 768, 1504, 0.9, "gelu_erf_u8"), (4096, 1024, 2240, 0.9, "s32"),
         (1024, 1024, 4480, 0.9, "requant_u8"), (2048, 1024, 1792, 0.9, "requant_u8"),
         (384, 512, 7, 0.9, "deq_f32"), (640, 1024, 225, 0.9, "gelu_tanh_u8"), (256, 16, 333, 0.0, "s32")]


def _sp_applies(plan) -> bool:
    h = image_header(np.asarray(plan.image))
    return h.tr_ok == 1 and h.tc_kpad <= 1024 and h.tc_mtiles >= 2 and h.K % 16 == 0


@pytest.mark.parametrize("kernel", ["sp", "ws"])
@pytest.mark.parametrize("m,k,n,ratio,kind", CASES)
def test_sp_kernel_bit_exact(m, k, n, ratio, kind, kernel):
    w, x, bias, scales = baseline_inputs(m, k, n, ratio, 900 + m + k + n)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales, a_zp=2)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    assert _sp_applies(plan), (m, k, n, ratio)
    act = K.relayout_tokens(np.ascontiguousarray(x.T))
    got = K.spmm_exec(plan, act, kernel=kernel).cpu().numpy()
    want = oracle.spmm_exec(sw, x, prog, bias)
    if want.dtype == np.float32 and kind.startswith("gelu") and not kind.endswith("u8"):
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
    else:
        bad = np.argwhere(got != want)
        assert len(bad) == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"


def test_sp_residual_counts_covered():
    """The cases above exercise pair tiles with 0, 1 and 2 residual MMAs."""
    seen = set()
    for m, k, n, ratio, kind in CASES:
        w, _, bias, scales = baseline_inputs(m, k, 1, ratio, 900 + m + k + n, with_x=False)
        from paper_2306_16601_b200.kernels.spmm import _build_image
        img, _ = _build_image(P.encode_sparse(w, scales), workloads.program("s32", scales), bias)
        h = image_header(img)
        cnt = img[h.off_tr_cnt: h.off_tr_cnt + 4 * h.tr_pairs].view(np.int32)
        seen |= set(cnt.tolist())
    assert {0, 1, 2} <= seen, seen


@pytest.mark.parametrize("kernel", ["sp", "ws"])
def test_sp_unsupported_is_refused(kernel):
    """[K, N] activations and K > 1024 are not K3's: an explicit request is
    refused (RuntimeError from SI_EUNSUPPORTED), AUTO routes elsewhere."""
    w, x, bias, scales = baseline_inputs(512, 2048, 300, 0.9, 5)
    sw = P.encode_sparse(w, scales)
    plan = K.plan_spmm(sw, 300, bias=bias)
    with pytest.raises(RuntimeError):
        K.spmm_exec(plan, K.relayout_tokens(np.ascontiguousarray(x.T)), kernel=kernel)
    with pytest.raises(RuntimeError):
        K.spmm_exec(plan, K.relayout_activation(x), kernel=kernel)
    got = K.spmm_exec(plan, K.relayout_tokens(np.ascontiguousarray(x.T))).cpu().numpy()
    assert np.array_equal(got, oracle.spmm_exec(sw, x, K.raw_program(sw), bias))


@pytest.mark.parametrize("kernel", ["sp", "ws"])
@pytest.mark.parametrize("cell", [c for c in workloads.CONFIG5 if c.k <= 1024], ids=lambda c: c.name)
def test_sp_config5_full(cell, kernel):
    """BASELINE config 5 at its full size on the 2:4 kernels (the linears with
    K <= 1024): all 65536 tokens, every output byte compared with the oracle.
    For K4 this is also the at-scale check that several MMA issuers
    accumulating into one tensor-memory accumulator lose no update."""
    w, x, bias, scales = baseline_inputs(cell.m, cell.k, cell.n, cell.ratio, cell.seed)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(cell.program, scales)
    plan = K.plan_spmm(sw, cell.n, program=prog, bias=bias)
    assert _sp_applies(plan)
    act = K.relayout_tokens(np.ascontiguousarray(x.T))
    want = oracle.spmm_exec(sw, x, prog, bias)
    for rep in range(2):     # a second launch right behind the first (PDL overlap)
        got = K.spmm_exec(plan, act, kernel=kernel)
    got = got.cpu().numpy()
    bad = np.argwhere(got != want)
    assert len(bad) == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"

