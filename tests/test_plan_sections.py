"""CPU checks of plan-image sections that the GPU kernels rely on:
the requant exactness proof (plan.cpp requant_row_exact) and the 2:4
images + residual lists of the 2:4 tensor-core images (K3)."""

import numpy as np
import pytest

import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import workloads as W
from paper_2306_16601_b200.kernels.spmm import _build_image
from helpers import image_header, image_section


def _plan(m, k, ratio, seed, program):
    w, _, bias, scales = W.baseline_inputs(m, k, 1, ratio, seed, with_x=False)
    sw = P.encode_sparse(w, scales)
    prog = W.program(program, scales)
    img, _ = _build_image(sw, prog, bias)
    return w, bias, prog, img


@pytest.mark.parametrize("m,k,ratio,seed,nrows", [(1024, 1024, 0.9, 11, 8), (512, 768, 0.8, 3, 8),
                                                   (256, 4096, 0.9, 13, 2)])
def test_requant_proof_brute_force(m, k, ratio, seed, nrows):
    """Rows the plan marks proven (rqg == 1) use out = rint(a * c' + zp)
    (one rounding, the device's fma form) with the plan's multiplier c' (rqp);
    enumerate every reachable accumulator and compare with the reference."""
    w, bias, prog, img = _plan(m, k, ratio, seed, "requant_u8")
    h = image_header(img)
    rqg = image_section(img, h.off_rqg, np.float32, m)
    rqp = image_section(img, h.off_rqp, np.float32, m)
    adj = image_section(img, h.off_adj, np.int32, m)
    proven = rqg >= 1
    assert proven.mean() > 0.9, "the multiplier search should prove most rows"
    g = rqg[~proven]
    assert ((g >= 0) & (g <= 0.25)).all(), "other rows carry the certificate guard"
    s_in = np.asarray(prog.scale_in, np.float32)
    fp = np.float32(np.asarray(prog.fparams).reshape(-1)[0])
    zp, lo, hi = (int(v) for v in np.asarray(prog.iparams).reshape(-1)[:3])
    rng = np.random.default_rng(0)
    for r in rng.choice(np.flatnonzero(proven), nrows, replace=False):
        A = 255 * int(np.abs(w[r].astype(np.int64)).sum()) + abs(int(adj[r]))
        assert A < 1 << 24 and (A < 1 << 22 or rqg[r] == 2)
        for a0 in range(-A, A + 1, 1 << 22):
            a = np.arange(a0, min(a0 + (1 << 22), A + 1), dtype=np.int64).astype(np.float64)
            dev = np.rint(a * np.float64(rqp[r]) + zp)      # exact: |a| < 2^24, 24-bit c'
            ref = np.rint(a * np.float64(s_in[r]) / np.float64(fp)) + zp
            np.testing.assert_array_equal(np.clip(dev, lo, hi), np.clip(ref, lo, hi), err_msg=f"row {r}")


@pytest.mark.parametrize("m,k,ratio", [(1024, 1024, 0.9), (200, 300, 0.5), (384, 200, 0.8)])
def test_sparse_images_reconstruct_weight(m, k, ratio):
    w, _, _, img = _plan(m, k, ratio, 5, "s32")
    h = image_header(img)
    mt, kch = h.tc_mtiles, h.tc_kpad // 128
    mt_pad = (mt + 1) // 2 * 2
    sp = image_section(img, h.off_sp_img, np.uint8, mt_pad * kch * 12288).reshape(mt_pad, kch, 12288)
    rptr = image_section(img, h.off_sp_rptr, np.int32, mt * 128 + 1)
    res = image_section(img, h.off_sp_res, np.int32, h.sp_nres)
    D = np.zeros((mt_pad * 128, kch * 128), np.int64)
    row = np.arange(128)[:, None]
    pb = np.arange(64)[None, :]
    rr = np.arange(128)
    for rt in range(mt_pad):
        for kc in range(kch):
            t = sp[rt, kc]
            a = t[(row // 8) * 512 + (pb // 16) * 128 + (row % 8) * 16 + pb % 16].view(np.int8).astype(np.int64)
            for mma in range(2):
                e = t[8192 + mma * 2048 + (row // 8) * 128 + (row % 8) * 16 + np.arange(8)[None, :]]
                for wm in range(16):
                    nib = ((e[:, wm // 2] >> (4 * (wm % 2))) & 0xF).astype(np.int64)
                    i0, i1 = nib & 3, nib >> 2
                    assert (i0 < i1).all()
                    wl = mma * 16 + wm
                    np.add.at(D, (rt * 128 + rr, kc * 128 + wl * 4 + i0), a[:, 2 * wl])
                    np.add.at(D, (rt * 128 + rr, kc * 128 + wl * 4 + i1), a[:, 2 * wl + 1])
    for r in range(mt * 128):
        for ent in res[rptr[r]:rptr[r + 1]]:
            D[r, ent >> 8] += np.int8(ent & 0xFF)
    np.testing.assert_array_equal(D[:m, :k], w.astype(np.int64))
    assert not D[m:].any() and not D[:, k:].any()


def _decode_sp_tile(t):
    """(dense [128, 128] over the tile's 128 k / slot positions) of one 12 KB 2:4 image."""
    row = np.arange(128)[:, None]
    pb = np.arange(64)[None, :]
    rr = np.arange(128)
    a = t[(row // 8) * 512 + (pb // 16) * 128 + (row % 8) * 16 + pb % 16].view(np.int8).astype(np.int64)
    D = np.zeros((128, 128), np.int64)
    for mma in range(2):
        e = t[8192 + mma * 2048 + (row // 8) * 128 + (row % 8) * 16 + np.arange(8)[None, :]]
        for wm in range(16):
            nib = ((e[:, wm // 2] >> (4 * (wm % 2))) & 0xF).astype(np.int64)
            i0, i1 = nib & 3, nib >> 2
            assert (i0 < i1).all()
            wl = mma * 16 + wm
            np.add.at(D, (rr, wl * 4 + i0), a[:, 2 * wl])
            np.add.at(D, (rr, wl * 4 + i1), a[:, 2 * wl + 1])
    return D


@pytest.mark.parametrize("m,k,ratio", [(1024, 1024, 0.9), (520, 272, 0.8), (768, 768, 0.85), (4096, 1024, 0.9)])
def test_k2t_residual_operand_reconstructs_weight(m, k, ratio):
    """K3: main 2:4 images + the per-pair-tile residual operand over slots
    (slot s = activation column tr_k[s], 0xFFFF when unused) sum to W exactly;
    slots beyond the tile's residual MMA count carry no weight."""
    w, _, _, img = _plan(m, k, ratio, 7, "s32")
    h = image_header(img)
    assert h.tr_ok == 1
    mt, kch = h.tc_mtiles, h.tc_kpad // 128
    pt_n = (mt + 1) // 2
    assert h.tr_pairs == pt_n
    sp = image_section(img, h.off_sp_img, np.uint8, 2 * pt_n * kch * 12288).reshape(2 * pt_n, kch, 12288)
    tri = image_section(img, h.off_tr_img, np.uint8, 2 * pt_n * 12288).reshape(2 * pt_n, 12288)
    trk = image_section(img, h.off_tr_k, np.uint16, pt_n * 128).reshape(pt_n, 128).astype(np.int64)
    cnt = image_section(img, h.off_tr_cnt, np.int32, pt_n)
    assert ((cnt >= 0) & (cnt <= 2)).all()
    D = np.zeros((2 * pt_n * 128, kch * 128), np.int64)
    for rt in range(2 * pt_n):
        for kc in range(kch):
            D[rt * 128:(rt + 1) * 128, kc * 128:(kc + 1) * 128] += _decode_sp_tile(sp[rt, kc])
        R = _decode_sp_tile(tri[rt])
        used = 64 * cnt[rt // 2]
        assert not R[:, used:].any()
        for s in range(used):
            if trk[rt // 2, s] == 0xFFFF:              # unused slot: no weight
                assert not R[:, s].any()
                continue
            D[rt * 128:(rt + 1) * 128, trk[rt // 2, s]] += R[:, s]
        assert (trk[rt // 2, used:] == 0xFFFF).all()
    np.testing.assert_array_equal(D[:m, :k], w.astype(np.int64))
    assert not D[m:].any() and not D[:, k:].any()


@pytest.mark.parametrize("kind", ["gelu_erf_u8", "gelu_tanh_u8"])
def test_linear_breakpoint_table_matches_threshold_search(kind):
    """EPI_DEQ_TABLE fast path: the linear buckets (one threshold each) give
    the same piece as a search over the thresholds, at every threshold, a few
    ulps either side of it, and at random points (the device's bucket function
    restated in extended precision)."""
    w, bias, prog, img = _plan(768, 256, 0.8, 3, kind)
    h = image_header(img)
    assert h.epi_mode == 4 and h.n_bp > 0
    assert h.bp_lin_n > 0, "BASELINE's GELU -> u8 programs must get the linear table"
    bx = image_section(img, h.off_bp_x, np.float32, h.n_bp)
    bv = image_section(img, h.off_bp_v, np.uint32, h.n_bp + 1).astype(np.int64)
    lin = image_section(img, h.off_bp_lin, np.uint32, 2 * h.bp_lin_n).reshape(-1, 2)
    thr = lin[:, 0].copy().view(np.float32)
    vlo = (lin[:, 1] & 0xFFFF).astype(np.int16).astype(np.int64)
    vhi = (lin[:, 1] >> 16).astype(np.int16).astype(np.int64)
    assert np.isfinite(thr).sum() == h.n_bp          # every threshold sits in its own bucket
    xs = [bx]
    for d in (1, 2, 3):
        up, dn = bx.copy(), bx.copy()
        for _ in range(d):
            up, dn = np.nextafter(up, np.float32(np.inf)), np.nextafter(dn, np.float32(-np.inf))
        xs += [up, dn]
    rng = np.random.default_rng(0)
    xs.append(rng.uniform(bx[0] - 1, bx[-1] + 1, 200000).astype(np.float32))
    xs.append(np.array([-1e30, 1e30, 0.0, -0.0], np.float32))
    x = np.concatenate(xs)
    t = (x.astype(np.longdouble) * np.longdouble(np.float32(h.bp_lin_inv)) + np.longdouble(np.float32(h.bp_lin_off)))
    t = np.clip(t.astype(np.float32), np.float32(0), np.float32(h.bp_lin_n - 1))
    b = np.rint(t).astype(np.int64)
    got = np.where(x >= thr[b], vhi[b], vlo[b])
    want = bv[np.searchsorted(bx, x, side="right")].astype(np.int32).astype(np.int64)
    bad = np.flatnonzero(got != want)
    assert len(bad) == 0, (len(bad), x[bad[:5]], got[bad[:5]], want[bad[:5]])
