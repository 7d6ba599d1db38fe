"""Shared test helpers: golden-case reconstruction and digests."""

from __future__ import annotations

import hashlib
from types import SimpleNamespace

import numpy as np

from paper_2306_16601_b200 import DType, encode_sparse
from paper_2306_16601_b200.workloads import baseline_inputs  # noqa: F401
from paper_2306_16601_b200.kernels.epilogue import EpilogueProgram

DT = {"f32": DType.F32, "s8": DType.S8, "u8": DType.U8, "s32": DType.S32}


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def golden_case(d, meta, i):
    """Rebuild (weight, x, bias, program, sides, expected) of golden case i."""
    c = meta[i]
    pre = f"c{i}_"
    w = d[pre + "w"]
    sw = encode_sparse(w, d[pre + "scales"])
    prog = EpilogueProgram(
        scale_in=d[pre + "p_scale_in"], a_zp=int(c["a_zp"]), ops=d[pre + "p_ops"],
        fparams=d[pre + "p_fparams"], iparams=d[pre + "p_iparams"], luts=d[pre + "p_luts"],
        chans=d[pre + "p_chans"], out_dtype=DT[c["out_dtype"]], n_sides=int(c["n_sides"]))
    side = d[pre + "side"] if c["has_side"] else None
    return SimpleNamespace(meta=c, w=w, sw=sw, x=d[pre + "x"], bias=d[pre + "bias"], prog=prog,
                           side=side, ref=d[pre + "ref"])


def has_gelu(prog) -> bool:
    return bool(np.isin(prog.ops, [3, 8]).any())


# ctypes mirror of the plan image header (csrc/image.h SiImage); test-side
# only, used to inspect plan sections
import ctypes as _ct  # noqa: E402


class SiImageHeader(_ct.Structure):
    _fields_ = [("magic", _ct.c_uint32), ("version", _ct.c_uint32), ("M", _ct.c_int32), ("K", _ct.c_int32),
                ("rows", _ct.c_int32), ("groups", _ct.c_int32), ("padded_blocks", _ct.c_int64),
                ("nnz_blocks", _ct.c_int64), ("tiles", _ct.c_int64), ("out_dtype", _ct.c_int32),
                ("a_zp", _ct.c_int32), ("n_ops", _ct.c_int32), ("n_luts", _ct.c_int32), ("n_chans", _ct.c_int32),
                ("n_sides", _ct.c_int32), ("epi_mode", _ct.c_int32), ("exact", _ct.c_int32),
                ("q_scale", _ct.c_float), ("q_inv", _ct.c_float), ("q_zp", _ct.c_int32), ("q_lo", _ct.c_int32),
                ("q_hi", _ct.c_int32), ("n_bp", _ct.c_int32), ("tc_mtiles", _ct.c_int32), ("tc_kpad", _ct.c_int32),
                ("pad0", _ct.c_int32), ("pad1", _ct.c_int32)] + \
               [(f, _ct.c_uint64) for f in ("off_tile_ptr", "off_tile_w", "off_tile_idx", "off_adj", "off_scale_in",
                                            "off_ops", "off_fparams", "off_finv", "off_iparams", "off_luts",
                                            "off_chans", "off_clut", "off_bp_x", "off_bp_v", "off_tc_wt",
                                            "total_bytes", "off_rqc")] + \
               [("bp_key_lo", _ct.c_int32), ("bp_shift", _ct.c_int32), ("bp_nbucket", _ct.c_int32),
                ("bp_occ", _ct.c_int32), ("off_bp_key", _ct.c_uint64), ("off_bp_bucket", _ct.c_uint64),
                ("tc_emax", _ct.c_int32), ("tc_nlists", _ct.c_int32), ("off_tc_eptr", _ct.c_uint64),
                ("off_tc_ent", _ct.c_uint64), ("off_rqg", _ct.c_uint64), ("off_sp_img", _ct.c_uint64),
                ("off_sp_rptr", _ct.c_uint64), ("off_sp_res", _ct.c_uint64), ("sp_nres", _ct.c_int32),
                ("sp_maxres", _ct.c_int32), ("off_rqp", _ct.c_uint64), ("off_tr_img", _ct.c_uint64),
                ("off_tr_k", _ct.c_uint64), ("off_tr_cnt", _ct.c_uint64), ("tr_ok", _ct.c_int32),
                ("tr_pairs", _ct.c_int32), ("off_tc_wrow", _ct.c_uint64), ("off_bp_lin", _ct.c_uint64),
                ("bp_lin_n", _ct.c_int32), ("bp_lin_inv", _ct.c_float), ("bp_lin_off", _ct.c_float),
                ("pad2", _ct.c_int32), ("reserved0", _ct.c_uint64)]


def image_header(img: np.ndarray) -> SiImageHeader:
    assert _ct.sizeof(SiImageHeader) == 432
    h = SiImageHeader.from_buffer_copy(img[:432].tobytes())
    assert h.total_bytes == img.size
    return h


def image_section(img: np.ndarray, off: int, dtype, count: int) -> np.ndarray:
    return img[off:off + np.dtype(dtype).itemsize * count].view(dtype)
