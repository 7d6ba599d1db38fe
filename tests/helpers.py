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
