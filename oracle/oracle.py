"""ctypes front-end of the C oracle (si_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package
never imports this module.

Objects are duck-typed so the same calls accept the reference's
``Sparse4x1Weight`` / ``EpilogueProgram`` and the product's mirrors:
weights need ``rows, cols, logical_rows, group_ptr, idx, vals``; programs
need ``scale_in, a_zp, ops, fparams, iparams, luts, chans, out_dtype``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libsi_oracle.so")
_lib = None

DT_CODES = {"f32": 0, "s8": 1, "u8": 2, "s32": 3}
DT_NP = {0: np.float32, 1: np.int8, 2: np.uint8, 3: np.int32}


class _Program(ctypes.Structure):
    _fields_ = [
        ("scale_in", ctypes.c_void_p),
        ("a_zp", ctypes.c_int32),
        ("n_ops", ctypes.c_int32),
        ("ops", ctypes.c_void_p),
        ("fparams", ctypes.c_void_p),
        ("iparams", ctypes.c_void_p),
        ("luts", ctypes.c_void_p),
        ("chans", ctypes.c_void_p),
        ("out_dtype", ctypes.c_int32),
    ]


def build() -> str:
    """Compile the oracle (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.orc_decode.argtypes = [i32, i32, i32, vp, vp, vp, vp]
        L.orc_decode.restype = ctypes.c_int
        L.orc_row_sums.argtypes = [i32, i32, vp, vp, vp]
        L.orc_ref_gemm_acc.argtypes = [vp, i32, i32, vp, i64, i64, vp, vp, i32, vp, ctypes.c_int]
        L.orc_apply_program.argtypes = [vp, i64, i64, ctypes.POINTER(_Program), vp, vp, ctypes.c_int]
        L.orc_spmm_exec.argtypes = [i32, i32, i32, vp, vp, vp, vp, i64, i64, vp, vp,
                                    ctypes.POINTER(_Program), vp, vp, ctypes.c_int, ctypes.c_int]
        L.orc_gelu_array.argtypes = [vp, vp, i64, ctypes.c_int]
        L.orc_softmax_rows.argtypes = [vp, vp, i64, i64]
        L.orc_layer_norm_rows.argtypes = [vp, vp, vp, ctypes.c_double, vp, i64, i64]
        L.orc_bmm.argtypes = [vp, vp, vp] + [i64] * 14 + [ctypes.c_int, ctypes.c_float]
        L.orc_quantize.argtypes = [vp, i64, ctypes.c_float, i32, i32, i32, vp, ctypes.c_int]
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _dt_code(dt) -> int:
    v = getattr(dt, "value", dt)
    return DT_CODES[v] if isinstance(v, str) else int(v)


class _Prog:
    """Keeps the contiguous arrays alive while the struct points at them."""

    def __init__(self, prog):
        self.scale_in = np.ascontiguousarray(prog.scale_in, dtype=np.float32)
        self.ops = np.ascontiguousarray(prog.ops, dtype=np.int32)
        self.fparams = np.ascontiguousarray(prog.fparams, dtype=np.float32)
        self.iparams = np.ascontiguousarray(prog.iparams, dtype=np.int32).reshape(-1)
        self.luts = np.ascontiguousarray(prog.luts, dtype=np.uint8).reshape(-1)
        self.chans = np.ascontiguousarray(prog.chans, dtype=np.float32).reshape(-1)
        self.out_code = _dt_code(prog.out_dtype)
        self.s = _Program(_p(self.scale_in), int(prog.a_zp), int(self.ops.shape[0]), _p(self.ops),
                          _p(self.fparams), _p(self.iparams), _p(self.luts), _p(self.chans),
                          self.out_code)


def decode(sw) -> np.ndarray:
    """decode_sparse (sparse.py:117-132)."""
    L = lib()
    gp = np.ascontiguousarray(sw.group_ptr, np.int32)
    idx = np.ascontiguousarray(sw.idx, np.int32)
    vals = np.ascontiguousarray(sw.vals, np.int8)
    wd = np.zeros((sw.logical_rows, sw.cols), np.int8)
    rc = L.orc_decode(sw.rows, sw.cols, sw.logical_rows, _p(gp), _p(idx), _p(vals), _p(wd))
    if rc == -1:
        raise ValueError("column index out of range")
    if rc:
        raise MemoryError("oracle decode failed")
    return wd


def row_sums(sw) -> np.ndarray:
    """Sparse4x1Weight.row_sums (sparse.py:51-62)."""
    comp = np.zeros(sw.logical_rows, np.int32)
    gp = np.ascontiguousarray(sw.group_ptr, np.int32)
    vals = np.ascontiguousarray(sw.vals, np.int8)
    lib().orc_row_sums(sw.rows, sw.logical_rows, _p(gp), _p(vals), _p(comp))
    return comp


def _bias(sw, bias):
    if bias is None:
        return np.zeros(sw.logical_rows, np.int32)
    return np.ascontiguousarray(bias, np.int32)


def _sides(n, m, sides):
    if sides is None:
        return None
    return np.ascontiguousarray(sides, np.float32)


def spmm_ref(sw, a: np.ndarray, program, bias=None, sides=None, threads: int | None = None):
    """spmm_ref (spmm.py:401-427): decode, dense wrapping GEMM, epilogue.

    ``a`` is the logical [K, N] u8 activation; returns [N, M]."""
    L = lib()
    a = np.ascontiguousarray(a, np.uint8)
    if a.ndim != 2 or a.shape[0] != sw.cols:
        raise ValueError(f"activation rows must equal K={sw.cols}")
    threads = threads or L.orc_max_threads()
    wd = decode(sw)
    comp = np.ascontiguousarray(wd.astype(np.int64).sum(axis=1).astype(np.int64), np.int64)
    comp = ((comp + 2**31) % 2**32 - 2**31).astype(np.int32)
    bias = _bias(sw, bias)
    n = a.shape[1]
    m = sw.logical_rows
    acc = np.empty((m, n), np.int32)
    pr = _Prog(program)
    L.orc_ref_gemm_acc(_p(wd), m, sw.cols, _p(a), n, n, _p(comp), _p(bias),
                       int(program.a_zp), _p(acc), threads)
    out = np.empty((n, m), DT_NP[pr.out_code])
    sd = _sides(n, m, sides)
    L.orc_apply_program(_p(acc), m, n, ctypes.byref(pr.s), _p(sd), _p(out), threads)
    return out


def spmm_exec(sw, a: np.ndarray, program, bias=None, sides=None, threads: int | None = None,
              bn: int = 64):
    """Tiled CPU path (spmm.py:192-333), threaded; identical bits to spmm_ref
    whenever the int32 accumulator does not overflow."""
    L = lib()
    a = np.ascontiguousarray(a, np.uint8)
    if a.ndim != 2 or a.shape[0] != sw.cols:
        raise ValueError(f"activation rows must equal K={sw.cols}")
    threads = threads or L.orc_max_threads()
    gp = np.ascontiguousarray(sw.group_ptr, np.int32)
    idx = np.ascontiguousarray(sw.idx, np.int32)
    vals = np.ascontiguousarray(sw.vals, np.int8)
    comp = row_sums(sw)
    bias = _bias(sw, bias)
    n = a.shape[1]
    m = sw.logical_rows
    pr = _Prog(program)
    out = np.empty((n, m), DT_NP[pr.out_code])
    sd = _sides(n, m, sides)
    L.orc_spmm_exec(sw.rows, sw.cols, m, _p(gp), _p(idx), _p(vals), _p(a), n, n,
                    _p(comp), _p(bias), ctypes.byref(pr.s), _p(sd), _p(out), bn, threads)
    return out


def gelu(x: np.ndarray, erf: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_gelu_array(_p(x), _p(y), x.size, 1 if erf else 0)
    return y


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---- dense f32 auxiliary operators (eltwise.py), config-4 encoder composition ----

def softmax_rows(x: np.ndarray) -> np.ndarray:
    """softmax_f32 (eltwise.py:34-59) over the last axis."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    n = x.shape[-1]
    lib().orc_softmax_rows(_p(x), _p(out), x.size // n, n)
    return out


def layer_norm(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """layer_norm_f32 (eltwise.py:62-99) over the last axis."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    gamma = np.ascontiguousarray(gamma, dtype=np.float32)
    beta = np.ascontiguousarray(beta, dtype=np.float32)
    out = np.empty_like(x)
    n = x.shape[-1]
    lib().orc_layer_norm_rows(_p(x), _p(gamma), _p(beta), float(eps), _p(out), x.size // n, n)
    return out


def batch_matmul(a: np.ndarray, b: np.ndarray, transpose_b: bool = False, alpha: float = 1.0) -> np.ndarray:
    """batch_matmul_f32 (eltwise.py:102-160): a [B, M, K], b [B, K, N] or [B, N, K]."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    bs, m, k = a.shape
    n = b.shape[1] if transpose_b else b.shape[2]
    out = np.empty((bs, m, n), np.float32)
    lib().orc_bmm(_p(a), _p(b), _p(out), bs, 1, m, k, n, m * k, 0, k, b.shape[1] * b.shape[2], 0, b.shape[2],
                  m * n, 0, n, 1 if transpose_b else 0, float(np.float32(alpha)))
    return out


def attention_context(q: np.ndarray, k: np.ndarray, v: np.ndarray, batch: int, seq: int, heads: int) -> np.ndarray:
    """Scaled dot-product attention of token-major q/k/v [batch*seq, H] per
    (sequence, head) with the reference's ops: bmm_nt * 1/sqrt(d), softmax,
    bmm_nn.  Returns the context [batch*seq, H] (heads concatenated)."""
    H = q.shape[1]
    d = H // heads
    qh = np.ascontiguousarray(q.reshape(batch, seq, heads, d).transpose(0, 2, 1, 3).reshape(-1, seq, d))
    kh = np.ascontiguousarray(k.reshape(batch, seq, heads, d).transpose(0, 2, 1, 3).reshape(-1, seq, d))
    vh = np.ascontiguousarray(v.reshape(batch, seq, heads, d).transpose(0, 2, 1, 3).reshape(-1, seq, d))
    alpha = np.float32(1.0 / np.sqrt(np.float64(d)))
    s = batch_matmul(qh, kh, transpose_b=True, alpha=alpha)
    p = softmax_rows(s)
    c = batch_matmul(p, vh)
    return np.ascontiguousarray(c.reshape(batch, heads, seq, d).transpose(0, 2, 1, 3).reshape(batch * seq, H))


def quantize(x: np.ndarray, scale, zp: int, lo: int = 0, hi: int = 255) -> np.ndarray:
    """quantize (tensor.py:140-151), per tensor."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, np.int8 if lo < 0 else np.uint8)
    lib().orc_quantize(_p(x), x.size, float(np.float32(scale)), int(zp), int(lo), int(hi), _p(out), 1 if lo < 0 else 0)
    return out
