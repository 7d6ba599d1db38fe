"""Fused epilogue programs ("post-op chains") for the SpMM kernels.

Host-side mirror of the reference's ``sparseinfer.kernels.epilogue``
(/root/reference/pkg/src/sparseinfer/kernels/epilogue.py).  A program is
the reference's opcode list -- same opcodes, same parameter arrays, same
build-time state machine and errors (epilogue.py:61-182).  The device
executes it inside the SpMM store path (csrc/epilogue.cuh); the plan
builder additionally compiles maximal unary runs into exact lookup forms
(256-entry LUTs for 8-bit -> 8-bit runs, f32 breakpoint tables for
DEQ_ACC -> GELU -> QUANT), which is the paper's LUT idea (Alg. 2).

Extension (not in the reference): ``("gelu_erf",)`` -> ``OP_GELU_ERF``,
exact-erf GELU f32(0.5*x*(1+erf(x*0.7071067811865476))) in f64, which
BASELINE config 3 asks for.  Its parity is defined by the repo's oracle
only (the reference has no erf GELU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..tensor import DType, QuantParams

OP_REQUANT = 0   # s32 acc -> 8-bit space at the layer's output params
OP_LUT = 1       # int -> int through a 256-entry table
OP_DEQ = 2       # int -> f32 at given params
OP_GELU = 3      # f32 tanh-approximation GELU (epilogue.py:190-194)
OP_ADD_SIDE = 4  # f32 += side tensor element (residual)
OP_ADD_CHAN = 5  # f32 += per-output-channel constant
OP_QUANT = 6     # f32 -> int at given params
OP_DEQ_ACC = 7   # s32 acc -> f32 directly
OP_GELU_ERF = 8  # extension: exact-erf GELU

_NI = 3  # iparams per op (epilogue.py:31)


@dataclass
class EpilogueProgram:
    """Opcode arrays plus the per-channel combined input scale (epilogue.py:34-50)."""

    scale_in: np.ndarray    # f32 [M] = f32(f64(act_scale) * f64(w_scale[m]))
    a_zp: int               # activation zero point
    ops: np.ndarray         # int32 [L]
    fparams: np.ndarray     # f32 [L]
    iparams: np.ndarray     # int32 [L, 3]
    luts: np.ndarray        # u8 [n_luts, 256]
    chans: np.ndarray       # f32 [n_chans, M]
    out_dtype: DType
    n_sides: int = 0

    @property
    def m(self) -> int:
        return self.scale_in.shape[0]


class _Builder:
    """Step list -> opcode arrays; ``state`` is the type of the live value."""

    def __init__(self, m: int):
        self.m = m
        self.ops: list[int] = []
        self.fp: list[float] = []
        self.ip: list[tuple[int, int, int]] = []
        self.luts: list[np.ndarray] = []
        self.chans: list[np.ndarray] = []
        self.n_sides = 0
        self.state = "s32"
        self.out = DType.S32

    def emit(self, op, f=0.0, i=(0, 0, 0)):
        self.ops.append(op)
        self.fp.append(f)
        self.ip.append(tuple(int(v) for v in i))

    def need(self, states, msg):
        if self.state not in states:
            raise ValueError(msg)

    def to_int(self, dt: DType):
        self.state = "s8" if dt is DType.S8 else "u8"
        self.out = dt

    def to_f32(self):
        self.state = "f32"
        self.out = DType.F32


def build_program(w_scales, act_scale: float, act_zp: int, out_q: QuantParams | None,
                  steps=()) -> EpilogueProgram:
    """Assemble an epilogue program (epilogue.py:61-182).

    ``out_q`` is the layer's requantization target (None: raw S32, or f32
    through a leading ("dequantize_acc",)).  Steps, applied in order:
    ("lut", table_u8_256, in_dtype, out_dtype), ("dequantize", QuantParams),
    ("gelu",), ("gelu_erf",), ("add_side", i), ("add_channel", f32[M]),
    ("quantize", QuantParams), ("dequantize_acc",) (first step only).
    """
    w_scales = np.asarray(w_scales, dtype=np.float32).reshape(-1)
    m = w_scales.shape[0]
    scale_in = (np.float64(act_scale) * w_scales.astype(np.float64)).astype(np.float32)
    b = _Builder(m)
    if out_q is not None:
        lo, hi = out_q.dtype.bounds
        b.emit(OP_REQUANT, out_q.scale_scalar(), (out_q.zero_point, lo, hi))
        b.to_int(out_q.dtype)
    for step in steps:
        kind = step[0]
        if kind == "dequantize_acc":
            if b.state != "s32" or b.ops:
                raise ValueError("dequantize_acc must be the only entry step")
            b.emit(OP_DEQ_ACC)
            b.to_f32()
        elif kind == "lut":
            b.need(("s8", "u8"), "lut step needs an 8-bit integer state")
            table = np.asarray(step[1], dtype=np.uint8).reshape(256)
            b.emit(OP_LUT, 0.0, (len(b.luts), int(step[2] is DType.S8), int(step[3] is DType.S8)))
            b.luts.append(table)
            b.to_int(step[3])
        elif kind == "dequantize":
            b.need(("s8", "u8"), "dequantize step needs an integer state")
            q = step[1]
            b.emit(OP_DEQ, q.scale_scalar(), (q.zero_point, 0, 0))
            b.to_f32()
        elif kind in ("gelu", "gelu_erf"):
            b.need(("f32",), "gelu needs an f32 state")
            b.emit(OP_GELU if kind == "gelu" else OP_GELU_ERF)
        elif kind == "add_side":
            b.need(("f32",), "add_side needs an f32 state")
            b.emit(OP_ADD_SIDE, 0.0, (int(step[1]), 0, 0))
            b.n_sides = max(b.n_sides, int(step[1]) + 1)
        elif kind == "add_channel":
            b.need(("f32",), "add_channel needs an f32 state")
            vec = np.asarray(step[1], dtype=np.float32).reshape(-1)
            if vec.shape[0] != m:
                raise ValueError("per-channel vector length must equal M")
            b.emit(OP_ADD_CHAN, 0.0, (len(b.chans), 0, 0))
            b.chans.append(vec)
        elif kind == "quantize":
            b.need(("f32",), "quantize needs an f32 state")
            q = step[1]
            lo, hi = q.dtype.bounds
            b.emit(OP_QUANT, q.scale_scalar(), (q.zero_point, lo, hi))
            b.to_int(q.dtype)
        else:
            raise ValueError(f"unknown epilogue step {kind!r}")
    return EpilogueProgram(
        scale_in=scale_in,
        a_zp=int(act_zp),
        ops=np.asarray(b.ops, dtype=np.int32),
        fparams=np.asarray(b.fp, dtype=np.float32),
        iparams=np.asarray(b.ip, dtype=np.int32).reshape(-1, _NI),
        luts=np.stack(b.luts) if b.luts else np.zeros((0, 256), np.uint8),
        chans=np.stack(b.chans) if b.chans else np.zeros((0, m), np.float32),
        out_dtype=b.out,
        n_sides=b.n_sides,
    )


def requant_program(w_scales, act_q: QuantParams, out_q: QuantParams | None):
    """Plain requantization, or raw S32 when out_q is None (epilogue.py:185-187)."""
    return build_program(w_scales, float(act_q.scale), act_q.zero_point, out_q)


def empty_sides(n: int, m: int) -> np.ndarray:
    return np.zeros((0, n, m), np.float32)


def pack_sides(sides, n: int, m: int):
    """Stack residual inputs into the f32 [n_sides, N, M] kernel form
    (epilogue.py:256-263).  CUDA tensors stay on the device."""
    if not sides:
        return empty_sides(n, m)
    try:
        import torch
        if all(isinstance(s, torch.Tensor) for s in sides):
            return torch.stack([s.reshape(n, m).to(torch.float32) for s in sides]).contiguous()
    except ImportError:  # pragma: no cover
        pass
    return np.stack([np.asarray(s, dtype=np.float32).reshape(n, m) for s in sides])
