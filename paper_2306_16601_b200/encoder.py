"""BERT-style encoder stack on the sparse SpMM path (BASELINE config 4).

The reference package has no graph module; its SPEC describes the sparse
attention block and the post-op fusion (Fig. 3).
This module is that composition written out by hand, one layer:

    xq  = quantize(h, qp_in)                                  u8 [N, H]
    qkv = spmm(Wqkv, xq)   [DEQ_ACC]                          f32 [N, 3H]  (Q|K|V stacked: one plan)
    s   = bmm_nt(q, k) * 1/sqrt(d) per (sequence, head)       f32
    p   = softmax(s)
    ctx = bmm_nn(p, v)                                        f32 [N, H]
    cq  = quantize(ctx, qp_ctx)
    a   = spmm(Wo, cq)     [DEQ_ACC, ADD_SIDE(h)]             f32 (residual fused)
    h1  = layer_norm(a)
    h1q = quantize(h1, qp_h1)
    f   = spmm(W1, h1q)    [DEQ_ACC, GELU, QUANT(qp_f)]       u8 [N, F] (GELU + requant fused)
    g   = spmm(W2, f)      [DEQ_ACC, ADD_SIDE(h1)]            f32
    h   = layer_norm(g)                                       next layer's input

Linears are 4x1-block sparse s8 weights (generate_pattern_weight) with
per-output-channel f32 scales and int32 bias; the epilogue programs are the
reference's build_program chains, so every SpMM is bit-exact with spmm_ref
given its inputs.  The f32 ops are kernels/eltwise.py (the reference's
summation orders).  Static per-tensor u8 activation params come from one
calibration pass (compute_quant_params' U8 rule on each tensor's min/max).

Random init, seeded: there is no checkpoint (no network); BASELINE asks for
random-init weights of the BERT-Base shape.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .kernels import build_program, plan_spmm, relayout_tokens, spmm_exec
from .kernels.eltwise import attention_fused, attention_scale, bmm_strided, layer_norm_f32, quantize_f32, softmax_f32
from .sparse import encode_sparse, generate_pattern_weight
from .tensor import DType, QuantParams, u8_params_from_range


@dataclass(frozen=True)
class EncoderConfig:
    """BASELINE config 4 defaults: BERT-Base, seq 128, batch 64, 85% sparse."""

    layers: int = 12
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    seq: int = 128
    batch: int = 64
    sparsity: float = 0.85
    seed: int = 4
    eps: float = 1e-5

    @property
    def tokens(self) -> int:
        return self.batch * self.seq

    def linears(self):
        """(name, M, K) of one layer's linears (Q|K|V stacked as one weight)."""
        H, F = self.hidden, self.ffn
        return (("qkv", 3 * H, H), ("o", H, H), ("ffn1", F, H), ("ffn2", H, F))


@dataclass
class LayerWeights:
    """Host arrays of one layer (dense s8 view kept for the oracle tests)."""

    w: dict            # name -> int8 [M, K]
    w_scale: dict      # name -> f32 [M]
    bias: dict         # name -> int32 [M]
    ln1: tuple         # (gamma, beta) f32 [H]
    ln2: tuple


def make_layer_weights(cfg: EncoderConfig, layer: int) -> LayerWeights:
    """Seeded random-init weights of one layer.  Each of Q, K, V is generated
    as its own H x H linear and stacked (rows are independent outputs)."""
    H = cfg.hidden
    w, ws, b = {}, {}, {}
    parts = {"q": (H, H), "k": (H, H), "v": (H, H), "o": (H, H), "ffn1": (cfg.ffn, H), "ffn2": (H, cfg.ffn)}
    for j, (name, (m, k)) in enumerate(parts.items()):
        seed = cfg.seed * 1000 + layer * 10 + j
        w[name] = generate_pattern_weight(m, k, cfg.sparsity, seed)
        rng = np.random.default_rng(seed + 7)
        # keep activations O(1): |w| ~ 73 (uniform +-[1,127]) at density (1 - r)
        base = 1.0 / (73.0 * math.sqrt((1.0 - cfg.sparsity) * k))
        ws[name] = (base * rng.uniform(0.8, 1.2, m)).astype(np.float32)
        b[name] = rng.integers(-1000, 1001, m).astype(np.int32)
    w["qkv"] = np.concatenate([w.pop("q"), w.pop("k"), w.pop("v")])
    ws["qkv"] = np.concatenate([ws.pop("q"), ws.pop("k"), ws.pop("v")])
    b["qkv"] = np.concatenate([b.pop("q"), b.pop("k"), b.pop("v")])
    rng = np.random.default_rng(cfg.seed * 1000 + layer * 10 + 9)
    ln = [((1.0 + 0.1 * rng.standard_normal(H)).astype(np.float32), (0.1 * rng.standard_normal(H)).astype(np.float32))
          for _ in range(2)]
    return LayerWeights(w, ws, b, ln[0], ln[1])


@dataclass
class LayerQuant:
    """Static per-tensor u8 params of one layer's quantization points."""

    qp_in: QuantParams
    qp_ctx: QuantParams
    qp_h1: QuantParams
    qp_f: QuantParams


def layer_programs(lw: LayerWeights, lq: LayerQuant):
    """The four epilogue programs of a layer (reference build_program chains)."""
    return {
        "qkv": build_program(lw.w_scale["qkv"], float(lq.qp_in.scale), lq.qp_in.zero_point, None,
                             [("dequantize_acc",)]),
        "o": build_program(lw.w_scale["o"], float(lq.qp_ctx.scale), lq.qp_ctx.zero_point, None,
                           [("dequantize_acc",), ("add_side", 0)]),
        "ffn1": build_program(lw.w_scale["ffn1"], float(lq.qp_h1.scale), lq.qp_h1.zero_point, None,
                              [("dequantize_acc",), ("gelu",), ("quantize", lq.qp_f)]),
        "ffn2": build_program(lw.w_scale["ffn2"], float(lq.qp_f.scale), lq.qp_f.zero_point, None,
                              [("dequantize_acc",), ("add_side", 0)]),
    }


def _minmax_params(t: torch.Tensor) -> QuantParams:
    lo, hi = torch.aminmax(t)
    return u8_params_from_range(float(lo), float(hi))


@dataclass
class _Layer:
    weights: LayerWeights
    sw: dict                      # name -> Sparse4x1Weight
    quant: LayerQuant | None = None
    plans: dict = field(default_factory=dict)
    gamma1: torch.Tensor | None = None
    beta1: torch.Tensor | None = None
    gamma2: torch.Tensor | None = None
    beta2: torch.Tensor | None = None


class BertEncoder:
    """The config-4 stack on one GPU.  ``calibrate`` fixes the activation
    quant params (and builds the plans that depend on them); ``forward`` then
    runs the whole stack with every linear on the sparse SpMM kernels."""

    def __init__(self, cfg: EncoderConfig = EncoderConfig(), device="cuda", kernel: str = "auto",
                 weights: list | None = None, fused_attention: bool = True):
        self.cfg = cfg
        self.device = torch.device(device)
        self.kernel = kernel
        self.fused_attention = fused_attention   # si_attention_f32; False = the three separate ops
        self.layers = []
        for li in range(cfg.layers):
            lw = weights[li] if weights is not None else make_layer_weights(cfg, li)
            sw = {name: encode_sparse(lw.w[name], lw.w_scale[name]) for name, _, _ in cfg.linears()}
            L = _Layer(lw, sw)
            dev = self.device
            L.gamma1, L.beta1 = (torch.from_numpy(a).to(dev) for a in lw.ln1)
            L.gamma2, L.beta2 = (torch.from_numpy(a).to(dev) for a in lw.ln2)
            self.layers.append(L)
        self.qp_embed: QuantParams | None = None

    # ---- plans -------------------------------------------------------------
    def _plan(self, L: _Layer, name: str, prog):
        return plan_spmm(L.sw[name], self.cfg.tokens, program=prog, bias=L.weights.bias[name], device=self.device)

    def set_quant(self, quants: list, qp_embed: QuantParams | None = None):
        """Install frozen per-layer quant params (e.g. from an earlier
        calibration) and build every plan."""
        if qp_embed is not None:
            self.qp_embed = qp_embed
        for L, q in zip(self.layers, quants):
            L.quant = q
            L.plans = {k: self._plan(L, k, p) for k, p in layer_programs(L.weights, q).items()}

    # ---- the layer -----------------------------------------------------------
    def _attention(self, qkv: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        B, S, H, nh = cfg.batch, cfg.seq, cfg.hidden, cfg.heads
        d = H // nh
        ld = 3 * H
        ctx = torch.empty((B * S, H), dtype=torch.float32, device=qkv.device)
        if self.fused_attention and attention_fused(qkv, ctx, B, S, nh, d, attention_scale(d)):
            return ctx
        scores = torch.empty((B, nh, S, S), dtype=torch.float32, device=qkv.device)
        # scores[b, h] = q[b, :, h] @ k[b, :, h]^T * 1/sqrt(d); q at column h*d, k at H + h*d
        bmm_strided(qkv, qkv[:, H:], scores, B, nh, S, d, S, (S * ld, d, ld), (S * ld, d, ld),
                    (nh * S * S, S * S, S), True, attention_scale(d))
        softmax_f32(scores, out=scores)
        bmm_strided(scores, qkv[:, 2 * H:], ctx, B, nh, S, S, d, (nh * S * S, S * S, S), (S * ld, d, ld),
                    (S * H, d, H), False, 1.0)
        return ctx

    def layer_forward(self, L: _Layer, h: torch.Tensor, xq: torch.Tensor | None = None, trace: dict | None = None,
                      calibrate: bool = False):
        """One layer.  ``xq`` is the already-quantized input (else quantized
        here with qp_in).  With calibrate=True the layer's quant params are
        taken from the tensors as they are produced and the plans built."""
        cfg = self.cfg
        k = self.kernel
        if calibrate:
            qp_in = _minmax_params(h)
            L.quant = LayerQuant(qp_in, qp_in, qp_in, qp_in)   # placeholders, filled below
        q = L.quant
        if xq is None:
            xq = quantize_f32(h, q.qp_in)
        if calibrate:
            L.plans["qkv"] = self._plan(L, "qkv", layer_programs(L.weights, q)["qkv"])
        qkv = spmm_exec(L.plans["qkv"], relayout_tokens(xq), kernel=k)
        ctx = self._attention(qkv)
        if calibrate:
            q.qp_ctx = _minmax_params(ctx)
        cq = quantize_f32(ctx, q.qp_ctx)
        if calibrate:
            L.plans["o"] = self._plan(L, "o", layer_programs(L.weights, q)["o"])
        a = spmm_exec(L.plans["o"], relayout_tokens(cq), sides=h.view(1, cfg.tokens, cfg.hidden), kernel=k)
        h1 = layer_norm_f32(a, L.gamma1, L.beta1, cfg.eps)
        if calibrate:
            q.qp_h1 = _minmax_params(h1)
        h1q = quantize_f32(h1, q.qp_h1)
        if calibrate:
            # the FFN-up output params come from its f32 GELU output
            p_f32 = build_program(L.weights.w_scale["ffn1"], float(q.qp_h1.scale), q.qp_h1.zero_point, None,
                                  [("dequantize_acc",), ("gelu",)])
            g32 = spmm_exec(self._plan(L, "ffn1", p_f32), relayout_tokens(h1q), kernel=k)
            q.qp_f = _minmax_params(g32)
            del g32
            progs = layer_programs(L.weights, q)
            L.plans["ffn1"] = self._plan(L, "ffn1", progs["ffn1"])
            L.plans["ffn2"] = self._plan(L, "ffn2", progs["ffn2"])
        f = spmm_exec(L.plans["ffn1"], relayout_tokens(h1q), kernel=k)
        g = spmm_exec(L.plans["ffn2"], relayout_tokens(f), sides=h1.view(1, cfg.tokens, cfg.hidden), kernel=k)
        out = layer_norm_f32(g, L.gamma2, L.beta2, cfg.eps)
        if trace is not None:
            trace.update(xq=xq, qkv=qkv, ctx=ctx, cq=cq, a=a, h1=h1, h1q=h1q, f=f, g=g, out=out)
        return out

    def calibrate(self, x: torch.Tensor) -> list:
        """One pass over a calibration batch fixing every quant point's u8
        params (compute_quant_params' U8 rule); returns the LayerQuant list."""
        h = x
        for L in self.layers:
            h = self.layer_forward(L, h, calibrate=True)
        return [L.quant for L in self.layers]

    def forward(self, x: torch.Tensor, traces: list | None = None) -> torch.Tensor:
        """x: f32 [batch*seq, hidden] on the device -> the last layer's f32 output."""
        if any(L.quant is None for L in self.layers):
            raise RuntimeError("calibrate() or set_quant() first")
        h = x
        for L in self.layers:
            tr = {} if traces is not None else None
            h = self.layer_forward(L, h, trace=tr)
            if traces is not None:
                traces.append(tr)
        return h

    __call__ = forward


def embeddings(cfg: EncoderConfig, seed: int = 0) -> np.ndarray:
    """BASELINE config 4 input: f32 embeddings N(0, 1), [batch*seq, hidden]."""
    return np.random.default_rng(seed).standard_normal((cfg.tokens, cfg.hidden)).astype(np.float32)


def spmm_ops(cfg: EncoderConfig) -> float:
    """Effective SpMM ops of one forward (2*nnz*N over every linear)."""
    total = 0.0
    for name, m, k in cfg.linears():
        nb = round((1.0 - cfg.sparsity) * (m / 4) * k) if name != "qkv" else 3 * round(
            (1.0 - cfg.sparsity) * (cfg.hidden / 4) * k)
        total += 2.0 * 4 * nb * cfg.tokens
    return total * cfg.layers
