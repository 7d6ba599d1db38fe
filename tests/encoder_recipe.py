"""The config-4 encoder layer written once against an "ops" namespace, so the
same composition runs on the reference's own kernels (tests/golden/
make_golden_eltwise.py, in the build container) and on the C oracle
(tests/test_encoder.py) -- the composition paper_2306_16601_b200/encoder.py
runs on the GPU.  Test infrastructure only.

ops must provide: quantize(x, qp) -> u8, spmm(sw, x_kn_u8, program, bias,
sides) -> [N, M], bmm(a, b, transpose_b, alpha), softmax(x), layer_norm(x,
gamma, beta, eps), encode(w, scales) -> weight, build_program(...),
calibrate(x) -> QuantParams-like (scale, zero_point).
"""

import math

import numpy as np


def attention(ops, qkv, batch, seq, heads):
    H = qkv.shape[1] // 3
    d = H // heads
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]

    def split(t):
        return np.ascontiguousarray(t.reshape(batch, seq, heads, d).transpose(0, 2, 1, 3).reshape(-1, seq, d))
    alpha = np.float32(1.0 / math.sqrt(float(d)))
    s = ops.bmm(split(q), split(k), True, alpha)
    p = ops.softmax(s)
    c = ops.bmm(p, split(v), False, np.float32(1.0))
    return np.ascontiguousarray(c.reshape(batch, heads, seq, d).transpose(0, 2, 1, 3).reshape(batch * seq, H))


def layer(ops, lw, lq, h, cfg, calibrate=False):
    """One layer (paper_2306_16601_b200/encoder.py docstring).  lq: dict with
    qp_in, qp_ctx, qp_h1, qp_f (filled in when calibrate=True).  Returns
    (out, intermediates)."""
    t = {}
    if calibrate:
        lq["qp_in"] = ops.calibrate(h)
    xq = ops.quantize(h, lq["qp_in"])
    sw = {n: ops.encode(lw.w[n], lw.w_scale[n]) for n in ("qkv", "o", "ffn1", "ffn2")}
    bp = ops.build_program
    p_qkv = bp(lw.w_scale["qkv"], float(lq["qp_in"].scale), lq["qp_in"].zero_point, None, [("dequantize_acc",)])
    qkv = ops.spmm(sw["qkv"], np.ascontiguousarray(xq.T), p_qkv, lw.bias["qkv"], None)
    ctx = attention(ops, qkv, cfg.batch, cfg.seq, cfg.heads)
    if calibrate:
        lq["qp_ctx"] = ops.calibrate(ctx)
    cq = ops.quantize(ctx, lq["qp_ctx"])
    p_o = bp(lw.w_scale["o"], float(lq["qp_ctx"].scale), lq["qp_ctx"].zero_point, None,
             [("dequantize_acc",), ("add_side", 0)])
    a = ops.spmm(sw["o"], np.ascontiguousarray(cq.T), p_o, lw.bias["o"], h[None])
    h1 = ops.layer_norm(a, lw.ln1[0], lw.ln1[1], cfg.eps)
    if calibrate:
        lq["qp_h1"] = ops.calibrate(h1)
    h1q = ops.quantize(h1, lq["qp_h1"])
    if calibrate:
        p_g = bp(lw.w_scale["ffn1"], float(lq["qp_h1"].scale), lq["qp_h1"].zero_point, None,
                 [("dequantize_acc",), ("gelu",)])
        lq["qp_f"] = ops.calibrate(ops.spmm(sw["ffn1"], np.ascontiguousarray(h1q.T), p_g, lw.bias["ffn1"], None))
    p_f = bp(lw.w_scale["ffn1"], float(lq["qp_h1"].scale), lq["qp_h1"].zero_point, None,
             [("dequantize_acc",), ("gelu",), ("quantize", lq["qp_f"])])
    f = ops.spmm(sw["ffn1"], np.ascontiguousarray(h1q.T), p_f, lw.bias["ffn1"], None)
    p_2 = bp(lw.w_scale["ffn2"], float(lq["qp_f"].scale), lq["qp_f"].zero_point, None,
             [("dequantize_acc",), ("add_side", 0)])
    g = ops.spmm(sw["ffn2"], np.ascontiguousarray(f.T), p_2, lw.bias["ffn2"], h1[None])
    out = ops.layer_norm(g, lw.ln2[0], lw.ln2[1], cfg.eps)
    t.update(xq=xq, qkv=qkv, ctx=ctx, cq=cq, a=a, h1=h1, h1q=h1q, f=f, g=g, out=out)
    return out, t
