"""Config-4 encoder path: the dense f32 auxiliary ops and the layer
composition, checked against golden vectors the reference itself produced
(tests/golden/make_golden_eltwise.py).

CPU: the C oracle's restatement of eltwise.py / quantize, and the oracle
composition (tests/encoder_recipe.py), bit for bit against the reference.
GPU: the device kernels and paper_2306_16601_b200.encoder.BertEncoder against
the same golden vectors (per op with the golden inputs, and end to end), plus
the BERT-Base-sized stack of BASELINE config 4 (calibrate + forward).
"""

import os

import numpy as np
import pytest

import encoder_recipe
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200.encoder import EncoderConfig, LayerQuant, make_layer_weights
from paper_2306_16601_b200.kernels import build_program
from paper_2306_16601_b200.tensor import DType, QuantParams

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "eltwise_cases.npz"))
TOY = EncoderConfig(layers=2, hidden=64, heads=4, ffn=128, seq=16, batch=2, sparsity=0.85, seed=3)
QNAMES = ("qp_in", "qp_ctx", "qp_h1", "qp_f")


def _qp(arr):
    return QuantParams(np.int32(arr[0]).view(np.float32), int(arr[1]), DType.U8)


def golden_quant(li):
    return {k: _qp(G[f"enc{li}_{k}"]) for k in QNAMES}


class OracleOps:
    """The C oracle behind the recipe's ops namespace."""

    @staticmethod
    def quantize(x, qp):
        return oracle.quantize(x, qp.scale, qp.zero_point)

    @staticmethod
    def calibrate(x):
        return P.compute_quant_params(x)

    @staticmethod
    def spmm(sw, x_kn, prog, bias, sides):
        return oracle.spmm_ref(sw, x_kn, prog, bias, sides)

    @staticmethod
    def bmm(a, b, transpose_b, alpha):
        return oracle.batch_matmul(a, b, transpose_b, alpha)

    @staticmethod
    def softmax(x):
        return oracle.softmax_rows(x)

    @staticmethod
    def layer_norm(x, g, b, eps):
        return oracle.layer_norm(x, g, b, eps)

    @staticmethod
    def encode(w, scales):
        return P.encode_sparse(w, scales)

    @staticmethod
    def build_program(*a):
        return build_program(*a)


def _n(prefix):
    return sorted({k.split("_")[0] for k in G.files if k.startswith(prefix)})


# ---------------------------------------------------------------- CPU: oracle pinned
@pytest.mark.parametrize("case", _n("softmax"))
def test_oracle_softmax_matches_reference(case):
    np.testing.assert_array_equal(oracle.softmax_rows(G[f"{case}_x"]), G[f"{case}_y"])


@pytest.mark.parametrize("case", _n("ln"))
def test_oracle_layer_norm_matches_reference(case):
    y = oracle.layer_norm(G[f"{case}_x"], G[f"{case}_g"], G[f"{case}_b"], float(G[f"{case}_eps"]))
    np.testing.assert_array_equal(y, G[f"{case}_y"])


@pytest.mark.parametrize("case", _n("bmm"))
def test_oracle_bmm_matches_reference(case):
    y = oracle.batch_matmul(G[f"{case}_a"], G[f"{case}_b"], bool(G[f"{case}_meta"][0]), float(G[f"{case}_alpha"]))
    np.testing.assert_array_equal(y, G[f"{case}_y"])


@pytest.mark.parametrize("case", ["q0", "q1", "q2"])
def test_calibration_and_quantize_match_reference(case):
    x = G[f"{case}_x"]
    qp = P.compute_quant_params(x)
    want = _qp(G[f"{case}_params"])
    assert np.float32(qp.scale) == np.float32(want.scale) and qp.zero_point == want.zero_point
    np.testing.assert_array_equal(oracle.quantize(x, qp.scale, qp.zero_point), G[f"{case}_y"])


def test_oracle_encoder_composition_matches_reference():
    """The recipe on the C oracle reproduces the reference-composed toy
    encoder bit for bit (every intermediate of both layers, calibration
    included)."""
    h = G["enc_x"]
    for li in range(TOY.layers):
        lw = make_layer_weights(TOY, li)
        lq = {}
        h, t = encoder_recipe.layer(OracleOps, lw, lq, h, TOY, calibrate=True)
        for k in QNAMES:
            assert np.float32(lq[k].scale) == np.float32(_qp(G[f"enc{li}_{k}"]).scale), (li, k)
            assert lq[k].zero_point == int(G[f"enc{li}_{k}"][1]), (li, k)
        for k, v in t.items():
            np.testing.assert_array_equal(v, G[f"enc{li}_{k}"], err_msg=f"layer {li} {k}")


# ---------------------------------------------------------------- GPU
def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.gpu
def test_gpu_eltwise_ops_match_reference():
    from paper_2306_16601_b200.kernels import eltwise as E
    for c in _n("ln"):
        y = E.layer_norm_f32(_cuda(G[f"{c}_x"]), _cuda(G[f"{c}_g"]), _cuda(G[f"{c}_b"]), float(G[f"{c}_eps"]))
        np.testing.assert_array_equal(y.cpu().numpy(), G[f"{c}_y"], err_msg=c)
    for c in _n("bmm"):
        y = E.batch_matmul_f32(_cuda(G[f"{c}_a"]), _cuda(G[f"{c}_b"]), bool(G[f"{c}_meta"][0]),
                               float(G[f"{c}_alpha"]))
        np.testing.assert_array_equal(y.cpu().numpy(), G[f"{c}_y"], err_msg=c)
    for c in _n("softmax"):
        # f64 exp: CUDA's vs glibc's may differ in the last f64 ulp, which
        # moves an f32 result by at most one ulp, rarely
        y = E.softmax_f32(_cuda(G[f"{c}_x"])).cpu().numpy()
        np.testing.assert_allclose(y, G[f"{c}_y"], rtol=1e-6, atol=0, err_msg=c)
        assert np.mean(y == G[f"{c}_y"]) > 0.99
    for c in ["q0", "q1", "q2"]:
        qp = _qp(G[f"{c}_params"])
        y = E.quantize_f32(_cuda(G[f"{c}_x"]), qp)
        np.testing.assert_array_equal(y.cpu().numpy(), G[f"{c}_y"], err_msg=c)


def _toy_encoder():
    from paper_2306_16601_b200.encoder import BertEncoder
    enc = BertEncoder(TOY, device="cuda")
    enc.set_quant([LayerQuant(**golden_quant(li)) for li in range(TOY.layers)])
    return enc


@pytest.mark.gpu
def test_gpu_encoder_ops_teacher_forced():
    """Each device op of each layer, fed the reference's own inputs, against
    the reference's output: SpMMs and integer outputs bit-exact, f32 within
    1e-5 relative."""
    enc = _toy_encoder()
    from paper_2306_16601_b200.kernels import relayout_tokens, spmm_exec
    from paper_2306_16601_b200.kernels import eltwise as E
    for li, L in enumerate(enc.layers):
        g = {k: G[f"enc{li}_{k}"] for k in ("xq", "qkv", "ctx", "cq", "a", "h1", "h1q", "f", "g", "out")}
        h_in = G["enc_x"] if li == 0 else G[f"enc{li - 1}_out"]
        q = L.quant
        np.testing.assert_array_equal(E.quantize_f32(_cuda(h_in), q.qp_in).cpu().numpy(), g["xq"])
        qkv = spmm_exec(L.plans["qkv"], relayout_tokens(_cuda(g["xq"])))
        np.testing.assert_array_equal(qkv.cpu().numpy(), g["qkv"])
        ctx = enc._attention(_cuda(g["qkv"])).cpu().numpy()
        np.testing.assert_allclose(ctx, g["ctx"], rtol=1e-5, atol=1e-6)
        a = spmm_exec(L.plans["o"], relayout_tokens(_cuda(g["cq"])), sides=_cuda(h_in)[None])
        np.testing.assert_array_equal(a.cpu().numpy(), g["a"])
        np.testing.assert_array_equal(E.layer_norm_f32(_cuda(g["a"]), L.gamma1, L.beta1, TOY.eps).cpu().numpy(),
                                      g["h1"])
        f = spmm_exec(L.plans["ffn1"], relayout_tokens(_cuda(g["h1q"])))
        np.testing.assert_array_equal(f.cpu().numpy(), g["f"])
        gg = spmm_exec(L.plans["ffn2"], relayout_tokens(_cuda(g["f"])), sides=_cuda(g["h1"])[None])
        np.testing.assert_array_equal(gg.cpu().numpy(), g["g"])


@pytest.mark.gpu
def test_gpu_encoder_end_to_end():
    """The whole toy stack on the device from the embeddings: final f32
    within 1e-5 relative of the reference (softmax's f64 exp may move a u8
    rounding point; then a layer's output moves by one quantization step at
    such elements, so the comparison allows a small fraction of them)."""
    enc = _toy_encoder()
    traces = []
    out = enc.forward(_cuda(G["enc_x"]), traces=traces).cpu().numpy()
    want = G[f"enc{TOY.layers - 1}_out"]
    close = np.isclose(out, want, rtol=1e-5, atol=1e-5)
    assert close.mean() > 0.999, f"{(~close).sum()} elements differ"
    for li, t in enumerate(traces):
        assert np.array_equal(t["xq"].cpu().numpy(), G[f"enc{li}_xq"]) or li > 0


@pytest.mark.gpu
def test_gpu_bert_base_stack_full_parity():
    """BASELINE config 4 at full size (12 layers x 768/3072, 12 heads, seq
    128, batch 64 = 8192 tokens, 85% sparse) against the C oracle, every
    element of every intermediate of every layer.

    Teacher forcing with the device's own tensors: each oracle op is fed the
    device's input of that op, so an op either reproduces the device output
    or the test names it.  Quantize, all four SpMMs (u8 GELU table and the
    residual epilogues included) and both LayerNorms must match bit for bit.
    The attention context is the one f32 tensor with a libm boundary: the
    reference's softmax takes f64 exp (glibc here, CUDA's exp on the
    device), so it is compared within 1e-5 relative.  Because the chain
    starts from the embeddings and every other op is exact, the device's
    final output equals the oracle composition with the device's attention
    contexts injected -- the only divergence class is that exp."""
    from paper_2306_16601_b200.encoder import BertEncoder, EncoderConfig, embeddings, layer_programs
    cfg = EncoderConfig()
    enc = BertEncoder(cfg, device="cuda")
    x = embeddings(cfg, 0)
    enc.calibrate(_cuda(x))
    traces = []
    enc.forward(_cuda(x), traces=traces)
    h_in = x
    ctx_diff = 0
    for li, (L, t) in enumerate(zip(enc.layers, traces)):
        q, lw = L.quant, L.weights
        tt = {k: v.cpu().numpy() for k, v in t.items()}
        progs = layer_programs(lw, q)

        def spmm(name, x_tok, sides=None):
            return oracle.spmm_exec(L.sw[name], np.ascontiguousarray(x_tok.T), progs[name], lw.bias[name],
                                    sides=sides)

        def same(got, want, what):
            assert got.dtype == want.dtype and np.array_equal(got, want), \
                f"layer {li} {what}: {int((got != want).sum())} elements differ"

        same(tt["xq"], oracle.quantize(h_in, q.qp_in.scale, q.qp_in.zero_point), "quantize(h)")
        same(tt["qkv"], spmm("qkv", tt["xq"]), "QKV SpMM")
        H = cfg.hidden
        ctx_ref = oracle.attention_context(tt["qkv"][:, :H], tt["qkv"][:, H:2 * H], tt["qkv"][:, 2 * H:],
                                           cfg.batch, cfg.seq, cfg.heads)
        np.testing.assert_allclose(tt["ctx"], ctx_ref, rtol=1e-5, atol=1e-6, err_msg=f"layer {li} attention")
        ctx_diff += int((tt["ctx"] != ctx_ref).sum())
        same(tt["cq"], oracle.quantize(tt["ctx"], q.qp_ctx.scale, q.qp_ctx.zero_point), "quantize(ctx)")
        same(tt["a"], spmm("o", tt["cq"], sides=h_in[None]), "O SpMM + residual")
        same(tt["h1"], oracle.layer_norm(tt["a"], lw.ln1[0], lw.ln1[1], cfg.eps), "LayerNorm 1")
        same(tt["h1q"], oracle.quantize(tt["h1"], q.qp_h1.scale, q.qp_h1.zero_point), "quantize(h1)")
        same(tt["f"], spmm("ffn1", tt["h1q"]), "FFN-up SpMM (GELU -> u8)")
        same(tt["g"], spmm("ffn2", tt["f"], sides=tt["h1"][None]), "FFN-down SpMM + residual")
        same(tt["out"], oracle.layer_norm(tt["g"], lw.ln2[0], lw.ln2[1], cfg.eps), "LayerNorm 2")
        h_in = tt["out"]
    # the attention contexts are close, not identical, only through exp
    assert ctx_diff < 0.01 * cfg.layers * cfg.tokens * cfg.hidden


@pytest.mark.gpu
def test_gpu_bert_base_stack_config4():
    """BASELINE config 4 at full size (12 layers, hidden 768, 12 heads, FFN
    3072, seq 128, batch 64, 85% sparse): calibrate on the batch, run the
    stack twice; deterministic, finite, LayerNorm-shaped output."""
    import torch
    from paper_2306_16601_b200.encoder import BertEncoder, embeddings
    cfg = EncoderConfig()
    enc = BertEncoder(cfg, device="cuda")
    x = _cuda(embeddings(cfg, 0))
    quants = enc.calibrate(x)
    assert len(quants) == cfg.layers
    y1 = enc.forward(x)
    y2 = enc.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.isfinite(y1).all()
    L = enc.layers[-1]
    # LayerNorm output: per-row mean of (y - beta)/gamma ~ 0
    z = (y1 - L.beta2) / L.gamma2
    assert float(z.mean(dim=1).abs().max()) < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("batch,seq,heads,d,pad", [(2, 128, 12, 64, 0), (2, 128, 12, 64, 5), (3, 77, 3, 48, 4),
                                                   (1, 1, 2, 8, 0), (4, 128, 2, 33, 5), (2, 5, 1, 64, 4)])
def test_gpu_fused_attention_equals_separate_ops(batch, seq, heads, d, pad):
    """si_attention_f32 (scores, softmax and context in one CTA per
    (sequence, head)) against the three separate ops: bit-equal, including
    ragged seq / head_dim and qkv / ctx row strides wider than the data
    (16-byte-aligned strides take the vector load path, the rest the scalar)."""
    import torch
    from paper_2306_16601_b200.kernels import eltwise as E
    H = heads * d
    rng = np.random.default_rng(seq * 7 + d)
    qkv = _cuda(rng.normal(0, 2, (batch * seq, 3 * H + pad)).astype(np.float32))
    alpha = E.attention_scale(d)
    fused = torch.zeros((batch * seq, H + 3), dtype=torch.float32, device="cuda")
    assert E.attention_fused(qkv, fused, batch, seq, heads, d, alpha)
    ld = qkv.stride(0)
    scores = torch.empty((batch, heads, seq, seq), dtype=torch.float32, device="cuda")
    E.bmm_strided(qkv, qkv[:, H:], scores, batch, heads, seq, d, seq, (seq * ld, d, ld), (seq * ld, d, ld),
                  (heads * seq * seq, seq * seq, seq), True, alpha)
    E.softmax_f32(scores, out=scores)
    ctx = torch.zeros((batch * seq, H + 3), dtype=torch.float32, device="cuda")
    E.bmm_strided(scores, qkv[:, 2 * H:], ctx, batch, heads, seq, seq, d, (heads * seq * seq, seq * seq, seq),
                  (seq * ld, d, ld), (seq * (H + 3), d, H + 3), False, 1.0)
    assert torch.equal(fused, ctx)


@pytest.mark.gpu
def test_gpu_fused_attention_unsupported_shape():
    import torch
    from paper_2306_16601_b200.kernels import eltwise as E
    qkv = torch.zeros((129, 3 * 64), dtype=torch.float32, device="cuda")
    ctx = torch.zeros((129, 64), dtype=torch.float32, device="cuda")
    assert not E.attention_fused(qkv, ctx, 1, 129, 1, 64, 0.125)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,n", [(70, 768), (33, 1024), (5, 4), (64, 12), (31, 770), (1, 3072)])
def test_gpu_layer_norm_paths_match_oracle(rows, n):
    """Both LayerNorm kernels (bulk-copy rows for n % 4 == 0, else the
    staged-lane kernel) against the oracle, bit for bit, on ragged row
    counts."""
    from paper_2306_16601_b200.kernels import eltwise as E
    rng = np.random.default_rng(rows * 31 + n)
    x = (rng.normal(0, 3, (rows, n)) + rng.normal(0, 5, (rows, 1))).astype(np.float32)
    g = rng.normal(1, 0.2, n).astype(np.float32)
    b = rng.normal(0, 0.2, n).astype(np.float32)
    y = E.layer_norm_f32(_cuda(x), _cuda(g), _cuda(b), 1e-12).cpu().numpy()
    np.testing.assert_array_equal(y, oracle.layer_norm(x, g, b, 1e-12))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4096, 4099, 8, 3])
def test_gpu_quantize_paths_match_oracle(n):
    """The four-per-thread quantize (n % 4 == 0) and the scalar one, u8 and
    s8, against the oracle, bit for bit."""
    from paper_2306_16601_b200.kernels import eltwise as E
    x = np.random.default_rng(n).normal(0, 40, n).astype(np.float32)
    for dt, lo, hi, zp in ((DType.U8, 0, 255, 128), (DType.S8, -128, 127, 0)):
        qp = QuantParams(np.float32(0.37), zp, dt)
        y = E.quantize_f32(_cuda(x), qp).cpu().numpy()
        np.testing.assert_array_equal(y, oracle.quantize(x, np.float32(0.37), zp, lo, hi))
