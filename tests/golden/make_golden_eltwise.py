"""Golden vectors for the config-4 encoder path, produced by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_eltwise.py

Imports the reference package (pure Python + numba, nothing copied) and
writes tests/golden/eltwise_cases.npz:

  * softmax_f32 / layer_norm_f32 / batch_matmul_f32 (NN and NT) / quantize
    and compute_quant_params on seeded inputs, with the reference's outputs;
  * a 2-layer toy encoder (hidden 64, 4 heads, FFN 128, seq 16, batch 2, 85%
    sparse) composed from the reference's own spmm_ref / build_program /
    eltwise kernels by tests/encoder_recipe.py (the composition
    paper_2306_16601_b200/encoder.py runs on the GPU), calibrated with the
    reference's compute_quant_params: every intermediate and the frozen quant
    params are stored.  Weights come from the package's seeded
    make_layer_weights (generate_pattern_weight is pinned against the
    reference's by golden_pins.json).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import sparseinfer as si  # noqa: E402
import sparseinfer.kernels as sk  # noqa: E402
from sparseinfer.tensor import DType, Granularity  # noqa: E402

import encoder_recipe  # noqa: E402
from paper_2306_16601_b200.encoder import EncoderConfig, make_layer_weights  # noqa: E402

TOY = EncoderConfig(layers=2, hidden=64, heads=4, ffn=128, seq=16, batch=2, sparsity=0.85, seed=3)


class RefOps:
    """The reference's own kernels behind the recipe's ops namespace."""

    @staticmethod
    def quantize(x, qp):
        return si.quantize(x, qp)

    @staticmethod
    def calibrate(x):
        return si.compute_quant_params(x, Granularity.PER_TENSOR, DType.U8)

    @staticmethod
    def spmm(sw, x_kn, prog, bias, sides):
        return sk.spmm_ref(sw, x_kn, program=prog, bias=bias, sides=sides)

    @staticmethod
    def bmm(a, b, transpose_b, alpha):
        return sk.batch_matmul_f32(a, b, transpose_b=transpose_b, alpha=float(alpha))

    @staticmethod
    def softmax(x):
        return sk.softmax_f32(x)

    @staticmethod
    def layer_norm(x, g, b, eps):
        return sk.layer_norm_f32(x, g, b, eps)

    @staticmethod
    def encode(w, scales):
        return si.encode_sparse(w, scales)

    @staticmethod
    def build_program(*a):
        return sk.build_program(*a)


def main():
    rng = np.random.default_rng(2024)
    out = {}
    # softmax: ragged widths, wide value ranges
    for i, (r, n, sd) in enumerate([(7, 128, 3.0), (5, 1, 1.0), (9, 33, 20.0), (4, 16, 0.01)]):
        x = (sd * rng.standard_normal((r, n))).astype(np.float32)
        out[f"softmax{i}_x"] = x
        out[f"softmax{i}_y"] = sk.softmax_f32(x)
    # layer norm
    for i, (r, n, eps) in enumerate([(6, 768, 1e-5), (5, 7, 1e-12), (3, 64, 1e-5)]):
        x = (2.0 * rng.standard_normal((r, n)) + 0.5).astype(np.float32)
        g = (1.0 + 0.1 * rng.standard_normal(n)).astype(np.float32)
        b = (0.1 * rng.standard_normal(n)).astype(np.float32)
        out[f"ln{i}_x"], out[f"ln{i}_g"], out[f"ln{i}_b"] = x, g, b
        out[f"ln{i}_eps"] = np.float64(eps)
        out[f"ln{i}_y"] = sk.layer_norm_f32(x, g, b, eps)
    # batch matmul
    for i, (bs, m, k, n, tb, alpha) in enumerate([(3, 16, 8, 16, True, 0.125), (2, 16, 16, 8, False, 1.0),
                                                  (1, 5, 33, 7, False, 0.5), (2, 9, 4, 3, True, 2.0)]):
        a = rng.standard_normal((bs, m, k)).astype(np.float32)
        b = rng.standard_normal((bs, n, k) if tb else (bs, k, n)).astype(np.float32)
        out[f"bmm{i}_a"], out[f"bmm{i}_b"] = a, b
        out[f"bmm{i}_meta"] = np.array([1 if tb else 0], np.int32)
        out[f"bmm{i}_alpha"] = np.float32(alpha)
        out[f"bmm{i}_y"] = sk.batch_matmul_f32(a, b, transpose_b=tb, alpha=alpha)
    # calibration + quantize
    for i, sd in enumerate([1.0, 7.5, 0.003]):
        x = (sd * rng.standard_normal(1000) + 0.3 * sd).astype(np.float32)
        qp = si.compute_quant_params(x, Granularity.PER_TENSOR, DType.U8)
        out[f"q{i}_x"] = x
        out[f"q{i}_params"] = np.array([np.float32(qp.scale).view(np.int32), qp.zero_point], np.int64)
        out[f"q{i}_y"] = si.quantize(x, qp)
    # toy encoder through the reference's kernels
    cfg = TOY
    h = np.random.default_rng(5).standard_normal((cfg.tokens, cfg.hidden)).astype(np.float32)
    out["enc_x"] = h
    for li in range(cfg.layers):
        lw = make_layer_weights(cfg, li)
        lq = {}
        h, t = encoder_recipe.layer(RefOps, lw, lq, h, cfg, calibrate=True)
        for k, qp in lq.items():
            out[f"enc{li}_{k}"] = np.array([np.float32(qp.scale).view(np.int32), qp.zero_point], np.int64)
        for k, v in t.items():
            out[f"enc{li}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "eltwise_cases.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
