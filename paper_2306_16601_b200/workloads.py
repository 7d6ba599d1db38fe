"""Seeded synthetic workloads for the BASELINE.json configs.

No dataset is involved: BASELINE's five configs are synthetic by definition
(SURVEY.md 8(d)).  One seed drives every array of a cell:

  W      generate_pattern_weight(M, K, ratio, seed)   exact block count, values +-[1,127]
  X      default_rng(seed+1).integers(0, 256, (K, N), u8)
  bias   default_rng(seed+2).integers(-1000, 1001, M) as int32
  scale  then, same generator, uniform(1e-4, 1e-3, M) as f32 (per output channel)

tests/golden/make_golden.py uses the identical recipe with the reference's
own generator, so hash pins taken from the reference apply to these inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kernels.epilogue import build_program
from .sparse import generate_pattern_weight
from .tensor import DType, QuantParams


def baseline_inputs(m: int, k: int, n: int, ratio: float, seed: int, with_x: bool = True):
    w = generate_pattern_weight(m, k, ratio, seed)
    x = np.random.default_rng(seed + 1).integers(0, 256, (k, n), dtype=np.uint8) if with_x else None
    rng = np.random.default_rng(seed + 2)
    bias = rng.integers(-1000, 1001, m).astype(np.int32)
    scales = rng.uniform(1e-4, 1e-3, m).astype(np.float32)
    return w, x, bias, scales


def program(kind: str, scales: np.ndarray, a_zp: int = 0):
    """Epilogue programs of the BASELINE configs."""
    if kind == "s32":
        return build_program(scales, 1.0, a_zp, None)
    if kind == "deq_f32":
        return build_program(scales, 1.0, a_zp, None, [("dequantize_acc",)])
    if kind in ("gelu_erf_u8", "gelu_tanh_u8"):
        g = "gelu_erf" if kind == "gelu_erf_u8" else "gelu"
        return build_program(scales, 1.0, a_zp, None,
                             [("dequantize_acc",), (g,),
                              ("quantize", QuantParams(np.float32(0.05), 0, DType.U8))])
    if kind == "requant_u8":
        # config 5: BASELINE gives no requant params; scale 2.0 / zp 128 keeps
        # >= 92% of outputs off the clamps on all three shapes (SURVEY probe9)
        return build_program(scales, 1.0, a_zp, QuantParams(np.float32(2.0), 128, DType.U8))
    raise KeyError(kind)


@dataclass(frozen=True)
class Cell:
    name: str
    m: int
    k: int
    n: int
    ratio: float
    seed: int
    program: str

    def nb(self) -> int:
        """Nonzero 4x1 blocks (sparse.py:155)."""
        return min(int(round((1.0 - self.ratio) * (self.m / 4) * self.k)), ((self.m + 3) // 4) * self.k)

    def ops(self, n: int | None = None) -> float:
        """Effective ops 2*nnz*N, nnz = 4*nb (BASELINE metric)."""
        return 2.0 * 4 * self.nb() * (self.n if n is None else n)

    def out_bytes(self) -> int:
        return 4 if self.program in ("s32", "deq_f32") else 1

    def hbm_bytes(self, n: int | None = None) -> float:
        """Algorithmic bytes per call: X + values + u16 column
        per block + group pointers + bias/scale + output."""
        n = self.n if n is None else n
        nb = self.nb()
        return (self.k * n + 4 * nb + 2 * nb + 4 * ((self.m + 3) // 4 + 1) + 8 * self.m
                + self.m * n * self.out_bytes())


CONFIG1 = [Cell("c1_s32", 768, 768, 128, 0.9, 11, "s32"), Cell("c1_f32", 768, 768, 128, 0.9, 11, "deq_f32")]
CONFIG3 = Cell("c3_ffn_up", 3072, 768, 4096, 0.8, 13, "gelu_erf_u8")
CONFIG5 = [Cell("c5a_1024x1024", 1024, 1024, 65536, 0.9, 15, "requant_u8"),
           Cell("c5b_4096x1024", 4096, 1024, 65536, 0.9, 17, "requant_u8"),
           Cell("c5c_1024x4096", 1024, 4096, 65536, 0.9, 19, "requant_u8")]
CONFIG2_SHAPES = [(256, 256), (768, 768), (3072, 768), (768, 3072), (1024, 1024), (4096, 1024), (1024, 4096)]
CONFIG2_N = [128, 512, 2048, 8192]
CONFIG2_RATIOS = [0.70, 0.75, 0.80, 0.85, 0.90]


def config2_cells():
    out = []
    for i, (m, k) in enumerate(CONFIG2_SHAPES):
        for n in CONFIG2_N:
            for j, r in enumerate(CONFIG2_RATIOS):
                out.append(Cell(f"c2_{m}x{k}_n{n}_r{int(r * 100)}", m, k, n, r, 200 + 10 * i + j, "deq_f32"))
    return out
