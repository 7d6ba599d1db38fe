"""4x1 block-sparse weight format (host side).

Mirror of the reference's ``sparseinfer.sparse``
(/root/reference/pkg/src/sparseinfer/sparse.py).  ``Sparse4x1Weight`` is
kept field-for-field, so a weight encoded by either package can be handed
to the other; the GPU tile formats are *derived* from it by the plan
builder (see ``kernels.spmm.plan_spmm`` and csrc/pack.cpp), never the other
way round.

Layout (sparse.py:23-41): output rows are grouped in fours; group g's
padded block range is ``group_ptr[g]:group_ptr[g+1]``; ``idx`` holds the
ascending column of each block (padding blocks: column 0, value 0); the
values are 16-byte micro-tiles, block p / row r at
``vals[(p // 4) * 16 + r * 4 + p % 4]`` -- i.e. each tile row is one
dp4a-ready s8x4 word.  The encoder here is vectorised (no per-group
Python loop) but produces the same arrays bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class SparseFormatError(ValueError):
    """Malformed weight / encoding (sparse.py:19-20)."""


@dataclass(frozen=True)
class Sparse4x1Weight:
    """Block-compressed S8 weight, 4 output rows per group (sparse.py:23-62)."""

    rows: int            # padded to a multiple of 4
    cols: int
    logical_rows: int
    group_ptr: np.ndarray   # int32 [groups + 1]
    idx: np.ndarray         # int32 [padded blocks]
    vals: np.ndarray        # int8  [padded blocks * 4] micro-tiles
    nnz: np.ndarray         # int32 [groups] unpadded block count
    scales: np.ndarray      # float32 [logical_rows]

    @property
    def groups(self) -> int:
        return self.rows // 4

    @property
    def nnz_blocks(self) -> int:
        return int(self.nnz.sum())

    def block_values(self) -> np.ndarray:
        """[padded blocks, 4] int8: the 4 row values of every block."""
        return self.vals.reshape(-1, 4, 4).transpose(0, 2, 1).reshape(-1, 4)

    def row_sums(self) -> np.ndarray:
        """Per-row weight sums as wrapped int32 (zero-point compensation)."""
        comp = np.zeros(self.rows, np.int64)
        if len(self.idx):
            bv = self.block_values().astype(np.int64)
            g = np.repeat(np.arange(self.groups), np.diff(self.group_ptr))
            np.add.at(comp.reshape(-1, 4), g, bv)
        return comp[: self.logical_rows].astype(np.int32)


def encode_sparse(w: np.ndarray, scales: np.ndarray | None = None) -> Sparse4x1Weight:
    """Dense S8 [M, K] -> 4x1 block format (sparse.py:65-114).

    A column joins a group's list iff any of the group's 4 rows is nonzero
    there; rows pad to 4N, block lists pad to 4N with zero blocks at col 0."""
    w = np.asarray(w)
    if w.dtype != np.int8:
        raise SparseFormatError(f"expected int8 weight, got {w.dtype}")
    if w.ndim != 2 or w.shape[0] < 1 or w.shape[1] < 1:
        raise SparseFormatError(f"expected non-empty 2-D weight, got {w.shape}")
    m, k = w.shape
    rows = -(-m // 4) * 4
    groups = rows // 4
    blk = np.zeros((rows, k), np.int8)
    blk[:m] = w
    blk = blk.reshape(groups, 4, k)
    present = (blk != 0).any(axis=1)                       # [groups, k]
    nnz = present.sum(axis=1).astype(np.int32)
    padded = (nnz + 3) // 4 * 4
    ptr = np.zeros(groups + 1, np.int32)
    np.cumsum(padded, out=ptr[1:])
    total = int(ptr[-1])
    gi, ci = np.nonzero(present)                           # group-major, columns ascending
    first = np.zeros(groups + 1, np.int64)
    np.cumsum(nnz, out=first[1:])
    dest = ptr[gi].astype(np.int64) + (np.arange(gi.size) - first[gi])
    idx = np.zeros(total, np.int32)
    idx[dest] = ci
    bvals = np.zeros((total, 4), np.int8)
    bvals[dest] = blk[gi, :, ci]
    vals = np.ascontiguousarray(bvals.reshape(-1, 4, 4).transpose(0, 2, 1)).reshape(-1)
    if scales is None:
        scales = np.ones(m, np.float32)
    scales = np.asarray(scales, dtype=np.float32).reshape(-1)
    if scales.shape[0] != m:
        raise SparseFormatError("need one weight scale per logical row")
    return Sparse4x1Weight(rows=rows, cols=k, logical_rows=m, group_ptr=ptr, idx=idx,
                           vals=vals, nnz=nnz, scales=scales)


def decode_sparse(s: Sparse4x1Weight) -> np.ndarray:
    """Block format -> dense S8 [logical_rows, K] (sparse.py:117-132)."""
    if s.idx.size and (s.idx.min() < 0 or s.idx.max() >= s.cols):
        raise SparseFormatError("column index out of range")
    dense = np.zeros((s.groups, 4, s.cols), np.int16)
    if s.idx.size:
        g = np.repeat(np.arange(s.groups), np.diff(s.group_ptr))
        # accumulate: padding blocks share column 0 and must not overwrite data
        np.add.at(dense.transpose(0, 2, 1), (g, s.idx.astype(np.int64)),
                  s.block_values().astype(np.int16))
    return dense.reshape(s.rows, s.cols)[: s.logical_rows].astype(np.int8)


def sparsity_ratio(s: Sparse4x1Weight) -> float:
    """1 - nonzero blocks / block grid, padding excluded (sparse.py:135-138)."""
    return 1.0 - s.nnz_blocks / (((s.logical_rows + 3) // 4) * s.cols)


def generate_pattern_weight(m: int, k: int, target_ratio: float, seed: int = 0) -> np.ndarray:
    """Seeded dense S8 [M, K] with exactly round((1-r)*(M/4)*K) nonzero 4x1
    blocks (sparse.py:141-167).  Consumes the generator in the reference's
    order -- block choice, magnitudes in [1,127], signs -- so the same seed
    yields the same matrix."""
    if not 0.0 <= target_ratio <= 1.0:
        raise ValueError("target_ratio must be in [0, 1]")
    rng = np.random.default_rng(seed)
    groups = (m + 3) // 4
    n_blocks = min(int(round((1.0 - target_ratio) * (m / 4) * k)), groups * k)
    w = np.zeros((groups, 4, k), np.int8)
    chosen = rng.choice(groups * k, size=n_blocks, replace=False)
    if n_blocks:
        g, col = np.divmod(np.sort(chosen), k)
        mags = rng.integers(1, 128, size=(n_blocks, 4))
        signs = rng.integers(0, 2, size=(n_blocks, 4)) * 2 - 1
        w[g, :, col] = (mags * signs).astype(np.int8)
    return w.reshape(groups * 4, k)[:m].copy()
