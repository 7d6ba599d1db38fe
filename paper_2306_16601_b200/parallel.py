"""Multi-GPU sharding of the SpMM: one process per GPU.

The reference is single-process CPU; its only parallelism is the disjoint
(group-range, panel-range) task cover of partition_tasks (spmm.py:136-157),
i.e. the output splits cleanly along tokens (N) and along row groups (M).
The two multi-GPU modes are those two axes:

* ``tokens`` -- N-sharding, no collective.  Each rank owns a contiguous
  token range (or its own batch); the full plan is replicated (the packed
  weight is < 1 MB per BERT-Large linear).  Output rows [n0:n1, :] of the
  token-major [N, M] result are contiguous, so the concatenation is the
  answer.  Weak or strong scaling depending on whether N grows with ranks.
* ``rows`` -- M-sharding with one exchange step.  Each rank owns a
  contiguous range of whole 4-row groups, reads the full activation and
  produces out[:, m0:m1].  The kernel writes that block straight into the
  rank's final [N, M] output (si_spmm takes out + m0 with ldo = M), so the
  local block is never copied.  Exchange:
    - ``symm`` (NCCL groups whose GPUs can map each other's memory): the
      output lives in torch symmetric memory and every rank pushes its block
      into the same columns of each peer's buffer over NVLink (strided peer
      copies), then a barrier -- the result lands in final layout on every
      rank, with no gathered intermediate and no re-layout pass;
    - ``gather`` (gloo / no peer mapping): one all-gather of equal-size
      blocks into [world, N, Mr], then the peer blocks are written into the
      final buffer's columns.

Everything here is host bookkeeping around the product's SpMM; the per-rank
compute is injectable, so the gloo-backed CPU tests
(tests/test_parallel_gloo.py) run RowShardedSpmm itself with the oracle as
the compute.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kernels.epilogue import EpilogueProgram
from .sparse import Sparse4x1Weight


def split_range(total: int, parts: int, index: int, align: int = 1) -> tuple[int, int]:
    """Contiguous balanced split of [0, total) in units of ``align``."""
    units = -(-total // align)
    base, rem = divmod(units, parts)
    lo = index * base + min(index, rem)
    hi = lo + base + (1 if index < rem else 0)
    return min(lo * align, total), min(hi * align, total)


def token_shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Token range of ``rank`` (N-sharding)."""
    return split_range(n, world, rank)


@dataclass(frozen=True)
class RowShard:
    weight: Sparse4x1Weight
    m0: int          # first logical row owned
    m1: int          # one past the last logical row owned
    rows_pad: int    # equal per-rank row count used by the all-gather buffer


def shard_rows(sw: Sparse4x1Weight, world: int, rank: int) -> RowShard:
    """Contiguous whole-group row shard of a Sparse4x1Weight (M-sharding).

    Groups are split evenly by count; the shard is itself a valid
    Sparse4x1Weight (group_ptr rebased, idx/vals sliced), so the same plan
    builder and kernels run on it unchanged."""
    g0, g1 = split_range(sw.groups, world, rank)
    m0 = min(4 * g0, sw.logical_rows)
    m1 = min(4 * g1, sw.logical_rows)
    p0, p1 = int(sw.group_ptr[g0]), int(sw.group_ptr[g1])
    gp = (sw.group_ptr[g0: g1 + 1] - p0).astype(np.int32)
    rows = 4 * (g1 - g0)
    shard = Sparse4x1Weight(rows=max(rows, 4), cols=sw.cols, logical_rows=max(m1 - m0, 0),
                            group_ptr=gp if g1 > g0 else np.zeros(2, np.int32),
                            idx=np.ascontiguousarray(sw.idx[p0:p1]),
                            vals=np.ascontiguousarray(sw.vals[4 * p0: 4 * p1]),
                            nnz=np.ascontiguousarray(sw.nnz[g0:g1]),
                            scales=np.ascontiguousarray(sw.scales[m0:m1]))
    rows_pad = 4 * (-(-sw.groups // world))
    return RowShard(shard, m0, m1, rows_pad)


def shard_program(prog: EpilogueProgram, m0: int, m1: int) -> EpilogueProgram:
    """Slice the per-channel parts of a program to rows [m0, m1)."""
    return EpilogueProgram(scale_in=np.ascontiguousarray(prog.scale_in[m0:m1]), a_zp=prog.a_zp,
                           ops=prog.ops, fparams=prog.fparams, iparams=prog.iparams, luts=prog.luts,
                           chans=np.ascontiguousarray(prog.chans[:, m0:m1]), out_dtype=prog.out_dtype,
                           n_sides=prog.n_sides)


def assemble_rows(gathered, n: int, m: int, world: int, rows_pad: int, bounds, out=None, skip: int = -1):
    """[world, N, rows_pad] gathered blocks -> columns of the [N, M] result
    (torch or numpy).  ``out`` is written in place when given (its block
    ``skip`` is left as it is: the rank's own block is already there)."""
    try:
        import torch
        is_torch = isinstance(gathered, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_torch = False
    if out is None:
        if is_torch:
            out = torch.empty((n, m), dtype=gathered.dtype, device=gathered.device)
        else:
            out = np.empty((n, m), dtype=gathered.dtype)
    for r in range(world):
        m0, m1 = bounds[r]
        if r != skip and m1 > m0:
            out[:, m0:m1] = gathered[r, :, : m1 - m0]
    return out


def _product_compute(plan, act, out, kernel):
    from .kernels import spmm as K
    K.spmm_exec(plan, act, out=out, kernel=kernel)


class RowShardedSpmm:
    """M-sharded SpMM over a torch.distributed group (NCCL on GPUs).

    ``run(act)`` computes this rank's block of rows with the product kernel,
    written straight into the final [N, M] buffer, exchanges the blocks and
    returns the full [N, M] on every rank.  ``compute(plan, act, out_view,
    kernel)`` replaces the per-rank SpMM (tests run the bookkeeping on CPU
    with the oracle); ``exchange`` is "auto" (symm when available), "symm" or
    "gather"."""

    def __init__(self, sw: Sparse4x1Weight, n: int, program: EpilogueProgram, bias=None, group=None,
                 device=None, compute=None, exchange: str = "auto"):
        import torch
        import torch.distributed as dist

        from .kernels import spmm as K
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.m = n, sw.logical_rows
        self.shards = [shard_rows(sw, self.world, r) for r in range(self.world)]
        mine = self.shards[self.rank]
        bias = np.zeros(sw.logical_rows, np.int32) if bias is None else np.asarray(bias, np.int32)
        self.plan = K.plan_spmm(mine.weight, n, program=shard_program(program, mine.m0, mine.m1),
                                bias=bias[mine.m0: mine.m1], device=device)
        self.compute = compute or _product_compute
        self.rows_pad = mine.rows_pad
        self.bounds = [(s.m0, s.m1) for s in self.shards]
        self.dtype = K._TORCH_DT[program.out_dtype]
        dev = self.plan.image_dev.device
        self.symm = None
        if exchange in ("auto", "symm") and dev.type == "cuda" and dist.get_backend(group) == "nccl":
            try:
                import torch.distributed._symmetric_memory as symm_mem
                self.out = symm_mem.empty((n, self.m), dtype=self.dtype, device=dev)
                self.symm = symm_mem.rendezvous(self.out, group=group or dist.group.WORLD)
            except Exception:
                if exchange == "symm":
                    raise
                self.symm = None
        if self.symm is None:
            self.out = torch.empty((n, self.m), dtype=self.dtype, device=dev)
            self.local = torch.zeros((n, self.rows_pad), dtype=self.dtype, device=dev)
            self.gathered = torch.empty((self.world, n, self.rows_pad), dtype=self.dtype, device=dev)
        self.exchange = "symm" if self.symm is not None else "gather"

    def run(self, act, kernel: str = "auto"):
        m0, m1 = self.bounds[self.rank]
        if m1 > m0:
            # the kernel writes its rows straight into the final buffer's columns (ldo = M)
            self.compute(self.plan, act, self.out[:, m0:m1], kernel)
        if self.world == 1:
            return self.out
        if self.exchange == "symm":
            # push this block into the same columns of every peer's buffer
            for p in range(self.world):
                if p != self.rank and m1 > m0:
                    peer = self.symm.get_buffer(p, (self.n, self.m), self.dtype)
                    peer[:, m0:m1].copy_(self.out[:, m0:m1])
            self.symm.barrier()
            return self.out
        if m1 > m0:
            self.local[:, : m1 - m0].copy_(self.out[:, m0:m1])
        gather_rows(self.gathered, self.local, self.group)
        return assemble_rows(self.gathered, self.n, self.m, self.world, self.rows_pad, self.bounds,
                             out=self.out, skip=self.rank)


def gather_rows(gathered, local, group=None):
    """all_gather of equal-size row blocks into [world, N, rows_pad]
    (one NCCL all-gather; gloo takes the list form)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, local, group=group)
    else:
        dist.all_gather(list(gathered.unbind(0)), local, group=group)
    return gathered
