"""Multi-process (world_size 2 and 3, gloo on CPU) tests of the sharding
bookkeeping.

Rows mode runs the product's RowShardedSpmm itself -- plan per shard, the
rank's block written into the final [N, M] buffer's columns, the all-gather
exchange and the column placement of the peer blocks -- with the C oracle
injected as the per-rank compute (no GPU in this container); on a GPU box the
same object runs the product kernel (tests/test_gpu_parallel.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_16601_b200 import encode_sparse, parallel, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, k, n = 70, 96, 50   # M not a multiple of world*4, odd N
        w, x, bias, scales = workloads.baseline_inputs(m, k, n, 0.7, 31)
        sw = encode_sparse(w, scales)
        prog = workloads.program("requant_u8", scales, a_zp=2)
        full = oracle.spmm_exec(sw, x, prog, bias)
        if mode == "rows":
            def oracle_compute(plan, act_kn, out_view, kernel):
                out_view[...] = torch.from_numpy(oracle.spmm_exec(plan.weight, act_kn, plan.program, plan.bias))
            rs = parallel.RowShardedSpmm(sw, n, prog, bias=bias, device="cpu", compute=oracle_compute)
            assert rs.exchange == "gather"
            got = rs.run(x).numpy()
            got2 = rs.run(x).numpy()   # reusable across calls
            assert np.array_equal(got, got2)
        else:
            n0, n1 = parallel.token_shard(n, world, rank)
            part = oracle.spmm_exec(sw, np.ascontiguousarray(x[:, n0:n1]), prog, bias)
            # no collective in the product path; gather only to check the union
            parts = [None] * world
            dist.all_gather_object(parts, (n0, n1, part))
            got = np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])], axis=0)
        q.put((rank, bool(np.array_equal(got, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("rows", 2), ("rows", 3), ("tokens", 2)])
def test_sharded_equals_single(mode, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def test_split_range_covers():
    for total in (1, 7, 192, 1024):
        for parts in (1, 2, 3, 8):
            spans = [parallel.split_range(total, parts, i) for i in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_shard_rows_roundtrip():
    w, _, _, scales = workloads.baseline_inputs(37, 20, 1, 0.5, 3, with_x=False)
    sw = encode_sparse(w, scales)
    from paper_2306_16601_b200 import decode_sparse
    for world in (1, 2, 3, 4):
        blocks = []
        for r in range(world):
            sh = parallel.shard_rows(sw, world, r)
            if sh.m1 > sh.m0:
                blocks.append(decode_sparse(sh.weight))
        assert np.array_equal(np.concatenate(blocks, axis=0), w)
