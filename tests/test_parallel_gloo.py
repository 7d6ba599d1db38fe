"""Multi-process (world_size 2, gloo on CPU) tests of the sharding bookkeeping.

The per-rank compute is the C oracle here (no GPU in this container); on a
GPU box the same bookkeeping wraps the product kernel (RowShardedSpmm)."""

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
            sh = parallel.shard_rows(sw, world, rank)
            sp = parallel.shard_program(prog, sh.m0, sh.m1)
            local = np.zeros((n, sh.rows_pad), np.uint8)
            if sh.m1 > sh.m0:
                local[:, : sh.m1 - sh.m0] = oracle.spmm_exec(sh.weight, x, sp, bias[sh.m0: sh.m1])
            gathered = torch.empty((world, n, sh.rows_pad), dtype=torch.uint8)
            parallel.gather_rows(gathered, torch.from_numpy(local))
            bounds = [(parallel.shard_rows(sw, world, r).m0, parallel.shard_rows(sw, world, r).m1)
                      for r in range(world)]
            got = parallel.assemble_rows(gathered, n, m, world, sh.rows_pad, bounds).numpy()
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


@pytest.mark.parametrize("mode", ["rows", "tokens"])
def test_sharded_equals_single(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


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
