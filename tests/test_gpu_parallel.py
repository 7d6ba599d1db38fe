"""RowShardedSpmm through the product kernel on the GPU (world size 1: the
bookkeeping around the kernel -- shard plan, in-place write of the rank's
rows into the final [N, M] buffer with ldo = M -- runs as on a multi-GPU
group; the exchange step is a no-op at one rank)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import parallel, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("m,k,n", [(1024, 1024, 4096), (4096, 1024, 2000), (300, 512, 777)])
def test_row_sharded_product_kernel(nccl_world1, m, k, n):
    w, x, bias, scales = workloads.baseline_inputs(m, k, n, 0.9, 61)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program("requant_u8", scales)
    rs = parallel.RowShardedSpmm(sw, n, prog, bias=bias, device="cuda")
    from paper_2306_16601_b200 import kernels as K
    out = rs.run(K.relayout_tokens(np.ascontiguousarray(x.T)))
    torch.cuda.synchronize()
    assert out.shape == (n, m)
    assert np.array_equal(out.cpu().numpy(), oracle.spmm_exec(sw, x, prog, bias))
