"""Multi-GPU path host logic on CPU: column shards + all-gather.

World size 2 over gloo on 127.0.0.1.  Each rank computes its row shard
[pN/P, (p+1)N/P) with the product's CPU lane, the shards are all-gathered in the
[P][B][N/P] layout hg_linear_sharded's NCCL all-gather produces, permuted to
[B, N] exactly as the library's gather_permute kernel does, and compared with
the unsharded oracle (bit-exact on small integers, tolerance otherwise).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _permute(gbuf, P, B, n_local):
    """[P][B][n_local] -> [B][P*n_local]  (library kernel gather_permute_kernel, glue_sm100.cu)."""
    return gbuf.reshape(P, B, n_local).transpose(1, 0, 2).reshape(B, P * n_local)


def _worker(rank, world, port, B, N, K, integer, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from harness import gen
    from paper_2403_01164_b200 import hg
    x, W, b = gen.linear_inputs(5, 1, "fc1", B, N, K, integer=integer)
    r0, r1 = oracle.shard(N, world, rank, 128)
    with hg.Context(-1, cpu_threads=2) as ctx:
        y_local = np.zeros((B, r1 - r0), np.float32)
        ctx.hg_host_gemv(x, B, r1 - r0, K, np.ascontiguousarray(W[r0:r1]), np.ascontiguousarray(b[r0:r1]),
                         y_local)
    out = torch.zeros(world * B * (r1 - r0), dtype=torch.float32)
    dist.all_gather_into_tensor(out, torch.from_numpy(y_local.reshape(-1)))
    y = _permute(out.numpy(), world, B, r1 - r0)
    if rank == 0:
        ref = oracle.linear(x, W, b)
        if integer:
            q.put(bool(np.array_equal(y.astype(np.float64), ref)))
        else:
            q.put(oracle.within_tol(y, ref)[0])
    dist.destroy_process_group()


@pytest.mark.parametrize("B,integer", [(1, 0), (3, 0), (2, 16)])
def test_two_rank_sharded_linear(B, integer):
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    N, K = 1024, 256
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, B, N, K, integer, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
