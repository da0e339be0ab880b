"""Multi-process (world size 2, gloo, CPU) tests of the K-sharded path's host
logic: row partition, per-rank generator offsets, the
rank-order combine of partial C's and the broadcast of C before TSMM.

Each rank computes its local result with the CPU oracle (the test's checker);
the GPU path is the same partition with libtsm kernels + NCCL on each rank.
Integer-mode inputs make every sum exact, so the sharded results must equal
the unsharded oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_03136_b200.shard import rank_order_sum, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, K, M, N, cplx, q):
    import oracle
    import tsminputs as ti
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, count = shard_range(K, world, rank)
        # this rank's rows of the global A, B: generator indices offset by start
        A = ti.rows(np.arange(start, start + count), M, "A", complex_=cplx, mode="int")
        B = ti.rows(np.arange(start, start + count), N, "B", complex_=cplx, mode="int")
        C_loc, _ = oracle.tsmttsm(A, B) if count else (np.zeros((M, N), A.dtype), None)
        t = torch.from_numpy(np.ascontiguousarray(C_loc))
        if cplx:
            t = torch.view_as_real(t)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        parts = [torch.view_as_complex(g).numpy() if cplx else g.numpy() for g in gathered]
        C = rank_order_sum(parts)
        # TSMM after a broadcast of C from rank 0
        Cb = torch.from_numpy(np.ascontiguousarray(C))
        Cb = torch.view_as_real(Cb).contiguous() if cplx else Cb
        dist.broadcast(Cb, src=0)
        Cb = torch.view_as_complex(Cb).numpy() if cplx else Cb.numpy()
        Bo, _ = oracle.tsmm(A, Cb) if count else (np.zeros((0, N), A.dtype), None)
        q.put((rank, start, count, C, Bo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("K,M,N,cplx", [(100003, 7, 5, False), (4097, 16, 16, True), (1, 3, 2, False)])
def test_sharded_tsmttsm_tsmm_world2(K, M, N, cplx):
    import oracle
    import tsminputs as ti
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, M, N, cplx, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = ti.matrix(K, M, "A", complex_=cplx, mode="int")
    B = ti.matrix(K, N, "B", complex_=cplx, mode="int")
    C_ref, _ = oracle.tsmttsm(A, B)
    for (rank, start, count, C, Bo) in res:
        assert np.array_equal(C, C_ref)  # every rank ends with the full C
        B_ref, _ = oracle.tsmm(A[start:start + count], C_ref)
        assert np.array_equal(Bo, B_ref)
    # shards tile [0, K) exactly
    assert res[0][1] == 0 and res[0][1] + res[0][2] == res[1][1] and res[1][1] + res[1][2] == K


@pytest.mark.parametrize("K,world", [(0, 3), (1, 2), (10, 3), (1 << 28, 8), (7, 8)])
def test_shard_range_partition(K, world):
    spans = [shard_range(K, world, r) for r in range(world)]
    assert spans[0][0] == 0
    for (s0, c0), (s1, _) in zip(spans, spans[1:]):
        assert s0 + c0 == s1
    assert sum(c for _, c in spans) == K
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
