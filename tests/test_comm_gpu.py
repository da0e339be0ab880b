"""GPU tests of the NCCL layer (include/libtsm.h tsm_comm_*).

gpurun provides one GPU, so the communicator has one rank; the calls still go
through NCCL (unique id created by libtsm, exchanged via torch.distributed,
ncclAllReduce / ncclAllGather + rank-order sum kernel / ncclBroadcast).  The
multi-rank host logic is covered by tests/test_shard_gloo.py.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
def test_allreduce_and_bcast_one_rank(pg, deterministic, cplx):
    from paper_1905_03136_b200 import binding as tsm
    comm = tsm.Comm(0, 1, 0, deterministic=deterministic)
    try:
        K, M, N = 100003, 24, 16
        A = ti.matrix(K, M, "A", complex_=cplx, mode="int")
        B = ti.matrix(K, N, "B", complex_=cplx, mode="int")
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        C = tsm.tsmttsm_allreduce(comm, dA, dB)
        Bo = tsm.tsmm_bcast(comm, dA, C, root=0)
        torch.cuda.synchronize()
        ref, _ = oracle.tsmttsm(A, B)
        assert np.array_equal(C.cpu().numpy(), ref)
        refb, _ = oracle.tsmm(A, ref)
        assert np.array_equal(Bo.cpu().numpy(), refb)
        # an empty local shard contributes zeros
        Z = tsm.tsmttsm_allreduce(comm, dA[:0], dB[:0])
        torch.cuda.synchronize()
        assert np.all(Z.cpu().numpy() == 0)
    finally:
        comm.close()


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
def test_cgs_step_through_comm(pg, deterministic, cplx):
    """tsm_cgs_step with a communicator: C summed over ranks (NCCL), then the
    local update B -= A C; exact with an orthonormal basis and integer B."""
    from paper_1905_03136_b200 import binding as tsm
    comm = tsm.Comm(0, 1, 0, deterministic=deterministic)
    try:
        j = 6
        K, M, N = 4 ** j, 16, 7
        A = ti.walsh(K, M, scale=2.0 ** -j)
        if cplx:
            A = 1j * A
        B0 = ti.matrix(K, N, "B", complex_=cplx, mode="int")
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B0).cuda()
        C = tsm.cgs_step(dA, dB, comm=comm)
        torch.cuda.synchronize()
        Cref, _ = oracle.tsmttsm(A, B0, conj=cplx)
        assert np.array_equal(C.cpu().numpy(), Cref)
        assert np.array_equal(dB.cpu().numpy(), oracle.tsmm_update(A, Cref, B0, -1, 1)[0])
        # an empty local shard: C = sum of nothing = 0, B untouched
        e = torch.zeros((0, N), dtype=dB.dtype, device="cuda")
        C0 = tsm.cgs_step(dA[:0], e, comm=comm)
        torch.cuda.synchronize()
        assert np.all(C0.cpu().numpy() == 0)
    finally:
        comm.close()
