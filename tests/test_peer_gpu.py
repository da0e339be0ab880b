"""NEXT N3: TSMTTSM with the grid reduction fused with the cross-GPU sum over
peer memory (include/libtsm.h tsm_peer_*).  One GPU here: world 1 in process,
and world 2 as two processes sharing cuda:0 (CUDA IPC on one device exercises
the same slot-buffer protocol as NVLink peers).  The fused result must equal
the rank-order sum of the per-rank local results bit for bit (the
TSM_COMM_DETERMINISTIC contract) and the oracle on the whole K within the
north-star tolerance."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


@pytest.mark.parametrize("dt,M,N", [("d", 8, 8), ("d", 64, 64), ("d", 33, 17), ("z", 32, 32), ("z", 17, 17),
                                    ("z", 5, 3), ("d", 1, 64)])
def test_world1_equals_local(tsm, dt, M, N):
    """world 1: the fused path writes the single slot and sums it -- C equals
    the plain TSMTTSM bit for bit, over several calls (alternating parities),
    including an empty shard (K = 0 -> zeros)."""
    peer = tsm.PeerComm(0, 1, 0)
    cplx = dt == "z"
    try:
        for K in (4099, 65537, 1000, 0, 3):
            A = torch.from_numpy(ti.matrix(K, M, "A", complex_=cplx, seed=K + 61)).cuda()
            B = torch.from_numpy(ti.matrix(K, N, "B", complex_=cplx, seed=K + 62)).cuda()
            got = tsm.tsmttsm_peer(peer, A, B)
            torch.cuda.synchronize()
            if K == 0:
                assert torch.count_nonzero(got).item() == 0
                continue
            ref = tsm.tsmttsm(A, B)
            torch.cuda.synchronize()
            assert torch.equal(got, ref), (dt, M, N, K)
        assert peer.error() == 0
    finally:
        peer.close()


WORKER = r"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["TSM_ROOT"])
import tsminputs as ti
from paper_1905_03136_b200 import binding as tsm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
cfg = json.loads(os.environ["TSM_CASE"])
peer = tsm.PeerComm(rank, world, 0)
out = {}
for case in cfg:
    dt, M, N, K, splits, mode = case
    cplx = dt == "z"
    A = ti.matrix(K, M, "A", complex_=cplx, mode=mode, seed=7 if mode == "int" else 42)
    B = ti.matrix(K, N, "B", complex_=cplx, mode=mode, seed=7 if mode == "int" else 42)
    lo, hi = splits[rank], splits[rank + 1]
    Ag = torch.from_numpy(np.ascontiguousarray(A[lo:hi])).cuda()
    Bg = torch.from_numpy(np.ascontiguousarray(B[lo:hi])).cuda()
    C = tsm.tsmttsm_peer(peer, Ag, Bg)
    torch.cuda.synchronize()
    loc = tsm.tsmttsm(Ag, Bg) if hi > lo else torch.zeros_like(C)
    torch.cuda.synchronize()
    key = "%s_%d_%d_%d_%s" % (dt, M, N, K, mode)
    np.save(os.path.join(os.environ["TSM_OUT"], "%s_r%d_C.npy" % (key, rank)), C.cpu().numpy())
    np.save(os.path.join(os.environ["TSM_OUT"], "%s_r%d_loc.npy" % (key, rank)), loc.cpu().numpy())
out["err"] = peer.error()
peer.close()
json.dump(out, open(os.path.join(os.environ["TSM_OUT"], "r%d.json" % rank), "w"))
dist.barrier()
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_processes_one_gpu(tsm, tmp_path):
    """world 2 (two processes on cuda:0, IPC-mapped slot buffers): uneven
    shards, an empty shard, D and Z (incl. a 3M / complex-as-real plan shape),
    FP and integer inputs.  Both ranks hold the same C; it equals the
    rank-order sum of the local results bitwise, the oracle within 1e-12
    |A|^T|B|, and (integer inputs) the oracle exactly."""
    cases = [("d", 32, 32, 70001, [0, 30000, 70001], "fp"),
             ("z", 24, 24, 50003, [0, 50003, 50003], "fp"),      # rank 1: empty shard
             ("d", 50, 50, 40000, [0, 12345, 40000], "int"),
             ("z", 17, 17, 30001, [0, 1, 30001], "int"),
             ("d", 8, 8, 1000000, [0, 500000, 1000000], "fp")]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE="2",
               TSM_ROOT=ROOT, TSM_OUT=str(tmp_path), TSM_CASE=json.dumps(cases))
    procs = [subprocess.Popen([sys.executable, "-c", WORKER], env=dict(env, RANK=str(r)), cwd=ROOT,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        outs.append(o)
    assert all(p.returncode == 0 for p in procs), "\n".join(o[-3000:] for o in outs)
    for r in range(2):
        assert json.load(open(tmp_path / f"r{r}.json"))["err"] == 0
    for (dt, M, N, K, splits, mode) in cases:
        key = f"{dt}_{M}_{N}_{K}_{mode}"
        C0 = np.load(tmp_path / f"{key}_r0_C.npy")
        C1 = np.load(tmp_path / f"{key}_r1_C.npy")
        assert np.array_equal(C0, C1), key
        l0 = np.load(tmp_path / f"{key}_r0_loc.npy")
        l1 = np.load(tmp_path / f"{key}_r1_loc.npy")
        assert np.array_equal(C0, l0 + l1), key  # rank-order sum, bitwise
        cplx = dt == "z"
        A = ti.matrix(K, M, "A", complex_=cplx, mode=mode, seed=7 if mode == "int" else 42)
        B = ti.matrix(K, N, "B", complex_=cplx, mode=mode, seed=7 if mode == "int" else 42)
        ref, bound = oracle.tsmttsm(A, B)
        if mode == "int":
            assert np.array_equal(C0, ref), key
        else:
            r, wi, _ = oracle.max_err_ratio(C0, ref, bound)
            assert r <= 1e-12, (key, r, wi)


FAILFAST_WORKER = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["TSM_ROOT"])
import numpy as np, torch, torch.distributed as dist
from paper_1905_03136_b200 import binding as tsm
rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=2)
peer = tsm.PeerComm(rank, 2, 0)
peer.set_timeout(0.05)
K, M = 20000, 16
A = torch.empty(K, M, dtype=torch.float64, device="cuda")
tsm.fill(A, "A", 42 + rank)
res = {}
C = tsm.tsmttsm_peer(peer, A, A)              # call 0: both ranks -> fine
torch.cuda.synchronize()
res["ok0"] = bool(torch.isfinite(C).all().item()) and peer.error() == 0
dist.barrier()
if rank == 0:                                  # call 1: rank 1 never arrives
    C = tsm.tsmttsm_peer(peer, A, A)
    torch.cuda.synchronize()
    res["timeout_nan"] = bool(torch.isnan(C).all().item())
    res["err1"] = peer.error()
    t0 = time.perf_counter()
    C = tsm.tsmttsm_peer(peer, A, A)           # call 2: fails fast (no 50 ms wait)
    torch.cuda.synchronize()
    res["failfast_s"] = time.perf_counter() - t0
    res["failfast_nan"] = bool(torch.isnan(C).all().item())
dist.barrier()
peer.reset()                                   # collective recovery
C = tsm.tsmttsm_peer(peer, A, A)
torch.cuda.synchronize()
loc = tsm.tsmttsm(A, A)
torch.cuda.synchronize()
res["after_reset_err"] = peer.error()
res["after_reset_finite"] = bool(torch.isfinite(C).all().item())
np.save(os.path.join(os.environ["TSM_OUT"], f"ff_r{rank}_C.npy"), C.cpu().numpy())
np.save(os.path.join(os.environ["TSM_OUT"], f"ff_r{rank}_loc.npy"), loc.cpu().numpy())
json.dump(res, open(os.path.join(os.environ["TSM_OUT"], f"ff_r{rank}.json"), "w"))
peer.close()
dist.destroy_process_group()
'''


def test_peer_timeout_failfast_reset(tsm, tmp_path):
    """a missing rank -> C = NaN and the error flag; every later
    call on that rank fails fast; tsm_peer_reset on every rank recovers."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE="2",
               TSM_ROOT=ROOT, TSM_OUT=str(tmp_path))
    procs = [subprocess.Popen([sys.executable, "-c", FAILFAST_WORKER], env=dict(env, RANK=str(r)), cwd=ROOT,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        outs.append(o)
    assert all(p.returncode == 0 for p in procs), "\n".join(o[-3000:] for o in outs)
    r0 = json.load(open(tmp_path / "ff_r0.json"))
    r1 = json.load(open(tmp_path / "ff_r1.json"))
    assert r0["ok0"] and r1["ok0"]
    assert r0["timeout_nan"] and r0["err1"] == 1
    assert r0["failfast_nan"] and r0["failfast_s"] < 0.04, r0
    for r in (r0, r1):
        assert r["after_reset_err"] == 0 and r["after_reset_finite"]
    C0, C1 = np.load(tmp_path / "ff_r0_C.npy"), np.load(tmp_path / "ff_r1_C.npy")
    l0, l1 = np.load(tmp_path / "ff_r0_loc.npy"), np.load(tmp_path / "ff_r1_loc.npy")
    assert np.array_equal(C0, C1) and np.array_equal(C0, l0 + l1)
