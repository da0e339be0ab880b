"""configs[4] at full size on one GPU: M = N = 32, K = 2^28 rows in total,
K-sharded (row-distributed block vectors).

The sharded result is the sum over ranks of each rank's local TSMTTSM over
its rows [r K/p, (r+1) K/p); on one GPU the ranks' shards are computed one
after the other with the same plans the ranks would use, and their C's are
summed in rank order (the TSM_COMM_DETERMINISTIC combination).  Checked
against the streaming oracle (rows regenerated from the
input generator segment by segment, PAPER.md:342-349 definition) on a 3 x 3
grid of C cells over all 2^28 rows; TSMM on every shard-boundary row plus
random rows of every shard, with C replicated as after the allreduce.
D: the whole K = 2^28 fits one GPU (A + B = 137 GB): the unsharded result and
p = 2, 8.  Z: A + B = 275 GB at 2^28, so the p = 2 shards (2^27 rows each)
are generated and computed one at a time.
"""
import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

pytestmark = pytest.mark.gpu

K4 = 1 << 28
W = 32
MS, NS = [0, 17, 31], [0, 9, 31]


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


def _oracle_cells(cplx):
    def rows(k0, k1):
        return (ti.columns(k1 - k0, W, MS, "A", complex_=cplx, row0=k0),
                ti.columns(k1 - k0, W, NS, "B", complex_=cplx, row0=k0))
    return oracle.tsmttsm_stream(K4, len(MS), len(NS), rows, cplx, seg_rows=1 << 24)


def _check_c(C, ref, bound, what):
    got = C[np.ix_(MS, NS)]
    r, wi, _ = oracle.max_err_ratio(got, ref, bound)
    assert r <= 1e-12, f"{what}: max err/bound {r:.3e} at {wi}"


def _check_inputs(A, B, row0, cplx):
    """Sampled rows of the device shard equal the host generator (global rows)."""
    rows = np.array([0, 1, A.shape[0] // 2, A.shape[0] - 1])
    a = ti.rows(rows + row0, W, "A", complex_=cplx)
    b = ti.rows(rows + row0, W, "B", complex_=cplx)
    idx = torch.from_numpy(rows).cuda()
    assert np.array_equal(A[idx].cpu().numpy(), a) and np.array_equal(B[idx].cpu().numpy(), b)


def _check_tsmm_shard(tsm, A_r, C, row0, O, rng, cplx, what):
    """B_r = A_r C on this rank's rows: shard-boundary rows + 256 random rows."""
    Kp = A_r.shape[0]
    plan = tsm.get_plan("tsmm", "z" if cplx else "d", W, W, 0)
    Ob = O[: Kp * W].view(Kp, W)
    tsm.tsmm(A_r, C, out=Ob, plan=plan)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, 1, Kp - 2, Kp - 1], rng.integers(0, Kp, 256)]))
    a = ti.rows(rows + row0, W, "A", complex_=cplx)
    Ch = C.cpu().numpy()
    ref, bound = oracle.tsmm(a, Ch)
    got = Ob[torch.from_numpy(rows).cuda()].cpu().numpy()
    r, wi, _ = oracle.max_err_ratio(got, ref, bound)
    assert r <= 1e-13, f"{what}: tsmm max err/bound {r:.3e} at shard row {rows[wi // W]}"


def test_configs4_d(tsm):
    """D, K = 2^28: unsharded and p = 2, 8 shards (rank-order sum of C)."""
    A = torch.empty(K4, W, dtype=torch.float64, device="cuda")
    B = torch.empty(K4, W, dtype=torch.float64, device="cuda")
    tsm.fill(A, "A", ti.SEED_FP, "fp")
    tsm.fill(B, "B", ti.SEED_FP, "fp")
    _check_inputs(A, B, 0, False)
    ref, bound = _oracle_cells(False)
    C_full = tsm.tsmttsm(A, B).cpu().numpy()
    _check_c(C_full, ref, bound, "unsharded K=2^28")
    C32 = None
    for p in (2, 8):
        Kp = K4 // p
        Csum = None
        for r in range(p):
            Cr = tsm.tsmttsm(A[r * Kp:(r + 1) * Kp], B[r * Kp:(r + 1) * Kp]).cpu().numpy()
            Csum = Cr.copy() if Csum is None else Csum + Cr
        _check_c(Csum, ref, bound, f"p={p} shards")
        C32 = Csum
    # TSMM on every p = 8 shard with the replicated C (B's buffer is reused as scratch)
    del B
    torch.cuda.empty_cache()
    O = torch.empty(K4 // 8 * W, dtype=torch.float64, device="cuda")
    Cd = torch.from_numpy(C32 / float(K4)).cuda()  # scaled to O(1) entries, as after a normalisation
    rng = np.random.default_rng(4)
    for r in range(8):
        Kp = K4 // 8
        _check_tsmm_shard(tsm, A[r * Kp:(r + 1) * Kp], Cd, r * Kp, O, rng, False, f"D shard {r}/8")
    del A, O
    torch.cuda.empty_cache()


def test_configs4_z(tsm):
    """Z, K = 2^28 as p = 2 shards of 2^27 rows, computed one after the other."""
    Kp = K4 // 2
    A = torch.empty(Kp, W, dtype=torch.complex128, device="cuda")
    B = torch.empty(Kp, W, dtype=torch.complex128, device="cuda")
    Csum = None
    for r in range(2):
        start = r * Kp * W * 2  # real-value index of the shard's first element
        tsm.fill(A, "A", ti.SEED_FP, "fp", start=start)
        tsm.fill(B, "B", ti.SEED_FP, "fp", start=start)
        _check_inputs(A, B, r * Kp, True)
        Cr = tsm.tsmttsm(A, B).cpu().numpy()
        Csum = Cr.copy() if Csum is None else Csum + Cr
    ref, bound = _oracle_cells(True)
    _check_c(Csum, ref, bound, "Z p=2 shards")
    # TSMM on the last shard (still resident), C replicated
    del B
    torch.cuda.empty_cache()
    O = torch.empty(Kp * W, dtype=torch.complex128, device="cuda")
    Cd = torch.from_numpy(Csum / float(K4)).cuda()
    _check_tsmm_shard(tsm, A, Cd, Kp, O, np.random.default_rng(5), True, "Z shard 1/2")
    del A, O
    torch.cuda.empty_cache()
