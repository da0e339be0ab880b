"""GPU parity: libtsm CUDA path (through the C ABI) vs the CPU oracle.

Tolerances are the north star's (BASELINE.json):
    TSMTTSM |C_gpu - C_ref| <= 1e-12 (|A|^T|B|)   elementwise
    TSMM    |B_gpu - B_ref| <= 1e-13 (|A||C|)      elementwise
with |.| the complex modulus for Z; integer-mode inputs must match bitwise.
Inputs come from tsminputs on the host (oracle side) and are copied to the
GPU; the full-size tests fill the device with libtsm's own generator and
check it against tsminputs on every sampled element first.
"""
import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

pytestmark = pytest.mark.gpu

TOL_TSMTTSM = 1e-12
TOL_TSMM = 1e-13


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run_tsmttsm(tsm, A, B):
    C = tsm.tsmttsm(dev(A), dev(B))
    return host(C)


def run_tsmm(tsm, A, C):
    B = tsm.tsmm(dev(A), dev(C))
    return host(B)


def check_tsmttsm(tsm, K, M, N, cplx, mode="fp", seed=None):
    A = ti.matrix(K, M, "A", complex_=cplx, mode=mode, seed=seed)
    B = ti.matrix(K, N, "B", complex_=cplx, mode=mode, seed=seed)
    got = run_tsmttsm(tsm, A, B)
    ref, bound = oracle.tsmttsm(A, B)
    if mode == "int":
        assert np.array_equal(got, ref), f"int-mode mismatch K={K} M={M} N={N} z={cplx}"
    r, wi, ma = oracle.max_err_ratio(got, ref, bound)
    assert r <= TOL_TSMTTSM, f"K={K} M={M} N={N} z={cplx}: max err/bound {r:.3e} at {wi} (abs {ma:.3e})"
    return r


def check_tsmm(tsm, K, M, N, cplx, mode="fp", seed=None):
    A = ti.matrix(K, M, "A", complex_=cplx, mode=mode, seed=seed)
    C = ti.matrix(M, N, "C", complex_=cplx, mode=mode, seed=seed)
    got = run_tsmm(tsm, A, C)
    ref, bound = oracle.tsmm(A, C)
    if mode == "int":
        assert np.array_equal(got, ref), f"int-mode mismatch K={K} M={M} N={N} z={cplx}"
    r, wi, ma = oracle.max_err_ratio(got, ref, bound)
    assert r <= TOL_TSMM, f"K={K} M={M} N={N} z={cplx}: max err/bound {r:.3e} at {wi} (abs {ma:.3e})"
    return r


# K values hit every tail case: single row, even/odd, < one chunk, several
# chunks with a ragged tail, more chunks than the persistent grid.
K_SMALL = [1, 2, 3, 33, 1000, 4099]
SQUARE = list(range(1, 65))
NONSQUARE = [(1, 64), (64, 1), (16, 48), (48, 16), (3, 5), (5, 3), (7, 2), (13, 29), (33, 17),
             (5, 64), (64, 5), (1, 7), (9, 1), (63, 64), (64, 63), (1, 2), (2, 1)]


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("w", SQUARE)
def test_tsmttsm_square(tsm, w, cplx):
    for K in (1, 3, 4099, 50001):
        check_tsmttsm(tsm, K, w, w, cplx)


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("w", SQUARE)
def test_tsmm_square(tsm, w, cplx):
    for K in (1, 3, 4099, 50001):
        check_tsmm(tsm, K, w, w, cplx)


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", NONSQUARE)
def test_nonsquare_all_tails(tsm, M, N, cplx):
    for K in K_SMALL:
        check_tsmttsm(tsm, K, M, N, cplx)
        check_tsmm(tsm, K, M, N, cplx)


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", [(1, 1), (8, 8), (32, 32), (64, 64), (16, 48), (64, 1), (1, 64), (7, 2)])
def test_int_mode_bitwise_many_chunks(tsm, M, N, cplx):
    # integer inputs: every summation order is exact -> bitwise equality
    K = (1 << 19) + 3 if M * N <= 1024 else (1 << 17) + 1
    check_tsmttsm(tsm, K, M, N, cplx, mode="int")
    check_tsmm(tsm, 4099, M, N, cplx, mode="int")


def test_config1_tsmttsm_d_8x8_k1e6(tsm):
    # BASELINE.json configs[0]: TSMTTSM D M=N=8, K=10^6 -- full oracle comparison
    check_tsmttsm(tsm, 10 ** 6, 8, 8, False)


def test_determinism(tsm):
    A = dev(ti.matrix(300001, 13, "A"))
    B = dev(ti.matrix(300001, 29, "B"))
    C1 = host(tsm.tsmttsm(A, B))
    C2 = host(tsm.tsmttsm(A, B))
    assert np.array_equal(C1, C2)
    Cm = dev(ti.matrix(13, 29, "C"))
    assert np.array_equal(host(tsm.tsmm(A, Cm)), host(tsm.tsmm(A, Cm)))


def test_walsh_orthogonality_gpu(tsm):
    # closed form at any size: Walsh columns -> A^T A = K I exactly
    K, M = 1 << 20, 32
    k = torch.arange(K, device="cuda", dtype=torch.int64)[:, None]
    m = torch.arange(M, device="cuda", dtype=torch.int64)[None, :]
    x = k & m
    par = torch.zeros_like(x)
    for b in range(6):
        par ^= (x >> b) & 1
    A = (1.0 - 2.0 * par.double()).contiguous()
    C = host(tsm.tsmttsm(A, A))
    assert np.array_equal(C, K * np.eye(M))
    Az = (A * (1 + 1j)).contiguous()
    Cz = host(tsm.tsmttsm(Az, Az))
    assert np.array_equal(Cz, 2j * K * np.eye(M))  # plain transpose (no conj)


def test_nan_propagation(tsm):
    K, M, N = 5000, 6, 4
    A = ti.matrix(K, M, "A")
    B = ti.matrix(K, N, "B")
    A[1234, 2] = np.nan
    C = run_tsmttsm(tsm, A, B)
    assert np.all(np.isnan(C[2])) and not np.any(np.isnan(np.delete(C, 2, axis=0)))
    Cm = ti.matrix(M, N, "C")
    Bo = run_tsmm(tsm, A, Cm)
    assert np.all(np.isnan(Bo[1234])) and not np.any(np.isnan(np.delete(Bo, 1234, axis=0)))


def test_error_paths(tsm):
    from paper_1905_03136_b200.binding import TsmError
    A = torch.zeros(100, 4, dtype=torch.float64, device="cuda")
    B = torch.zeros(100, 4, dtype=torch.float64, device="cuda")
    plan = tsm.get_plan("tsmttsm", "d", 4, 4, 0)
    ws = torch.zeros(plan.workspace_bytes(100), dtype=torch.uint8, device="cuda")
    C = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    with pytest.raises(TsmError, match="MISALIGNED"):  # 8-byte offset view
        tsm.tsmttsm_d(plan.handle, 99, A.data_ptr() + 8, B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel(), s)
    with pytest.raises(TsmError, match="WORKSPACE"):
        tsm.tsmttsm_d(plan.handle, 100, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), 16, s)
    with pytest.raises(TsmError, match="INVALID_VALUE"):  # K = 0
        tsm.tsmttsm_d(plan.handle, 0, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel(), s)
    with pytest.raises(TsmError, match="INVALID_VALUE"):  # output overlaps input
        tsm.tsmttsm_d(plan.handle, 100, A.data_ptr(), B.data_ptr(), A.data_ptr(), ws.data_ptr(), ws.numel(), s)
    with pytest.raises(TsmError, match="INVALID_VALUE"):  # op mismatch
        tsm.tsmm_d(plan.handle, 100, A.data_ptr(), C.data_ptr(), B.data_ptr(), s)
    # a good call after the failures still works (workspace counters untouched)
    tsm.tsmttsm_d(plan.handle, 100, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel(), s)
    torch.cuda.synchronize()


def test_device_generator_matches_host(tsm):
    for cplx in (False, True):
        for mode in ("fp", "int"):
            t = torch.empty(1000, 7, dtype=torch.complex128 if cplx else torch.float64, device="cuda")
            tsm.fill(t, "B", 42 if mode == "fp" else 7, mode)
            ref = ti.matrix(1000, 7, "B", complex_=cplx, mode=mode)
            assert np.array_equal(host(t), ref)


# Full BASELINE sizes (K = 2^24 / 2^25) for every tuned plan: tests/test_fullsize_gpu.py


def test_workspace_reuse_across_shapes(tsm):
    # the cached workspace's counters are left at zero after each call, so the
    # same buffer serves different plans and K back to back
    for (M, N, K) in [(4, 4, 100), (64, 64, 3), (8, 2, 200001), (4, 4, 77777)]:
        check_tsmttsm(tsm, K, M, N, False)


def test_grid_reduce_solo_and_multi_finisher(tsm):
    # T4 has two finishing schemes: one finisher (nfin == 1, ticket G-1: no wait,
    # plain counter reset) and several (spin on the ticket counter, reset by
    # the last of them).  Alternate them on one cached workspace, repeat each
    # call, and check every result against the oracle and bitwise repeatability.
    seen = set()
    cases = [(4, 4, 1 << 20), (8, 8, 1000003), (4, 4, 9999), (8, 8, 4099), (1, 1, 300001),
             (32, 32, 200001), (4, 4, 1 << 20), (64, 64, 70001)]
    for (M, N, K) in cases:
        nfin = tsm.Plan("tsmttsm", "d", M, N).describe(K)["nfin"]
        seen.add("solo" if nfin == 1 else "multi")
        A = ti.matrix(K, M, "A")
        B = ti.matrix(K, N, "B")
        got = [run_tsmttsm(tsm, A, B) for _ in range(3)]
        ref, bound = oracle.tsmttsm(A, B)
        for g in got:
            r, wi, _ = oracle.max_err_ratio(g, ref, bound)
            assert r <= TOL_TSMTTSM, f"M={M} N={N} K={K} nfin={nfin}: err/bound {r:.3e} at {wi}"
            assert np.array_equal(g, got[0]), f"M={M} N={N} K={K} nfin={nfin}: not repeatable"
    assert seen == {"solo", "multi"}, seen


# ---------------------------------------------------------------------------
# Shapes outside the AOT set: NVRTC run-time instantiation of the same
# templates; explicit configurations (the autotuner's search space).
# ---------------------------------------------------------------------------
JIT_SHAPES = [(12, 20), (37, 5), (2, 63), (64, 9), (11, 12)]


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", JIT_SHAPES)
def test_jit_shapes(tsm, M, N, cplx):
    for K in (1, 4099, 70001):
        check_tsmttsm(tsm, K, M, N, cplx)
        check_tsmm(tsm, K, M, N, cplx)
    p = tsm.get_plan("tsmttsm", "z" if cplx else "d", M, N, 0)
    assert p.describe(1000)["jit"] is True


@pytest.mark.parametrize("cfg", [
    dict(threads=128, rows_per_chunk=64, p0=4, p1=8, p2=0, stages=3, ctas_per_sm=2),
    dict(threads=256, rows_per_chunk=32, p0=8, p1=8, p2=0, stages=4, ctas_per_sm=1),
    dict(threads=64, rows_per_chunk=130, p0=2, p1=1, p2=0, stages=2, ctas_per_sm=8),
])
def test_explicit_config_tsmttsm(tsm, cfg):
    M, N, K = 32, 16, 100003
    p = tsm.Plan("tsmttsm", "d", M, N, 0, config=cfg)
    got = p.config()
    for k in ("threads", "rows_per_chunk", "p0", "p1"):
        assert got[k] == cfg[k]
    A = ti.matrix(K, M, "A")
    B = ti.matrix(K, N, "B")
    C = host(tsm.tsmttsm(dev(A), dev(B), plan=p))
    ref, bound = oracle.tsmttsm(A, B)
    assert oracle.max_err_ratio(C, ref, bound)[0] <= TOL_TSMTTSM


@pytest.mark.parametrize("cfg", [
    dict(threads=128, rows_per_chunk=64, p0=16, p1=1, p2=4, stages=3, ctas_per_sm=2),
    dict(threads=256, rows_per_chunk=256, p0=4, p1=8, p2=2, stages=2, ctas_per_sm=1),
])
def test_explicit_config_tsmm(tsm, cfg):
    M, N, K = 24, 16, 100003
    p = tsm.Plan("tsmm", "z", M, N, 0, config=cfg)
    A = ti.matrix(K, M, "A", complex_=True)
    Cm = ti.matrix(M, N, "C", complex_=True)
    Bo = host(tsm.tsmm(dev(A), dev(Cm), plan=p))
    ref, bound = oracle.tsmm(A, Cm)
    assert oracle.max_err_ratio(Bo, ref, bound)[0] <= TOL_TSMM


def test_bad_config_rejected(tsm):
    from paper_1905_03136_b200.binding import TsmError
    with pytest.raises(TsmError, match="INVALID_VALUE"):
        tsm.Plan("tsmttsm", "d", 8, 8, 0, config=dict(threads=100, rows_per_chunk=64, p0=2, p1=2,
                                                     p2=0, stages=2, ctas_per_sm=1))
    with pytest.raises(TsmError, match="INVALID_VALUE"):
        tsm.Plan("tsmm", "d", 8, 8, 0, config=dict(threads=128, rows_per_chunk=63, p0=8, p1=4,
                                                  p2=1, stages=2, ctas_per_sm=1))


def test_aot_path_parity():
    """Plans load NVRTC kernels (precompiled into kcache); TSM_PREFER_AOT=1
    selects the nvcc-compiled AOT instantiations instead -- same results."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle, tsminputs as ti
from paper_1905_03136_b200 import binding as tsm
for op, dt, M, N in [("tsmttsm", "d", 64, 64), ("tsmttsm", "z", 24, 24), ("tsmm", "d", 41, 41), ("tsmm", "z", 33, 17)]:
    p = tsm.Plan(op, dt, M, N, 0)
    assert p.describe(1000)["jit"] is False, p.describe(1000)
    z = dt == "z"
    A = ti.matrix(20001, M, "A", complex_=z, mode="int")
    if op == "tsmttsm":
        B = ti.matrix(20001, N, "B", complex_=z, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=p).cpu().numpy()
        ref = oracle.tsmttsm(A, B)[0]
    else:
        C = ti.matrix(M, N, "C", complex_=z, mode="int")
        got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda(), plan=p).cpu().numpy()
        ref = oracle.tsmm(A, C)[0]
    assert np.array_equal(got, ref), (op, dt, M, N)
print("ok")
'''
    import os
    env = dict(os.environ, TSM_PREFER_AOT="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
