"""NEXT rows N1 / N2 on the GPU, against the oracle:

  N2  conjugate variants: TSMTTSM C = A^H B and TSMM B = A conj(C) (plan flag
      TSM_FLAG_CONJ) on every Z kernel family (DFMA, DMMA, DMMA+TMA, edge
      warps, complex-as-real, C-stationary);
  N1  TSMM update B <- alpha A C + beta B (bulk / TMA reduce-add for beta = 1,
      a scaling pass first for other beta) on every TSMM family, and the
      classical Gram-Schmidt step C = A^T B, B -= A C.
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gen_instances as gi  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


def families(tsm, op, M, N, z, conj=False):
    """One plan per kernel family the generator offers for this shape."""
    seen = {}
    for c in gi.candidates(op, M, N, z):
        key = (c.get("impl", 0), c.get("EDGE", 0) > 0, c.get("PAIR", 0), c.get("ZR", 0))
        if key in seen:
            continue
        try:
            seen[key] = (c, tsm.Plan(op, "z" if z else "d", M, N, 0, config=gi.to_tsm_config(op, c, 3, 1),
                                     conj=conj))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
    return seen


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("M,N", [(3, 5), (8, 8), (17, 17), (24, 40), (33, 20), (64, 64)])
def test_conj_tsmttsm_every_family(tsm, M, N):
    fams = families(tsm, "tsmttsm", M, N, True, conj=True)
    assert fams
    for key, (c, plan) in sorted(fams.items()):
        assert tsm.tsm_plan_get_flags(plan.handle) == tsm.TSM_FLAG_CONJ
        for K in (1, 7, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 21)
            B = ti.matrix(K, N, "B", complex_=True, seed=K + 22)
            got = tsm.tsmttsm(cu(A), cu(B), plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B, conj=True)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", complex_=True, mode="int")
        Bi = ti.matrix(30001, N, "B", complex_=True, mode="int")
        got = tsm.tsmttsm(cu(Ai), cu(Bi), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi, conj=True)[0]), (key, c)


def test_conj_flag_rules(tsm):
    with pytest.raises(tsm.TsmError) as e:
        tsm.Plan("tsmttsm", "d", 8, 8, 0, conj=True)
    assert e.value.status == 1
    h = tsm.ctypes.c_void_p()
    assert tsm.lib.tsm_plan_create_ex(tsm.ctypes.byref(h), 0, 1, 8, 8, 0, None, 64) == 1  # unknown flag
    # conj plan differs from the plain plan exactly by the sign of Im(A)
    A = ti.matrix(1000, 9, "A", complex_=True, mode="int")
    B = ti.matrix(1000, 4, "B", complex_=True, mode="int")
    c1 = tsm.tsmttsm(cu(A), cu(B), conj=True).cpu().numpy()
    c2 = tsm.tsmttsm(cu(np.conj(A)), cu(B)).cpu().numpy()
    assert np.array_equal(c1, c2)


UPD = [(1.0, 0.0), (-1.0, 1.0), (2.5, 0.5), (0.0, 1.0), (0.0, 0.0), (-0.75, -2.0)]
UPDZ = [(1.0, 0.0), (-1.0, 1.0), (0.5 - 2j, 0.25j), (1j, -1.0)]


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", [(1, 1), (5, 3), (16, 16), (32, 32), (41, 41), (64, 48), (24, 24)])
def test_tsmm_update_every_family(tsm, M, N, cplx):
    fams = families(tsm, "tsmm", M, N, cplx, conj=False)
    assert fams
    for conj in ([False, True] if cplx else [False]):
        for key, (c, plan0) in sorted(fams.items()):
            plan = tsm.Plan("tsmm", "z" if cplx else "d", M, N, 0, config=plan0.config(), conj=conj) \
                if conj else plan0
            for K, (alpha, beta) in zip((1, 6, 4099, 65537, 3, 20001), UPDZ * 2 if cplx else UPD):
                A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 31)
                Cm = ti.matrix(M, N, "C", complex_=cplx, seed=K + 32)
                B0 = ti.matrix(K, N, "B", complex_=cplx, seed=K + 33)
                Bd = cu(B0)
                tsm.tsmm_update(cu(A), cu(Cm), Bd, alpha, beta, plan=plan)
                torch.cuda.synchronize()
                ref, bound = oracle.tsmm_update(A, Cm, B0, alpha, beta, conj=conj)
                r, wi, _ = oracle.max_err_ratio(Bd.cpu().numpy(), ref, bound)
                assert r <= 1e-13, (M, N, key, conj, c, K, alpha, beta, r, wi)
            # integer mode, the Gram-Schmidt coefficients: bit-exact
            K = 50001
            A = ti.matrix(K, M, "A", complex_=cplx, mode="int")
            Cm = ti.matrix(M, N, "C", complex_=cplx, mode="int")
            B0 = ti.matrix(K, N, "B", complex_=cplx, mode="int")
            Bd = cu(B0)
            tsm.tsmm_update(cu(A), cu(Cm), Bd, -1.0, 1.0, plan=plan)
            torch.cuda.synchronize()
            assert np.array_equal(Bd.cpu().numpy(), oracle.tsmm_update(A, Cm, B0, -1, 1, conj=conj)[0]), key


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", [(16, 5), (32, 32), (8, 64), (64, 8)])
def test_cgs_step_exact_projection(tsm, M, N, cplx):
    # orthonormal scaled-Walsh basis (x i for Z) and integer B: the projection
    # is exact, so A^T B' = 0 (A^H for Z) and B' equals the oracle bit for bit.
    j = 7
    K = 4 ** j
    A = ti.walsh(K, M, scale=2.0 ** -j)
    if cplx:
        A = 1j * A
    B0 = ti.matrix(K, N, "B", complex_=cplx, mode="int")
    Ad, Bd = cu(A), cu(B0)
    C = tsm.cgs_step(Ad, Bd)
    torch.cuda.synchronize()
    Cref, _ = oracle.tsmttsm(A, B0, conj=cplx)
    assert np.array_equal(C.cpu().numpy(), Cref)
    Bref, _ = oracle.tsmm_update(A, Cref, B0, -1, 1)
    assert np.array_equal(Bd.cpu().numpy(), Bref)
    R = tsm.tsmttsm(Ad, Bd, conj=cplx).cpu().numpy()
    assert np.count_nonzero(R) == 0


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
def test_cgs_step_fp(tsm, cplx):
    K, M, N = 1 << 20, 24, 12
    A = ti.matrix(K, M, "A", complex_=cplx)
    B0 = ti.matrix(K, N, "B", complex_=cplx)
    Bd = cu(B0)
    C = tsm.cgs_step(cu(A), Bd).cpu().numpy()
    torch.cuda.synchronize()
    Cref, cb = oracle.tsmttsm(A, B0, conj=cplx)
    assert oracle.max_err_ratio(C, Cref, cb)[0] <= 1e-12
    # the update is checked against the oracle applied to the GPU's C
    Bref, bb = oracle.tsmm_update(A, C, B0, -1, 1)
    assert oracle.max_err_ratio(Bd.cpu().numpy(), Bref, bb)[0] <= 1e-13


STRIDED_SHAPES = [(16, 16), (32, 48), (64, 20), (8, 8), (1, 1), (3, 5), (7, 1), (1, 64), (33, 33), (57, 57),
                  (63, 64), (12, 9), (2, 2), (64, 1)]


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("offs", [(6, 80, 40), (3, 71, 17)], ids=["even", "odd"])
@pytest.mark.parametrize("M,N", STRIDED_SHAPES)
def test_strided_views(tsm, M, N, cplx, offs):
    """N4: column subsets of a wider block vector (row stride ld > width) through
    tsmttsm_ld / tsmm_ld for every width class: TMA kernels (16-byte row
    strides and bases), else the gather-capable kernels (any width; odd column
    offsets give 8-byte aligned D bases).  Ragged K (odd: the last-row path);
    the columns around the TSMM output view stay untouched."""
    for K in (1, 4099, 70001):
        W = 151  # odd row stride: no 16-byte rows for D
        big = ti.matrix(K, W, "A", complex_=cplx, seed=5 + K)
        G = cu(big)
        a0, b0, o0 = offs
        A, B = G[:, a0:a0 + M], G[:, b0:b0 + N]
        C = tsm.tsmttsm(A, B)
        torch.cuda.synchronize()
        ref, bound = oracle.tsmttsm(big[:, a0:a0 + M], big[:, b0:b0 + N])
        r = oracle.max_err_ratio(C.cpu().numpy(), ref, bound)[0]
        assert r <= 1e-12, (M, N, K, offs, r)
        Cm = ti.matrix(M, N, "C", complex_=cplx, seed=6)
        out = torch.zeros((K, W), dtype=G.dtype, device="cuda")
        Bv = out[:, o0:o0 + N]
        tsm.tsmm(A, cu(Cm), out=Bv)
        torch.cuda.synchronize()
        refm, bm = oracle.tsmm(big[:, a0:a0 + M], Cm)
        got = out.cpu().numpy()
        r2 = oracle.max_err_ratio(np.ascontiguousarray(got[:, o0:o0 + N]), refm, bm)[0]
        assert r2 <= 1e-13, (M, N, K, offs, r2)
        assert np.count_nonzero(got[:, :o0]) == 0 and np.count_nonzero(got[:, o0 + N:]) == 0  # untouched


def test_strided_rules(tsm):
    # a dense-tuned plan that is neither a TMA nor a gather-capable kernel refuses strided calls
    p = tsm.Plan("tsmttsm", "d", 8, 8, 0)
    A = torch.zeros((100, 40), dtype=torch.float64, device="cuda")
    if p.config()["kernel"] & 15 == 0:
        with pytest.raises(tsm.TsmError) as e:
            tsm.tsmttsm(A[:, :8], A[:, 10:18], plan=p)
        assert e.value.status == 2
    # every shape has a strided plan: odd D widths get the gather kernel
    ps = tsm.Plan("tsmttsm", "d", 33, 33, 0, strided=True)
    assert ps.config()["kernel"] & 15 == 1
    pg = tsm.Plan("tsmm", "d", 32, 32, 0, gather=True)
    assert pg.config()["kernel"] & 15 == 4
    # a TMA strided plan refuses row strides that are not 16-byte multiples
    pt = tsm.Plan("tsmm", "d", 32, 32, 0, strided=True)
    if pt.config()["kernel"] & 15 in (2, 3):
        X = torch.zeros((100, 41), dtype=torch.float64, device="cuda")
        with pytest.raises(tsm.TsmError) as e:
            tsm.tsmm(X[:, :32], torch.zeros(32, 32, dtype=torch.float64, device="cuda"),
                     out=torch.zeros((100, 41), dtype=torch.float64, device="cuda")[:, :32], plan=pt)
        assert e.value.status == 2
    # strided plans still serve dense calls
    for plan in (pt, pg):
        A = ti.matrix(5000, 32, "A")
        Cm = ti.matrix(32, 32, "C")
        got = tsm.tsmm(cu(A), cu(Cm), plan=plan).cpu().numpy()
        ref, b = oracle.tsmm(A, Cm)
        assert oracle.max_err_ratio(got, ref, b)[0] <= 1e-13
