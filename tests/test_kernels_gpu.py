"""Every kernel family, forced through explicit configurations (the autotuner's
search space), against the oracle on ragged K -- so a variant that the tuned
table does not currently pick is still proven correct before it can be picked.

  TSMTTSM: 0 register-tile DFMA, 1 DMMA bulk copies, 2 DMMA + TMA tensor maps
  TSMM:    0 DFMA, 1 DMMA bulk copies, 2 DMMA + TMA, 3 C-stationary DMMA + TMA
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

SHAPES = [(64, 64), (48, 16), (16, 40), (32, 32), (24, 24), (8, 8), (33, 17), (3, 5)]
K_LIST = [1, 7, 4099, 65537]


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


def per_impl(tsm, op, M, N, z):
    """First candidate of each kernel family for this shape that fits the
    device (some candidates exceed shared memory; the autotuner skips those)."""
    seen = {}
    for c in gi.candidates(op, M, N, z):
        impl = c.get("impl", 0)
        if impl in seen:
            continue
        try:
            seen[impl] = (c, tsm.Plan(op, "z" if z else "d", M, N, 0,
                                      config=gi.to_tsm_config(op, c, 3, 2)))
        except tsm.TsmError as e:
            if e.status != 2:  # only TSM_ERR_UNSUPPORTED (resources) may be skipped
                raise
    return seen


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", SHAPES)
def test_every_family(tsm, M, N, cplx):
    dt = "z" if cplx else "d"
    for op in ("tsmttsm", "tsmm"):
        fams = per_impl(tsm, op, M, N, cplx)
        assert fams
        for impl, (c, plan) in sorted(fams.items()):
            assert plan.config()["kernel"] == impl
            for K in K_LIST:
                A = ti.matrix(K, M, "A", complex_=cplx, seed=K)
                if op == "tsmttsm":
                    B = ti.matrix(K, N, "B", complex_=cplx, seed=K)
                    got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
                    ref, bound = oracle.tsmttsm(A, B)
                    tol = 1e-12
                else:
                    Cm = ti.matrix(M, N, "C", complex_=cplx, seed=K)
                    got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), plan=plan)
                    ref, bound = oracle.tsmm(A, Cm)
                    tol = 1e-13
                torch.cuda.synchronize()
                r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
                assert r <= tol, (op, dt, M, N, impl, c, K, r, wi)


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
def test_cstationary_int_bitwise(tsm, cplx):
    M, N, K = 64, 48, 100001
    dt = "z" if cplx else "d"
    cands = gi.tsmm_cst_configs(M, N, cplx)
    assert cands
    A = ti.matrix(K, M, "A", complex_=cplx, mode="int")
    Cm = ti.matrix(M, N, "C", complex_=cplx, mode="int")
    ref, _ = oracle.tsmm(A, Cm)
    for c in cands[:: max(1, len(cands) // 4)]:
        plan = tsm.Plan("tsmm", dt, M, N, 0, config=gi.to_tsm_config("tsmm", c, 3, 1))
        got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), ref), c


@pytest.mark.parametrize("cplx", [False, True], ids=["D", "Z"])
@pytest.mark.parametrize("M,N", [(49, 49), (33, 17), (17, 33), (57, 58), (9, 10), (50, 50), (42, 34)])
def test_dmma_edge_warp(tsm, M, N, cplx):
    """DMMA core + DFMA edge warps (kernel | 16, warp count in bits 6-7): every edge candidate family."""
    dt = "z" if cplx else "d"
    cands = gi.edge_candidates(M, N, cplx)
    assert cands
    picked = {}
    for c in cands:
        picked.setdefault((c["impl"], c["EDGE"], c.get("PAIR", 0)), c)  # 1, 2, 4 edge warps; paired core
    for (impl, _, _), c in picked.items():
        plan = tsm.Plan("tsmttsm", dt, M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 2))
        assert plan.config()["kernel"] == impl | (gi.flags(c) << 4)
        assert "edge" in plan.describe(1000)["kernel"]
        for K in (1, 7, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 1)
            B = ti.matrix(K, N, "B", complex_=cplx, seed=K + 2)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, impl, c, K, r, wi)
        Ai = ti.matrix(70001, M, "A", complex_=cplx, mode="int")
        Bi = ti.matrix(70001, N, "B", complex_=cplx, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi)[0])


@pytest.mark.parametrize("M,N", [(64, 64), (48, 16), (40, 40), (34, 18), (16, 16), (62, 50), (20, 64), (56, 56), (56, 24)])
def test_dmma_pair_loads(tsm, M, N):
    """Real DMMA TSMTTSM with paired 16-byte fragment loads (kernel | 32):
    bulk-copy (padded conflict-free strides) and TMA (swizzle-aware k-row remap)
    variants, ragged K and an integer-valued bitwise check of the C-cell mapping."""
    cands = gi.pair_candidates(M, N, False)
    assert cands
    picked = {}
    for c in cands:
        picked.setdefault((c["impl"], c["NT"]), c)
    assert {i for i, _ in picked} >= ({2} if M % 2 == 0 else set())
    for (impl, _), c in sorted(picked.items()):
        try:
            plan = tsm.Plan("tsmttsm", "d", M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] == impl | 32
        assert "pair" in plan.describe(1000)["kernel"]
        for K in (1, 6, 4099, 65537):
            A = ti.matrix(K, M, "A", seed=K + 3)
            B = ti.matrix(K, N, "B", seed=K + 4)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, impl, c, K, r, wi)
        Ai = ti.matrix(70001, M, "A", mode="int")
        Bi = ti.matrix(70001, N, "B", mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi)[0]), c


@pytest.mark.parametrize("op", ["tsmttsm", "tsmm"])
@pytest.mark.parametrize("M,N", [(17, 17), (9, 12), (33, 20), (8, 8), (25, 25), (40, 48)])
def test_complex_as_real(tsm, op, M, N):
    """Z through the real kernels on the interleaved 2M x 2N view (kernel | 256):
    every family the generator offers (TMA / bulk, pair, edge), ragged K, and
    integer-valued inputs bit-exact against the oracle."""
    cands = gi.zr_candidates(op, M, N)
    if not cands:
        pytest.skip("no complex-as-real candidate for this shape")
    picked = {}
    for c in cands:
        picked.setdefault((c.get("impl"), c.get("PAIR", 0), c.get("EDGE", 0)), c)
    ran = 0
    for key, c in sorted(picked.items()):
        try:
            plan = tsm.Plan(op, "z", M, N, 0, config=gi.to_tsm_config(op, c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 256
        assert "complex-as-real" in plan.describe(1000)["kernel"]
        ran += 1
        for K in (1, 5, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 11)
            if op == "tsmttsm":
                B = ti.matrix(K, N, "B", complex_=True, seed=K + 12)
                got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
                ref, bound = oracle.tsmttsm(A, B)
                tol = 1e-12
            else:
                Cm = ti.matrix(M, N, "C", complex_=True, seed=K + 13)
                got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), plan=plan)
                ref, bound = oracle.tsmm(A, Cm)
                tol = 1e-13
            torch.cuda.synchronize()
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= tol, (op, M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", complex_=True, mode="int")
        if op == "tsmttsm":
            Bi = ti.matrix(30001, N, "B", complex_=True, mode="int")
            got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan)
            ref = oracle.tsmttsm(Ai, Bi)[0]
        else:
            Ci = ti.matrix(M, N, "C", complex_=True, mode="int")
            got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
            ref = oracle.tsmm(Ai, Ci)[0]
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), ref), (key, c)
    assert ran


@pytest.mark.parametrize("conj", [False, True], ids=["T", "H"])
@pytest.mark.parametrize("M,N", [(32, 32), (17, 17), (25, 9), (40, 48), (64, 64), (8, 8), (3, 20)])
def test_tsmttsm_3m(tsm, M, N, conj):
    """Z TSMTTSM by 3M / Gauss products (kernel | 512): T1 = Ar^T Br,
    T2 = Ai^T Bi, T3 = (Ar+Ai)^T (Br+Bi); every family the generator offers
    (bulk / TMA, edge warps), plain and conjugate (A^H B), ragged K within the
    1e-12 |A|^T|B| tolerance, integer-valued inputs bit-exact."""
    base = [c for c in gi.candidates("tsmttsm", M, N, True) if c.get("G3")]
    if not base:
        pytest.skip("no DMMA candidate for this shape")
    picked = {}
    for c in base:
        picked.setdefault((c.get("impl"), c.get("EDGE", 0)), c)
    ran = 0
    for key, c in sorted(picked.items()):
        try:
            plan = tsm.Plan("tsmttsm", "z", M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1), conj=conj)
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 512 and "+3m" in plan.describe(1000)["kernel"]
        ran += 1
        for K in (1, 6, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 21)
            B = ti.matrix(K, N, "B", complex_=True, seed=K + 22)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan, conj=conj)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B, conj=conj)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", complex_=True, mode="int")
        Bi = ti.matrix(30001, N, "B", complex_=True, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan, conj=conj)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi, conj=conj)[0]), (key, c)
    assert ran


@pytest.mark.parametrize("dt,M,N", [("d", 41, 41), ("d", 50, 50), ("d", 57, 57), ("d", 33, 20), ("d", 12, 9),
                                    ("z", 17, 17), ("z", 33, 33), ("z", 9, 25), ("z", 20, 20)])
def test_tsmttsm_inline_edge(tsm, dt, M, N):
    """Inline edge (kernel | 2048): DMMA core + the edge strips computed by the
    consumer warps between their DMMAs -- every family the generator offers
    (bulk / TMA, pair, 3M, complex-as-real), plain and conjugate for Z, ragged
    K within tolerance, integer inputs bit-exact."""
    cplx = dt == "z"
    base = [c for c in gi.candidates("tsmttsm", M, N, cplx) if c.get("EI")]
    if not base:
        pytest.skip("no inline-edge candidate for this shape")
    picked = {}
    for c in base:
        picked.setdefault((c.get("impl"), c.get("PAIR", 0), c.get("G3", 0), c.get("ZR", 0)), c)
    ran = 0
    for key, c in sorted(picked.items()):
        for conj in ([False, True] if cplx else [False]):
            try:
                plan = tsm.Plan("tsmttsm", dt, M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1), conj=conj)
            except tsm.TsmError as e:
                if e.status != 2:
                    raise
                continue
            assert plan.config()["kernel"] & 2048 and "inline-edge" in plan.describe(1000)["kernel"]
            ran += 1
            for K in (1, 7, 4099, 65537):
                A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 71)
                B = ti.matrix(K, N, "B", complex_=cplx, seed=K + 72)
                got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan, conj=conj)
                torch.cuda.synchronize()
                ref, bound = oracle.tsmttsm(A, B, conj=conj)
                r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
                assert r <= 1e-12, (M, N, key, c, conj, K, r, wi)
            Ai = ti.matrix(30001, M, "A", complex_=cplx, mode="int")
            Bi = ti.matrix(30001, N, "B", complex_=cplx, mode="int")
            got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan, conj=conj)
            torch.cuda.synchronize()
            assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi, conj=conj)[0]), (key, c, conj)
    assert ran


@pytest.mark.parametrize("M,N,cfg", [
    (64, 64, {"G3": 1, "NBW": 1, "NT": 544, "R": 32, "WR": 1, "impl": 3}),
    (57, 57, {"G3": 1, "NBW": 1, "NT": 544, "R": 32, "WR": 2, "impl": 3}),
    (49, 49, {"EDGE": 1, "G3": 1, "NBW": 1, "NT": 416, "R": 16, "WR": 1, "impl": 3}),
])
def test_tsmm_3m_recomputed_sums(tsm, M, N, cfg):
    """3M C-stationary configurations whose C slice (Re c, Im c, Re c + Im c)
    exceeds the register budget: the kernel keeps Re c, Im c and recomputes
    the sum per k-step (TsmmCstCfg::G3R).  Tolerance on ragged K, plain and
    conjugate; integer-valued inputs bit-exact."""
    for conj in (False, True):
        plan = tsm.Plan("tsmm", "z", M, N, 0, config=gi.to_tsm_config("tsmm", cfg, 4, 1), conj=conj)
        assert plan.config()["kernel"] & 512
        for K in (1, 33, 4099, 100003):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 41)
            Cm = ti.matrix(M, N, "C", complex_=True, seed=K + 42)
            B0 = np.zeros((K, N), dtype=np.complex128)
            got = torch.from_numpy(B0).cuda()
            tsm.tsmm_update(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), got, 1.0, 0.0,
                            plan=plan, conj=conj)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmm_update(A, Cm, B0, 1.0, 0.0, conj=conj)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-13, (M, N, cfg, conj, K, r, wi)
        Ai = ti.matrix(20001, M, "A", complex_=True, mode="int")
        Ci = ti.matrix(M, N, "C", complex_=True, mode="int")
        B0 = np.zeros((20001, N), dtype=np.complex128)
        got = torch.from_numpy(B0).cuda()
        tsm.tsmm_update(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), got, 1.0, 0.0,
                        plan=plan, conj=conj)
        torch.cuda.synchronize()
        ref = oracle.tsmm_update(Ai, Ci, B0, 1.0, 0.0, conj=conj)[0]
        assert np.array_equal(got.cpu().numpy(), ref), (M, N, cfg, conj)


@pytest.mark.parametrize("conj", [False, True], ids=["C", "conjC"])
@pytest.mark.parametrize("M,N", [(32, 32), (17, 17), (24, 40), (64, 64), (9, 8), (50, 13)])
def test_tsmm_3m(tsm, M, N, conj):
    """Z TSMM by 3M / Gauss products (C-stationary kernel 3 | 512, with and
    without DFMA edge columns): B = A C and the update B <- alpha A C + beta B
    (conj: A conj(C)) within the 1e-13 |A||C| tolerance on ragged K;
    integer-valued inputs bit-exact."""
    cands = [c for c in gi.candidates("tsmm", M, N, True) if c.get("G3")]
    if not cands:
        pytest.skip("no C-stationary candidate for this shape")
    picked = {}
    for c in cands:
        picked.setdefault((c.get("EDGE", 0), c["NBW"]), c)
    ran = 0
    for key, c in sorted(picked.items()):
        try:
            plan = tsm.Plan("tsmm", "z", M, N, 0, config=gi.to_tsm_config("tsmm", c, 3, 1), conj=conj)
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 512 and "+3m" in plan.describe(1000)["kernel"]
        ran += 1
        for K in (1, 9, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 31)
            Cm = ti.matrix(M, N, "C", complex_=True, seed=K + 32)
            B0 = ti.matrix(K, N, "B", complex_=True, seed=K + 33)
            Bg = torch.from_numpy(B0).cuda()
            alpha, beta = (0.5 - 0.25j), (1.0 if K % 2 else 0.0)
            tsm.tsmm_update(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), Bg, alpha, beta,
                            plan=plan, conj=conj)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmm_update(A, Cm, B0, alpha, beta, conj=conj)
            r, wi, _ = oracle.max_err_ratio(Bg.cpu().numpy(), ref, bound)
            assert r <= 1e-13, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(20001, M, "A", complex_=True, mode="int")
        Ci = ti.matrix(M, N, "C", complex_=True, mode="int")
        if conj:
            got = torch.zeros(20001, N, dtype=torch.complex128, device="cuda")
            tsm.tsmm_update(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), got, 1.0, 0.0,
                            plan=plan, conj=True)
            ref = oracle.tsmm(Ai, np.conj(Ci))[0]
        else:
            got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
            ref = oracle.tsmm(Ai, Ci)[0]
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), ref), (key, c)
    assert ran


@pytest.mark.parametrize("cplx,zr", [(False, False), (True, False), (True, True)], ids=["D", "Z", "ZR"])
@pytest.mark.parametrize("M,N", [(50, 50), (42, 34), (16, 20), (17, 17), (9, 12), (64, 57)])
def test_tsmm_edge_columns(tsm, M, N, cplx, zr):
    """C-stationary TSMM with the last N mod 8 columns by DFMA (kernel 3 | 16):
    ragged K, integer bit-exact; complex native and complex-as-real."""
    if zr:
        cands = [c for c in gi.zr_candidates("tsmm", M, N) if c.get("EDGE")]
    else:
        cands = gi.tsmm_cst_configs(M, N, cplx, edge=True)
    if not cands:
        pytest.skip("no edge-column configuration for this shape")
    dt = "z" if cplx else "d"
    for c in cands[:: max(1, len(cands) // 3)]:
        try:
            plan = tsm.Plan("tsmm", dt, M, N, 0, config=gi.to_tsm_config("tsmm", c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 16 and "edge-columns" in plan.describe(1000)["kernel"]
        for K in (1, 9, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 41)
            Cm = ti.matrix(M, N, "C", complex_=cplx, seed=K + 42)
            got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmm(A, Cm)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-13, (M, N, c, K, r, wi)
        Ai = ti.matrix(40001, M, "A", complex_=cplx, mode="int")
        Ci = ti.matrix(M, N, "C", complex_=cplx, mode="int")
        got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmm(Ai, Ci)[0]), c


@pytest.mark.parametrize("op", ["tsmttsm", "tsmm"])
@pytest.mark.parametrize("dt,M,N", [("d", 48, 48), ("d", 56, 56), ("d", 41, 41), ("z", 32, 32), ("d", 63, 63)])
def test_plain_warp_order(tsm, op, dt, M, N):
    """The tuned DMMA plan with the consumer-warp order flipped (kernel ^ 1024,
    a launch argument): same cells, other warp -> (slot, tile) assignment;
    ragged K within tolerance, integer-valued inputs bit-exact."""
    base = tsm.get_plan(op, dt, M, N, 0)
    if not base.config()["kernel"] & 15:
        pytest.skip("not a DMMA plan")
    cfg = dict(base.config())
    cfg["kernel"] ^= 1024
    plan = tsm.Plan(op, dt, M, N, 0, config=cfg)
    assert plan.config()["kernel"] == cfg["kernel"]
    assert ("plain-warp-order" in plan.describe(1000)["kernel"]) == bool(cfg["kernel"] & 1024)
    cplx = dt == "z"
    for K in (3, 4099, 65537):
        A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 51)
        if op == "tsmttsm":
            B = ti.matrix(K, N, "B", complex_=cplx, seed=K + 52)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
            ref, bound = oracle.tsmttsm(A, B)
            tol = 1e-12
        else:
            Cm = ti.matrix(M, N, "C", complex_=cplx, seed=K + 53)
            got = tsm.tsmm(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), plan=plan)
            ref, bound = oracle.tsmm(A, Cm)
            tol = 1e-13
        torch.cuda.synchronize()
        r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
        assert r <= tol, (op, dt, M, N, cfg, K, r, wi)
    Ai = ti.matrix(30001, M, "A", complex_=cplx, mode="int")
    if op == "tsmttsm":
        Bi = ti.matrix(30001, N, "B", complex_=cplx, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan)
        ref = oracle.tsmttsm(Ai, Bi)[0]
    else:
        Ci = ti.matrix(M, N, "C", complex_=cplx, mode="int")
        got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
        ref = oracle.tsmm(Ai, Ci)[0]
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), ref), cfg


@pytest.mark.parametrize("dt,M,N", [("d", 57, 57), ("d", 49, 49), ("d", 41, 41), ("d", 63, 63), ("d", 13, 29),
                                    ("d", 9, 9), ("z", 17, 17), ("z", 25, 11), ("z", 9, 31)])
def test_tsmm_cstb_edge_columns(tsm, dt, M, N):
    """C-stationary bulk-copy TSMM (kernel 4) with the last N mod 8 columns by
    DFMA (kernel | 16): every NBW / WR class the generator offers, B = A C and
    the update B <- alpha A C + beta B (beta 0, 1, 2: store, bulk reduce-add,
    scale pass) on ragged K (odd K: the global last-row path) within the 1e-13
    |A||C| tolerance; integer-valued inputs bit-exact."""
    cplx = dt == "z"
    cands = [c for c in gi.candidates("tsmm", M, N, cplx) if c.get("impl") == 4 and c.get("EDGE")]
    assert cands, "no kernel-4 edge-column candidate"
    picked = {}
    for c in cands:
        picked.setdefault((c["NBW"], c["WR"]), c)
    ran = 0
    for key, c in sorted(picked.items())[:4]:
        try:
            plan = tsm.Plan("tsmm", dt, M, N, 0, config=gi.to_tsm_config("tsmm", c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 16 and "dfma-edge-columns" in plan.describe(1000)["kernel"]
        ran += 1
        for K, beta in ((1, 0.0), (9, 1.0), (4099, 2.0), (65537, 0.0), (65536, 1.0)):
            A = ti.matrix(K, M, "A", complex_=cplx, seed=K + 41)
            Cm = ti.matrix(M, N, "C", complex_=cplx, seed=K + 42)
            B0 = ti.matrix(K, N, "B", complex_=cplx, seed=K + 43)
            Bg = torch.from_numpy(B0).cuda()
            alpha = (0.5 - 0.25j) if cplx else 0.75
            tsm.tsmm_update(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), Bg, alpha, beta, plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmm_update(A, Cm, B0, alpha, beta)
            r, wi, _ = oracle.max_err_ratio(Bg.cpu().numpy(), ref, bound)
            assert r <= 1e-13, (M, N, key, c, K, beta, r, wi)
        Ai = ti.matrix(20001, M, "A", complex_=cplx, mode="int")
        Ci = ti.matrix(M, N, "C", complex_=cplx, mode="int")
        got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmm(Ai, Ci)[0]), (key, c)
    assert ran


@pytest.mark.parametrize("M,N", [(57, 57), (63, 63), (33, 20), (9, 41), (41, 9), (49, 49)])
def test_tsmm_win16_row_windows(tsm, M, N):
    """TSMM kernels 1 (dense) and 4 with an odd-width D stage and WR even use
    16-row windows (win16_row) for the MMA rows: every such candidate (and the
    edge-column variants) on ragged K, store and reduce-add (beta = 1),
    within tolerance; integer-valued inputs bit-exact."""
    cands = [c for c in gi.candidates("tsmm", M, N, False)
             if c.get("impl") in (1, 4) and c.get("WR", 1) % 2 == 0 and c.get("AP", M) % 2 == 1]
    picked = {}
    for c in cands:
        picked.setdefault((c["impl"], c["WR"], c.get("EDGE", 0), c.get("NBW", 0)), c)
    assert picked, "no window candidate"
    ran = 0
    for key, c in sorted(picked.items())[:6]:
        try:
            plan = tsm.Plan("tsmm", "d", M, N, 0, config=gi.to_tsm_config("tsmm", c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        ran += 1
        for K, beta in ((1, 0.0), (17, 1.0), (4099, 0.0), (65537, 1.0), (65536, 0.0)):
            A = ti.matrix(K, M, "A", seed=K + 51)
            Cm = ti.matrix(M, N, "C", seed=K + 52)
            B0 = ti.matrix(K, N, "B", seed=K + 53)
            Bg = torch.from_numpy(B0).cuda()
            tsm.tsmm_update(torch.from_numpy(A).cuda(), torch.from_numpy(Cm).cuda(), Bg, 1.0, beta, plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmm_update(A, Cm, B0, 1.0, beta)
            r, wi, _ = oracle.max_err_ratio(Bg.cpu().numpy(), ref, bound)
            assert r <= 1e-13, (M, N, key, c, K, beta, r, wi)
        Ai = ti.matrix(20001, M, "A", mode="int")
        Ci = ti.matrix(M, N, "C", mode="int")
        got = tsm.tsmm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Ci).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmm(Ai, Ci)[0]), (key, c)
    assert ran


@pytest.mark.parametrize("M,N", [(57, 57), (49, 49), (41, 41), (33, 33), (9, 9), (58, 58), (60, 60), (17, 42),
                                 (50, 11), (35, 59)])
def test_tsmttsm_lblocks(tsm, M, N):
    """L-blocks (kernel | 4096, D): the cells outside the 8-aligned core on MMA
    blocks pairing edge rows with core columns and core rows with edge columns
    -- every family the generator offers (bulk / TMA, pair loads) on ragged K
    (odd K: the global last-row path) within the 1e-12 |A|^T|B| tolerance,
    integer-valued inputs bit-exact (every edge cell written exactly once)."""
    base = [c for c in gi.candidates("tsmttsm", M, N, False) if c.get("LB")]
    if not base:
        pytest.skip("L-blocks do not pay for this shape")
    picked = {}
    for c in base:
        picked.setdefault((c.get("impl"), c.get("PAIR", 0), c["MT"], c["NTL"]), c)
    ran = 0
    for key, c in sorted(picked.items())[:6]:
        try:
            plan = tsm.Plan("tsmttsm", "d", M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1))
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert plan.config()["kernel"] & 4096 and "l-blocks" in plan.describe(1000)["kernel"]
        ran += 1
        for K in (1, 7, 4099, 65537):
            A = ti.matrix(K, M, "A", seed=K + 81)
            B = ti.matrix(K, N, "B", seed=K + 82)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", mode="int")
        Bi = ti.matrix(30001, N, "B", mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi)[0]), (key, c)
    assert ran


@pytest.mark.parametrize("conj", [False, True], ids=["T", "H"])
@pytest.mark.parametrize("M,N", [(17, 17), (21, 21), (33, 33), (57, 57), (25, 9)])
def test_tsmttsm_zr_lblocks(tsm, M, N, conj):
    """Z TSMTTSM as the real kernel on the interleaved 2M x 2N view
    (complex-as-real, kernel | 256) with L-blocks on that real product
    (kernel | 4096): plain and conjugate, ragged K within tolerance, integer
    inputs bit-exact."""
    base = [c for c in gi.candidates("tsmttsm", M, N, True) if c.get("LB") and c.get("ZR")]
    if not base:
        pytest.skip("no complex-as-real L-block candidate")
    picked = {}
    for c in base:
        picked.setdefault((c.get("impl"), c.get("PAIR", 0)), c)
    ran = 0
    for key, c in sorted(picked.items()):
        try:
            plan = tsm.Plan("tsmttsm", "z", M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1), conj=conj)
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        kname = plan.describe(1000)["kernel"]
        assert "l-blocks" in kname and "complex-as-real" in kname
        ran += 1
        for K in (1, 7, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 91)
            B = ti.matrix(K, N, "B", complex_=True, seed=K + 92)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan, conj=conj)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B, conj=conj)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", complex_=True, mode="int")
        Bi = ti.matrix(30001, N, "B", complex_=True, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan, conj=conj)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi, conj=conj)[0]), (key, c)
    assert ran


@pytest.mark.parametrize("conj", [False, True], ids=["T", "H"])
@pytest.mark.parametrize("M,N", [(17, 17), (33, 33), (57, 57), (9, 9), (25, 41)])
def test_tsmttsm_z_lblocks(tsm, M, N, conj):
    """Native complex TSMTTSM with L-blocks (kernel | 4096): the 4-DMMA and
    the 3M (kernel | 512) forms, bulk / TMA, plain and conjugate, ragged K
    within the 1e-12 |A|^T|B| tolerance, integer inputs bit-exact."""
    base = [c for c in gi.candidates("tsmttsm", M, N, True) if c.get("LB") and not c.get("ZR")]
    if not base:
        pytest.skip("no native complex L-block candidate")
    picked = {}
    for c in base:
        picked.setdefault((c.get("impl"), c.get("G3", 0)), c)
    ran = 0
    for key, c in sorted(picked.items()):
        try:
            plan = tsm.Plan("tsmttsm", "z", M, N, 0, config=gi.to_tsm_config("tsmttsm", c, 3, 1), conj=conj)
        except tsm.TsmError as e:
            if e.status != 2:
                raise
            continue
        assert "l-blocks" in plan.describe(1000)["kernel"]
        ran += 1
        for K in (1, 7, 4099, 65537):
            A = ti.matrix(K, M, "A", complex_=True, seed=K + 95)
            B = ti.matrix(K, N, "B", complex_=True, seed=K + 96)
            got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan, conj=conj)
            torch.cuda.synchronize()
            ref, bound = oracle.tsmttsm(A, B, conj=conj)
            r, wi, _ = oracle.max_err_ratio(got.cpu().numpy(), ref, bound)
            assert r <= 1e-12, (M, N, key, c, K, r, wi)
        Ai = ti.matrix(30001, M, "A", complex_=True, mode="int")
        Bi = ti.matrix(30001, N, "B", complex_=True, mode="int")
        got = tsm.tsmttsm(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), plan=plan, conj=conj)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), oracle.tsmttsm(Ai, Bi, conj=conj)[0]), (key, c)
    assert ran
