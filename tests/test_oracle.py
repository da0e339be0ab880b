"""Pins for the CPU oracle (-m "not gpu").

The oracle is checked against things other than itself: values printed in
SPEC.md's worked examples, hand-worked complex cases, exact rational / integer
arithmetic, closed forms (all-ones, Walsh orthogonality), metamorphic
identities and a library routine (numpy matmul).  Each test names the passage
it follows.  A plausible oracle mistake -- a dropped term, a wrong sign, a
transposed operand, a conjugation, a mis-indexed C -- fails at least one of
them (non-square shapes everywhere catch index/transposition mistakes).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tsminputs as ti

U = 2.0 ** -53


def gamma(n):
    return n * U / (1 - n * U)


# --------------------------------------------------------------------------- #
# Worked examples (tests/golden/, each with its citation)                     #
# --------------------------------------------------------------------------- #
def test_spec_example_d(golden):
    g = golden("spec_example_d.json")
    C, bound = oracle.tsmttsm(g["A"], g["B"])
    assert np.array_equal(C, g["C"])
    assert np.array_equal(bound, np.abs(g["A"]).T @ np.abs(g["B"]))


def test_spec_example_z_i_times_i(golden):
    g = golden("spec_example_z_i.json")  # plain transpose -> -1
    C, _ = oracle.tsmttsm(g["A"], g["B"])
    assert C[0, 0] == -1 + 0j


def test_hand_z_2x2(golden):
    g = golden("hand_z_2x2_tsmttsm.json")
    C, _ = oracle.tsmttsm(g["A"], g["B"])
    assert np.array_equal(C, g["C"])
    h = golden("hand_z_2x2_tsmm.json")
    B, _ = oracle.tsmm(h["A"], h["C"])
    assert np.array_equal(B, h["B"])


@pytest.mark.parametrize("K,M", [(1, 1), (37, 5), (1000, 64), (3, 17)])
@pytest.mark.parametrize("cplx", [False, True])
def test_tsmm_identity(K, M, cplx):
    # TSMM with C = identity gives B = A exactly.
    A = ti.matrix(K, M, "A", complex_=cplx)
    I = np.eye(M, dtype=np.complex128 if cplx else np.float64)
    B, bound = oracle.tsmm(A, I)
    assert np.array_equal(B, A)
    assert np.allclose(bound, np.abs(A), rtol=4e-16, atol=0)  # |a|*1 (hypot vs np.abs rounding)


# --------------------------------------------------------------------------- #
# Exact rational brute force on tiny inputs (Listing 1 evaluated exactly)     #
# --------------------------------------------------------------------------- #
def _exact_tsmttsm(A, B):
    K, M = A.shape
    N = B.shape[1]
    C = [[0] * N for _ in range(M)]
    cplx = np.iscomplexobj(A)
    for m in range(M):
        for n in range(N):
            if cplx:
                re = Fraction(0)
                im = Fraction(0)
                for k in range(K):
                    ar, ai = Fraction(A[k, m].real), Fraction(A[k, m].imag)
                    br, bi = Fraction(B[k, n].real), Fraction(B[k, n].imag)
                    re += ar * br - ai * bi
                    im += ar * bi + ai * br
                C[m][n] = (re, im)
            else:
                C[m][n] = sum((Fraction(A[k, m]) * Fraction(B[k, n]) for k in range(K)), Fraction(0))
    return C


def _exact_tsmm(A, C):
    K, M = A.shape
    N = C.shape[1]
    cplx = np.iscomplexobj(A)
    B = [[0] * N for _ in range(K)]
    for k in range(K):
        for n in range(N):
            if cplx:
                re = Fraction(0)
                im = Fraction(0)
                for m in range(M):
                    ar, ai = Fraction(A[k, m].real), Fraction(A[k, m].imag)
                    cr, ci = Fraction(C[m, n].real), Fraction(C[m, n].imag)
                    re += ar * cr - ai * ci
                    im += ar * ci + ai * cr
                B[k][n] = (re, im)
            else:
                B[k][n] = sum((Fraction(A[k, m]) * Fraction(C[m, n]) for m in range(M)), Fraction(0))
    return B


def _check_exact(got, exact, bound, nterms, cplx):
    # Error of an fma chain of n terms is <= gamma_n * sum|terms| (Higham,
    # Accuracy and Stability, Thm 3.1 with fma); complex: each of re/im is a
    # 2n-term real chain bounded by sum |a||b|, modulus adds sqrt(2).
    rows, cols = got.shape
    for i in range(rows):
        for j in range(cols):
            if cplx:
                er = abs(Fraction(got[i, j].real) - exact[i][j][0])
                ei = abs(Fraction(got[i, j].imag) - exact[i][j][1])
                err = math.hypot(float(er), float(ei))
                lim = math.sqrt(2) * gamma(2 * nterms) * bound[i, j]
            else:
                err = float(abs(Fraction(got[i, j]) - exact[i][j]))
                lim = gamma(nterms) * bound[i, j]
            assert err <= lim * 1.0000001 + 1e-300, (i, j, err, lim)


@pytest.mark.parametrize("K,M,N", [(1, 1, 1), (5, 3, 2), (17, 2, 5), (40, 4, 3), (3, 1, 6)])
@pytest.mark.parametrize("cplx", [False, True])
def test_tsmttsm_exact_bruteforce(K, M, N, cplx):
    A = ti.matrix(K, M, "A", complex_=cplx, seed=1000 + K)
    B = ti.matrix(K, N, "B", complex_=cplx, seed=2000 + K)
    C, bound = oracle.tsmttsm(A, B)
    _check_exact(C, _exact_tsmttsm(A, B), bound, K, cplx)


@pytest.mark.parametrize("K,M,N", [(1, 1, 1), (4, 3, 2), (6, 7, 5), (2, 64, 3)])
@pytest.mark.parametrize("cplx", [False, True])
def test_tsmm_exact_bruteforce(K, M, N, cplx):
    A = ti.matrix(K, M, "A", complex_=cplx, seed=3000 + M)
    C = ti.matrix(M, N, "C", complex_=cplx, seed=4000 + M)
    B, bound = oracle.tsmm(A, C)
    _check_exact(B, _exact_tsmm(A, C), bound, M, cplx)


# --------------------------------------------------------------------------- #
# Integer mode: every summation order is exact -> bitwise vs exact integers   #
# --------------------------------------------------------------------------- #
def _int64(a):
    return np.asarray(a).astype(np.int64)


@pytest.mark.parametrize("K,M,N", [(70001, 3, 5), (4099, 64, 64), (131073, 1, 2), (1000, 16, 48)])
def test_tsmttsm_int_exact_d(K, M, N):
    A = ti.matrix(K, M, "A", mode="int")
    B = ti.matrix(K, N, "B", mode="int")
    C, bound = oracle.tsmttsm(A, B)
    ref = _int64(A).T @ _int64(B)  # exact int64 matmul (numpy, no BLAS)
    assert np.array_equal(C, ref.astype(np.float64))
    assert np.array_equal(bound, (np.abs(_int64(A)).T @ np.abs(_int64(B))).astype(np.float64))


@pytest.mark.parametrize("K,M,N", [(66000, 2, 3), (2049, 9, 7)])
def test_tsmttsm_int_exact_z(K, M, N):
    A = ti.matrix(K, M, "A", mode="int", complex_=True)
    B = ti.matrix(K, N, "B", mode="int", complex_=True)
    C, _ = oracle.tsmttsm(A, B)
    Ar, Ai, Br, Bi = _int64(A.real), _int64(A.imag), _int64(B.real), _int64(B.imag)
    re = Ar.T @ Br - Ai.T @ Bi  # plain transpose: no conjugation
    im = Ar.T @ Bi + Ai.T @ Br
    assert np.array_equal(C.real, re.astype(np.float64))
    assert np.array_equal(C.imag, im.astype(np.float64))


@pytest.mark.parametrize("cplx", [False, True])
def test_tsmm_int_exact(cplx):
    K, M, N = 5000, 13, 6
    A = ti.matrix(K, M, "A", mode="int", complex_=cplx)
    C = ti.matrix(M, N, "C", mode="int", complex_=cplx)
    B, _ = oracle.tsmm(A, C)
    if cplx:
        Ar, Ai, Cr, Ci = _int64(A.real), _int64(A.imag), _int64(C.real), _int64(C.imag)
        assert np.array_equal(B.real, (Ar @ Cr - Ai @ Ci).astype(np.float64))
        assert np.array_equal(B.imag, (Ar @ Ci + Ai @ Cr).astype(np.float64))
    else:
        assert np.array_equal(B, (_int64(A) @ _int64(C)).astype(np.float64))


# --------------------------------------------------------------------------- #
# Closed forms                                                               #
# --------------------------------------------------------------------------- #
def test_all_ones():
    K, M, N = 200003, 4, 3
    C, _ = oracle.tsmttsm(np.ones((K, M)), np.ones((K, N)))
    assert np.all(C == K)
    one_i = np.full((K, M), 1 + 1j)
    Cz, _ = oracle.tsmttsm(one_i, np.full((K, N), 1 + 1j))
    assert np.all(Cz == 2j * K)  # (1+i)^2 = 2i; conj would give 2


@pytest.mark.parametrize("K,M", [(4096, 64), (65536 * 2, 33), (64, 64)])
def test_walsh_orthogonal(K, M):
    # Walsh columns are mutually orthogonal: A^T A = K I exactly.
    A = ti.walsh(K, M)
    C, _ = oracle.tsmttsm(A, A)
    assert np.array_equal(C, K * np.eye(M))
    Az = (1 + 1j) * A
    Cz, _ = oracle.tsmttsm(Az, Az)
    assert np.array_equal(Cz, 2j * K * np.eye(M))  # conj(A)^T A would be 2K I


def test_scaled_walsh_orthonormal():
    # K = 4^j, scale 2^-j: orthonormal columns, A^T A = I exactly.
    j = 8
    A = ti.walsh(4 ** j, 32, scale=2.0 ** -j)
    C, _ = oracle.tsmttsm(A, A)
    assert np.array_equal(C, np.eye(32))


def test_column_sums():
    # B = ones(K x 1) -> C = column sums of A; compare with the correctly
    # rounded math.fsum (a library routine) within the oracle's tolerance.
    K, M = 300001, 5
    A = ti.matrix(K, M, "A")
    C, bound = oracle.tsmttsm(A, np.ones((K, 1)))
    for m in range(M):
        ref = math.fsum(A[:, m])
        assert abs(C[m, 0] - ref) <= 1e-15 * bound[m, 0]


# --------------------------------------------------------------------------- #
# Metamorphic identities (exact in integer mode)                             #
# --------------------------------------------------------------------------- #
def test_k_split_additivity():
    K, K1, M, N = 150000, 70001, 6, 5
    A = ti.matrix(K, M, "A", mode="int")
    B = ti.matrix(K, N, "B", mode="int")
    C, _ = oracle.tsmttsm(A, B)
    C1, _ = oracle.tsmttsm(A[:K1], B[:K1])
    C2, _ = oracle.tsmttsm(A[K1:], B[K1:])
    assert np.array_equal(C, C1 + C2)


def test_row_sum_identity():
    # C 1 = A^T (B 1)
    K, M, N = 20000, 7, 9
    A = ti.matrix(K, M, "A", mode="int")
    B = ti.matrix(K, N, "B", mode="int")
    C, _ = oracle.tsmttsm(A, B)
    b1 = B.sum(axis=1, keepdims=True)  # exact: |row sums| < 2^53
    C1, _ = oracle.tsmttsm(A, b1)
    assert np.array_equal(C.sum(axis=1, keepdims=True), C1)


def test_gram_schmidt_identity():
    # A^T (A C) = (A^T A) C  (the two ops chained)
    K, M, N = 4096, 8, 3
    A = ti.matrix(K, M, "A", mode="int")
    Cm = ti.matrix(M, N, "C", mode="int")
    AC, _ = oracle.tsmm(A, Cm)
    lhs, _ = oracle.tsmttsm(A, AC)
    G, _ = oracle.tsmttsm(A, A)
    rhs = (_int64(G) @ _int64(Cm)).astype(np.float64)
    assert np.array_equal(lhs, rhs)


# --------------------------------------------------------------------------- #
# Library cross-check, determinism, negative controls                        #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("K,M,N", [(65536 + 17, 8, 8), (100000, 1, 64), (30000, 64, 1), (20000, 16, 48)])
@pytest.mark.parametrize("cplx", [False, True])
def test_numpy_crosscheck(K, M, N, cplx):
    A = ti.matrix(K, M, "A", complex_=cplx)
    B = ti.matrix(K, N, "B", complex_=cplx)
    C, bound = oracle.tsmttsm(A, B)
    r, _, _ = oracle.max_err_ratio(A.T @ B, C, bound)
    assert r <= 1e-13
    Cm = ti.matrix(M, N, "C", complex_=cplx)
    Bo, bb = oracle.tsmm(A, Cm)
    r, _, _ = oracle.max_err_ratio(A @ Cm, Bo, bb)
    assert r <= 1e-14


def test_thread_count_determinism():
    A = ti.matrix(300000, 5, "A")
    B = ti.matrix(300000, 4, "B")
    n0 = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        C1, _ = oracle.tsmttsm(A, B)
        oracle.set_num_threads(max(2, n0))
        C2, _ = oracle.tsmttsm(A, B)
    finally:
        oracle.set_num_threads(n0)
    assert np.array_equal(C1, C2)


def test_negative_control():
    A = ti.matrix(5000, 3, "A")
    B = ti.matrix(5000, 4, "B")
    C, bound = oracle.tsmttsm(A, B)
    bad = C.copy()
    bad[2, 1] *= 1 + 1e-9
    r, wi, _ = oracle.max_err_ratio(bad, C, bound)
    assert r > 1e-12 and wi == 2 * 4 + 1
    # a transposed result (B^T A instead of A^T B) must be caught
    As, Bs = A[:, :3], B[:, :3]
    Cs, bs = oracle.tsmttsm(As, Bs)
    r, _, _ = oracle.max_err_ratio(oracle.tsmttsm(Bs, As)[0], Cs, bs)
    assert r > 1e-3
    # ... and so must a conjugated transpose
    Az = ti.matrix(100, 2, "A", complex_=True)
    Bz = ti.matrix(100, 2, "B", complex_=True)
    Cz, bz = oracle.tsmttsm(Az, Bz)
    r, _, _ = oracle.max_err_ratio(Az.conj().T @ Bz, Cz, bz)
    assert r > 1e-3


def test_generator_splitmix_reference(golden):
    g = golden("splitmix64.json")
    inp = np.array([int(x, 16) for x in g["inputs"]], dtype=np.uint64)
    out = [int(x) for x in ti.mix64(inp)]
    assert out == [int(x, 16) for x in g["outputs"]]


def test_generator_ranges():
    x = ti.raw_values(1 << 16, 42, "A", "fp")
    assert x.min() >= -1 and x.max() < 1 and abs(x.mean()) < 0.02
    y = ti.raw_values(1 << 16, 7, "B", "int")
    assert y.min() >= -1024 and y.max() <= 1023 and np.all(y == np.round(y))
    # complex interleaving: element e is (flat 2e, flat 2e+1)
    z = ti.matrix(3, 2, "C", complex_=True, seed=5)
    flat = ti.raw_values(12, 5, "C", "fp")
    assert np.array_equal(z.reshape(-1).view(np.float64), flat)


# --------------------------------------------------------------------------- #
# NEXT rows N1 (TSMM update / Gram-Schmidt step) and N2 (conjugate variants)   #
# --------------------------------------------------------------------------- #
def _z(a):
    a = np.array(a, dtype=np.float64)
    return np.ascontiguousarray(a[..., 0] + 1j * a[..., 1])


def test_conj_hand_z_2x2(golden):
    g = golden("hand_z_2x2_tsmttsm_conj.json")
    C, bound = oracle.tsmttsm(g["A"], g["B"], conj=True)
    assert np.array_equal(C, g["C"])
    # the bound is conjugation-invariant (|conj a| = |a|)
    assert np.array_equal(bound, oracle.tsmttsm(g["A"], g["B"])[1])


def test_conj_i_times_i():
    # conj(i) * i = 1 (the plain transpose gives -1)
    C, _ = oracle.tsmttsm(np.array([[1j]]), np.array([[1j]]), conj=True)
    assert C[0, 0] == 1 + 0j


@pytest.mark.parametrize("K,M", [(4096, 64), (64, 33)])
def test_conj_walsh(K, M):
    # (1+i) Walsh: A^H A = |1+i|^2 K I = 2K I exactly (plain: 2iK I)
    Az = (1 + 1j) * ti.walsh(K, M)
    C, _ = oracle.tsmttsm(Az, Az, conj=True)
    assert np.array_equal(C, 2 * K * np.eye(M))


def test_conj_int_exact():
    # integer mode: exact, equals conj(A)^T B computed in exact int64 arithmetic
    K, M, N = 3001, 5, 4
    A = ti.matrix(K, M, "A", complex_=True, mode="int")
    B = ti.matrix(K, N, "B", complex_=True, mode="int")
    C, _ = oracle.tsmttsm(A, B, conj=True)
    ar, ai, br, bi = (_int64(x) for x in (A.real, A.imag, B.real, B.imag))
    re = ar.T @ br + ai.T @ bi
    im = ar.T @ bi - ai.T @ br
    assert np.array_equal(C, re.astype(np.float64) + 1j * im.astype(np.float64))


def test_update_hand(golden):
    g = golden("hand_tsmm_update.json")
    d = g["d"]
    out, bound = oracle.tsmm_update(np.array(d["A"], float), np.array(d["C"], float), np.array(d["B"], float),
                                    d["alpha"], d["beta"])
    assert np.array_equal(out, np.array(d["out"], float))
    assert np.array_equal(bound, [[2 * 3 + 3 * 10], [2 * 4 + 3 * 4]])
    z = g["z_conj"]
    out, _ = oracle.tsmm_update(_z(z["A"]), _z(z["C"]), _z(z["B"]), complex(*z["alpha"]), complex(*z["beta"]),
                                conj=True)
    assert np.array_equal(out, _z(z["out"]))


@pytest.mark.parametrize("cplx", [False, True])
def test_update_reduces_to_tsmm(cplx):
    # alpha = 1, beta = 0: exactly the TSMM oracle (fma(1, s, 0) = s)
    K, M, N = 777, 9, 6
    A = ti.matrix(K, M, "A", complex_=cplx)
    Cm = ti.matrix(M, N, "C", complex_=cplx)
    B0 = ti.matrix(K, N, "B", complex_=cplx)
    out, _ = oracle.tsmm_update(A, Cm, B0, 1, 0)
    ref, _ = oracle.tsmm(A, Cm)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("cplx", [False, True])
def test_update_int_exact(cplx):
    # integer mode: B_new = alpha A C + beta B exactly (int64 arithmetic)
    K, M, N = 2000, 7, 5
    A = ti.matrix(K, M, "A", complex_=cplx, mode="int")
    Cm = ti.matrix(M, N, "C", complex_=cplx, mode="int")
    B0 = ti.matrix(K, N, "B", complex_=cplx, mode="int")
    alpha, beta = (-3, 2) if not cplx else (-3 + 1j, 2 - 2j)
    out, _ = oracle.tsmm_update(A, Cm, B0, alpha, beta)
    if cplx:
        ac = (_int64(A.real) @ _int64(Cm.real) - _int64(A.imag) @ _int64(Cm.imag)) + \
            1j * (_int64(A.real) @ _int64(Cm.imag) + _int64(A.imag) @ _int64(Cm.real))
    else:
        ac = _int64(A) @ _int64(Cm)
    assert np.array_equal(out, alpha * ac + beta * B0)


@pytest.mark.parametrize("cplx", [False, True])
def test_gram_schmidt_projection_exact(cplx):
    # classical Gram-Schmidt of B against an orthonormal A:
    # C = A^T B (A^H B for Z), B' = B - A C  =>  A^T B' = 0.  With the scaled
    # Walsh basis (entries +-2^-j, K = 4^j) and integer B every product and
    # sum is a dyadic rational within 53 bits: the projection is exact.
    j = 6
    K, M, N = 4 ** j, 16, 5
    A = ti.walsh(K, M, scale=2.0 ** -j)
    B = ti.matrix(K, N, "B", complex_=cplx, mode="int")
    if cplx:
        A = 1j * A  # unit-modulus phase: A^H A = I (the plain transpose gives -I)
    C, _ = oracle.tsmttsm(A, B, conj=cplx)
    Bp, _ = oracle.tsmm_update(A, C, B, -1, 1)
    R, _ = oracle.tsmttsm(A, Bp, conj=cplx)
    assert np.count_nonzero(R) == 0
    # and the update removed exactly the projection A C
    AC, _ = oracle.tsmm(A, C)
    assert np.array_equal(Bp, B - AC)


# --------------------------------------------------------------------------- #
# The tolerance scale (bound) and the comparator, pinned by hand values       #
# (a too-large Z bound would loosen every Z test).   #
# --------------------------------------------------------------------------- #
def _r2(v):
    """[a, b] -> a + b*sqrt(2) (hand values of tests/golden/hand_z_bounds.json)."""
    a = np.array(v, dtype=np.float64)
    return a[..., 0] + a[..., 1] * math.sqrt(2)


def test_z_bound_hand_tsmttsm(golden):
    g = golden("hand_z_2x2_tsmttsm.json")
    b = golden("hand_z_bounds.json")
    _, bound = oracle.tsmttsm(g["A"], g["B"])
    assert np.allclose(bound, _r2(b["tsmttsm_bound"]), rtol=4 * U, atol=0)
    # the complex modulus, never |Re|+|Im| (which would give 4 at [0][0], not 2 sqrt 2)
    assert abs(bound[0, 0] - 2 * math.sqrt(2)) <= 12 * U
    _, bc = oracle.tsmttsm(g["A"], g["B"], conj=True)
    assert np.allclose(bc, _r2(b["tsmttsm_bound"]), rtol=4 * U, atol=0)


def test_z_bound_hand_tsmm(golden):
    h = golden("hand_z_2x2_tsmm.json")
    b = golden("hand_z_bounds.json")
    _, bound = oracle.tsmm(h["A"], h["C"])
    assert np.allclose(bound, _r2(b["tsmm_bound"]), rtol=4 * U, atol=0)


def test_z_update_bound_hand(golden):
    u = golden("hand_z_bounds.json")["update_z"]
    out, bound = oracle.tsmm_update(_z(u["A"]), _z(u["C"]), _z(u["B"]), complex(*u["alpha"]),
                                    complex(*u["beta"]))
    assert np.array_equal(out, _z(u["out"]))
    assert np.allclose(bound, _r2(u["bound"]), rtol=4 * U, atol=0)


def test_z_bound_scaling_laws():
    # modulus laws the bound must obey: a unit phase (i^p) on an operand leaves it
    # unchanged, a power-of-two scale s multiplies it by s exactly
    K, M, N = 513, 7, 4
    A = ti.matrix(K, M, "A", complex_=True)
    B = ti.matrix(K, N, "B", complex_=True)
    _, b0 = oracle.tsmttsm(A, B)
    _, b1 = oracle.tsmttsm(1j * A, -1j * B)
    assert np.array_equal(b0, b1)
    _, b2 = oracle.tsmttsm(4.0 * A, B)
    assert np.array_equal(b2, 4.0 * b0)
    Cm = ti.matrix(M, N, "C", complex_=True)
    _, t0 = oracle.tsmm(A, Cm)
    _, t1 = oracle.tsmm(1j * A, 1j * Cm)
    assert np.array_equal(t0, t1)
    # the bound dominates |C| (triangle inequality) and equals the real bound of the moduli
    C, _ = oracle.tsmttsm(A, B)
    assert np.all(np.abs(C) <= b0 * (1 + 1e-12))
    _, br = oracle.tsmttsm(np.abs(A), np.abs(B))
    assert np.allclose(b0, br, rtol=1e-13, atol=0)


def test_comparator_rules():
    # max |got - ref| / bound (north star); Z: modulus of the difference
    ref = np.array([1.0, 2.0, 3.0])
    bound = np.array([1.0, 4.0, 0.25])
    got = np.array([1.0, 4.0, 3.0 - 0.25])
    r, wi, ma = oracle.max_err_ratio(got, ref, bound)
    assert (r, wi, ma) == (1.0, 2, 2.0)  # ratios 0, 0.5, 1.0; the max abs error is at index 1
    # zero bound: exact agreement is ratio 0, any difference is +inf
    r, _, _ = oracle.max_err_ratio(np.array([0.0, 5.0]), np.array([0.0, 5.0]), np.array([0.0, 0.0]))
    assert r == 0.0
    r, wi, _ = oracle.max_err_ratio(np.array([0.0, 5.0 + 2 ** -40]), np.array([0.0, 5.0]), np.array([0.0, 0.0]))
    assert r == math.inf and wi == 1
    # NaN anywhere in the difference: the ratio is NaN, so every "r <= tol" check fails
    r, wi, _ = oracle.max_err_ratio(np.array([1.0, np.nan]), np.array([1.0, 1.0]), np.array([1.0, 1.0]))
    assert math.isnan(r) and wi == 1 and not (r <= 1e-12)
    r, _, _ = oracle.max_err_ratio(np.array([np.inf]), np.array([np.inf]), np.array([1.0]))
    assert math.isnan(r)  # inf - inf
    # complex: |(3+4i) - 0| = 5 (modulus, not max(|re|, |im|) = 4 or |re| + |im| = 7)
    r, _, ma = oracle.max_err_ratio(np.array([3 + 4j]), np.array([0j]), np.array([10.0]))
    assert ma == 5.0 and r == 0.5


def test_generator_c_matches_numpy():
    """tsminputs/gen.c (used for full-size host regeneration) equals the numpy
    definition element for element, real and complex, fp and int modes."""
    import tsminputs as ti
    for mode, seed in (("fp", 42), ("int", 7)):
        for mat in ("A", "B", "C"):
            ref = ti.raw_values_numpy(5000, seed, mat, mode, start=123456789)
            got = ti.raw_values(5000, seed, mat, mode, start=123456789)
            assert np.array_equal(ref, got)
    K, w = 3001, 13
    for cplx in (False, True):
        full = np.stack([ti.values_at(np.arange(K * w * (2 if cplx else 1), dtype=np.uint64), 42, "A", "fp")])[0]
        full = full.view(np.complex128).reshape(K, w) if cplx else full.reshape(K, w)
        cols = [0, 5, 12]
        assert np.array_equal(ti.columns(K, w, cols, "A", complex_=cplx), full[:, cols])
        assert np.array_equal(ti.column(K, w, 12, "A", complex_=cplx), full[:, 12])
        assert np.array_equal(ti.matrix(K, w, "A", complex_=cplx), full)


def test_streaming_mode_equals_one_shot():
    """oracle.tsmttsm_stream (rows regenerated segment by segment, SURVEY.md
    §8(c) streaming mode) equals the one-shot oracle bit for bit, D / Z / conj,
    with a ragged last block and segments of several blocks."""
    import tsminputs as ti
    K = 5 * (1 << 16) + 777
    for cplx, conj in ((False, False), (True, False), (True, True)):
        M, N = 3, 4
        A = ti.columns(K, 7, [0, 2, 6], "A", complex_=cplx)
        B = ti.columns(K, 9, [1, 2, 3, 8], "B", complex_=cplx)

        def rows(k0, k1):
            return (ti.columns(k1 - k0, 7, [0, 2, 6], "A", complex_=cplx, row0=k0),
                    ti.columns(k1 - k0, 9, [1, 2, 3, 8], "B", complex_=cplx, row0=k0))
        ref, rb = oracle.tsmttsm(A, B, conj=conj)
        got, gb = oracle.tsmttsm_stream(K, M, N, rows, cplx, conj=conj, seg_rows=2 << 16)
        assert np.array_equal(got, ref) and np.array_equal(gb, rb)
        # the columns of the full matrices are the same values
        full = ti.matrix(K, 7, "A", complex_=cplx)
        assert np.array_equal(full[:, [0, 2, 6]], A)
