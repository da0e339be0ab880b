"""CPU oracle for libtsm -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_1905_03136_b200`` never imports it, and the two share no code: the
arithmetic lives in ``oracle/oracle.c`` (plain C + OpenMP, explicit ``fma``),
this module only marshals numpy arrays into it.

Definitions (PAPER.md is the authority):
  * TSMTTSM ``C = A^T B``, ``C[m][n] = sum_k A[k][m] B[k][n]``
    -- PAPER.md:64-68 (op definitions), PAPER.md:342-349 (Listing 1).
  * TSMM ``B = A C``, ``B[k][n] = sum_m A[k][m] C[m][n]``
    -- PAPER.md:64-68, PAPER.md:372-375 (reduction along the short M axis).
  * Z = complex128, plain (non-conjugating) transpose -- DESIGN.md reading R1;
    ``conj=True`` gives the conjugate variants of NEXT row N2 (A^H B, A conj(C)).
  * TSMM update ``B <- alpha A C + beta B`` -- NEXT row N1, the classical
    Gram-Schmidt step of PAPER.md:108-112 (alpha = -1, beta = 1).

Every function returns ``(result, bound)`` where ``bound`` is the north-star
tolerance scale ``|A|^T |B|`` (TSMTTSM) or ``|A||C|`` (TSMM).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

# -march=x86-64-v3: AVX2 + FMA so that fma() is one instruction; no fast-math,
# no contraction beyond the explicit fma() calls, no FTZ/DAZ.
CFLAGS = ["-O3", "-march=x86-64-v3", "-fno-fast-math", "-ffp-contract=off",
          "-fopenmp", "-shared", "-fPIC", "-std=c99"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        for name in ("oracle_tsmttsm_d", "oracle_tsmttsm_z", "oracle_tsmttsm_zc", "oracle_tsmm_d",
                     "oracle_tsmm_z"):
            f = getattr(lib, name)
            f.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp]
            f.restype = None
        d, i = ctypes.c_double, ctypes.c_int
        lib.oracle_tsmm_update_d.argtypes = [ctypes.c_int64, i, i, d, dp, dp, d, dp, dp]
        lib.oracle_tsmm_update_d.restype = None
        lib.oracle_tsmm_update_z.argtypes = [ctypes.c_int64, i, i, d, d, dp, dp, d, d, dp, dp, i]
        lib.oracle_tsmm_update_z.restype = None
        i64 = ctypes.c_int64
        lib.oracle_tsmttsm_d_blocks.argtypes = [i64, i, i, dp, dp, dp]
        lib.oracle_tsmttsm_d_blocks.restype = None
        lib.oracle_tsmttsm_z_blocks.argtypes = [i64, i, i, dp, dp, dp, i]
        lib.oracle_tsmttsm_z_blocks.restype = None
        for name in ("oracle_tsmttsm_d_combine", "oracle_tsmttsm_z_combine"):
            getattr(lib, name).argtypes = [i64, i, i, dp, dp, dp]
            getattr(lib, name).restype = None
        lib.oracle_max_err_ratio.argtypes = [ctypes.c_int64, ctypes.c_int, dp, dp, dp,
                                             ctypes.POINTER(ctypes.c_int64), dp]
        lib.oracle_max_err_ratio.restype = ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prep(x: np.ndarray, is_complex: bool) -> np.ndarray:
    dt = np.complex128 if is_complex else np.float64
    if x.dtype != dt:
        raise TypeError(f"oracle expects {dt}, got {x.dtype}")
    return np.ascontiguousarray(x)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def tsmttsm(A: np.ndarray, B: np.ndarray, conj: bool = False):
    """C = A^T B (plain transpose; conj=True: A^H B, complex only -- NEXT N2).
    A: K x M, B: K x N -> (C M x N, bound M x N)."""
    is_c = np.iscomplexobj(A)
    if conj and not is_c:
        raise ValueError("conj applies to complex inputs")
    A = _prep(A, is_c)
    B = _prep(B, is_c)
    K, M = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("A and B must have the same row count K")
    C = np.zeros((M, N), dtype=A.dtype)
    bound = np.zeros((M, N), dtype=np.float64)
    f = (_load().oracle_tsmttsm_zc if conj else _load().oracle_tsmttsm_z) if is_c else _load().oracle_tsmttsm_d
    f(K, M, N, _ptr(A), _ptr(B), _ptr(C), _ptr(bound))
    return C, bound


ORACLE_BLOCK = 1 << 16  # rows per block of the TSMTTSM summation structure (oracle.c)


def tsmttsm_stream(K: int, M: int, N: int, rows, is_complex: bool, conj: bool = False,
                   seg_rows: int = 1 << 22):
    """Streaming TSMTTSM: C = A^T B over K rows without a
    host copy of A or B.  ``rows(k0, k1)`` returns (A[k0:k1], B[k0:k1]) as
    arrays (e.g. regenerated by tsminputs).  Segments are whole 2^16-row
    blocks, so the result equals ``tsmttsm`` on the full arrays bit for bit.
    -> (C M x N, bound M x N)."""
    if seg_rows % ORACLE_BLOCK:
        raise ValueError("segments must be whole oracle blocks")
    lib = _load()
    MN = M * N
    nblk = (K + ORACLE_BLOCK - 1) // ORACLE_BLOCK
    per = 5 if is_complex else 3
    bs = np.zeros(nblk * MN * per + 1, dtype=np.float64)
    for k0 in range(0, K, seg_rows):
        k1 = min(K, k0 + seg_rows)
        A, B = rows(k0, k1)
        A, B = _prep(A, is_complex), _prep(B, is_complex)
        if A.shape != (k1 - k0, M) or B.shape != (k1 - k0, N):
            raise ValueError("rows() returned the wrong shape")
        b0 = k0 // ORACLE_BLOCK
        view = bs[b0 * MN * per:]
        if is_complex:
            lib.oracle_tsmttsm_z_blocks(k1 - k0, M, N, _ptr(A), _ptr(B), _ptr(view), int(conj))
        else:
            lib.oracle_tsmttsm_d_blocks(k1 - k0, M, N, _ptr(A), _ptr(B), _ptr(view))
    C = np.zeros((M, N), dtype=np.complex128 if is_complex else np.float64)
    bound = np.zeros((M, N), dtype=np.float64)
    (lib.oracle_tsmttsm_z_combine if is_complex else lib.oracle_tsmttsm_d_combine)(nblk, M, N, _ptr(bs),
                                                                                   _ptr(C), _ptr(bound))
    return C, bound


def tsmm(A: np.ndarray, C: np.ndarray):
    """B = A C.  A: K x M, C: M x N -> (B K x N, bound K x N)."""
    is_c = np.iscomplexobj(A)
    A = _prep(A, is_c)
    C = _prep(C, is_c)
    K, M = A.shape
    M2, N = C.shape
    if M != M2:
        raise ValueError("A columns must equal C rows")
    B = np.zeros((K, N), dtype=A.dtype)
    bound = np.zeros((K, N), dtype=np.float64)
    f = _load().oracle_tsmm_z if is_c else _load().oracle_tsmm_d
    f(K, M, N, _ptr(A), _ptr(C), _ptr(B), _ptr(bound))
    return B, bound


def tsmm_update(A: np.ndarray, C: np.ndarray, B: np.ndarray, alpha, beta, conj: bool = False):
    """B_new = alpha * A C + beta * B (conj=True: A conj(C), complex only) --
    NEXT N1, the classical Gram-Schmidt update of PAPER.md:108-112 (alpha=-1,
    beta=1).  B is not modified.  -> (B_new K x N, bound K x N)."""
    is_c = np.iscomplexobj(A)
    if conj and not is_c:
        raise ValueError("conj applies to complex inputs")
    A = _prep(A, is_c)
    C = _prep(C, is_c)
    out = _prep(np.array(B, copy=True), is_c)
    K, M = A.shape
    M2, N = C.shape
    if M != M2 or out.shape != (K, N):
        raise ValueError("shape mismatch")
    bound = np.zeros((K, N), dtype=np.float64)
    lib = _load()
    if is_c:
        al, be = complex(alpha), complex(beta)
        lib.oracle_tsmm_update_z(K, M, N, ctypes.c_double(al.real), ctypes.c_double(al.imag), _ptr(A), _ptr(C),
                                 ctypes.c_double(be.real), ctypes.c_double(be.imag), _ptr(out), _ptr(bound),
                                 int(conj))
    else:
        lib.oracle_tsmm_update_d(K, M, N, ctypes.c_double(float(alpha)), _ptr(A), _ptr(C),
                                 ctypes.c_double(float(beta)), _ptr(out), _ptr(bound))
    return out, bound


def max_err_ratio(got: np.ndarray, ref: np.ndarray, bound: np.ndarray):
    """Return (max |got-ref|/bound, worst flat index, max |got-ref|).

    Complex inputs use the complex modulus of the difference (north star)."""
    is_c = np.iscomplexobj(ref)
    got = _prep(np.asarray(got), is_c)
    ref = _prep(np.asarray(ref), is_c)
    bound = np.ascontiguousarray(bound, dtype=np.float64)
    if got.shape != ref.shape or bound.size != ref.size:
        raise ValueError(f"shape mismatch {got.shape} {ref.shape} {bound.shape}")
    wi = ctypes.c_int64(0)
    ma = ctypes.c_double(0)
    r = _load().oracle_max_err_ratio(ref.size, int(is_c), _ptr(got), _ptr(ref), _ptr(bound),
                                     ctypes.byref(wi), ctypes.byref(ma))
    return r, int(wi.value), float(ma.value)
