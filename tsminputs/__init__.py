"""Seeded, counter-based synthetic inputs for libtsm.

This module holds NONE of the method's arithmetic: it only produces input
matrices.  It is shared by the oracle side (tests) and the product side
(bench.py host buffers); the CUDA library implements the *same* counter-based
generator independently (``tsm_fill_d``/``tsm_fill_z`` in libtsm), and
tests/test_inputs*.py check that the two agree on sampled indices.

Generator (splitmix64 finaliser, "splitmix-style 64-bit mix
of (seed, index)"):

    mix64(z): z += 0x9E3779B97F4A7C15
              z  = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
              z  = (z ^ (z >> 27)) * 0x94D049BB133111EB
              z ^= z >> 31
    h = mix64(seed * 0xD1B54A32D192ED03 + (id << 48) + i)      (mod 2^64)

``id`` names the matrix (A=1, B=2, C=3); ``i`` is the flat element index of
the row-major matrix (complex: ``i = 2*elem + {0: re, 1: im}``).

    mode "fp" : x = ((h >> 11) - 2^52) * 2^-52   uniform in [-1, 1), exact
    mode "int": x = (h >> 53) - 1024             integers in [-1024, 1023]

"int" mode makes every partial sum an exactly representable integer
(|C| <= K * 2^20 < 2^53 for K < 2^33), so any summation order is exact and
GPU and oracle must agree bit for bit.

The shapes mirror the paper's workload (K >= 10^6 rows,
1..64 columns; K = 2^29/M in PAPER.md:741); values are value-independent for
performance (no data-dependent control flow in any kernel).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

MAT_ID = {"A": 1, "B": 2, "C": 3}
SEED_FP = 42
SEED_INT = 7

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SEEDMUL = np.uint64(0xD1B54A32D192ED03)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def key(seed: int, mat: str) -> np.uint64:
    """Base counter for (seed, matrix id): seed * C + (id << 48) mod 2^64."""
    return np.uint64((int(seed) * 0xD1B54A32D192ED03 + (MAT_ID[mat] << 48)) % (1 << 64))


# ---------------------------------------------------------------------------
# gen.c: the same generator in C (OpenMP), for full-size host regeneration.
# ---------------------------------------------------------------------------
_HERE = os.path.dirname(os.path.abspath(__file__))
_GEN_SRC = os.path.join(_HERE, "gen.c")
_GEN_LIB = os.path.join(_HERE, "libtsmgen.so")
_gen = None
_MODE = {"fp": 0, "int": 1}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_GEN_LIB) or os.path.getmtime(_GEN_LIB) < os.path.getmtime(_GEN_SRC):
        tmp = _GEN_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c99", "-o", tmp, _GEN_SRC])
        os.replace(tmp, _GEN_LIB)
    return _GEN_LIB


def _lib():
    global _gen
    if _gen is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        u64, i64 = ctypes.c_uint64, ctypes.c_int64
        lib.tsmgen_strided.argtypes = [dp, i64, u64, u64, u64, ctypes.c_int]
        lib.tsmgen_strided.restype = None
        lib.tsmgen_columns.argtypes = [dp, i64, i64, i64, ctypes.POINTER(i64), ctypes.c_int, u64, ctypes.c_int,
                                       ctypes.c_int]
        lib.tsmgen_columns.restype = None
        _gen = lib
    return _gen


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def raw_values(n: int, seed: int, mat: str, mode: str, start: int = 0) -> np.ndarray:
    """Flat stream of n real values for indices start .. start+n-1 (gen.c)."""
    if mode not in _MODE:
        raise ValueError(f"unknown mode {mode!r}")
    out = np.empty(n, dtype=np.float64)
    _lib().tsmgen_strided(_dptr(out), n, start, 1, int(key(seed, mat)), _MODE[mode])
    return out


def columns(K: int, width: int, cols, mat: str, *, complex_: bool = False, mode: str = "fp",
            seed: int | None = None, row0: int = 0) -> np.ndarray:
    """Rows [row0, row0 + K) of columns `cols` of a `width`-column generator
    matrix as a K x len(cols) array (gen.c)."""
    if seed is None:
        seed = SEED_FP if mode == "fp" else SEED_INT
    c = np.ascontiguousarray(cols, dtype=np.int64)
    if c.size and (c.min() < 0 or c.max() >= width):
        raise ValueError("column out of range")
    out = np.empty((K, c.size), dtype=np.complex128 if complex_ else np.float64)
    _lib().tsmgen_columns(_dptr(out), row0, K, width, c.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), c.size,
                          int(key(seed, mat)), _MODE[mode], int(complex_))
    return out


def raw_values_numpy(n: int, seed: int, mat: str, mode: str, start: int = 0) -> np.ndarray:
    """numpy version of raw_values (the readable definition; tests compare the two)."""
    base = key(seed, mat)
    out = np.empty(n, dtype=np.float64)
    step = 1 << 22
    for s in range(0, n, step):
        e = min(n, s + step)
        with np.errstate(over="ignore"):
            idx = np.arange(start + s, start + e, dtype=np.uint64) + base
        h = mix64(idx)
        if mode == "fp":
            v = (h >> np.uint64(11)).astype(np.int64) - (1 << 52)
            out[s:e] = v.astype(np.float64) * 2.0 ** -52
        elif mode == "int":
            v = (h >> np.uint64(53)).astype(np.int64) - 1024
            out[s:e] = v.astype(np.float64)
        else:
            raise ValueError(f"unknown mode {mode!r}")
    return out


def values_at(idx: np.ndarray, seed: int, mat: str, mode: str) -> np.ndarray:
    """Real values at arbitrary flat indices (same generator as raw_values)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = mix64(idx + key(seed, mat))
    if mode == "fp":
        return ((h >> np.uint64(11)).astype(np.int64) - (1 << 52)).astype(np.float64) * 2.0 ** -52
    if mode == "int":
        return ((h >> np.uint64(53)).astype(np.int64) - 1024).astype(np.float64)
    raise ValueError(f"unknown mode {mode!r}")


def column(K: int, width: int, col: int, mat: str, *, complex_: bool = False, mode: str = "fp",
           seed: int | None = None) -> np.ndarray:
    """Column `col` (length K) of the K x width matrix(K, width, mat, ...)."""
    return columns(K, width, [col], mat, complex_=complex_, mode=mode, seed=seed)[:, 0].copy()


def rows(row_idx: np.ndarray, width: int, mat: str, *, complex_: bool = False, mode: str = "fp",
         seed: int | None = None) -> np.ndarray:
    """Selected rows (len(row_idx) x width) of matrix(K, width, mat, ...)."""
    if seed is None:
        seed = SEED_FP if mode == "fp" else SEED_INT
    r = np.asarray(row_idx, dtype=np.uint64)[:, None]
    elem = r * np.uint64(width) + np.arange(width, dtype=np.uint64)[None, :]
    if complex_:
        re = values_at(2 * elem, seed, mat, mode)
        im = values_at(2 * elem + np.uint64(1), seed, mat, mode)
        return re + 1j * im
    return values_at(elem, seed, mat, mode)


def matrix(rows: int, cols: int, mat: str, *, complex_: bool = False, mode: str = "fp",
           seed: int | None = None) -> np.ndarray:
    """Row-major rows x cols matrix (float64 or complex128) from the generator."""
    if seed is None:
        seed = SEED_FP if mode == "fp" else SEED_INT
    if complex_:
        flat = raw_values(2 * rows * cols, seed, mat, mode)
        return flat.view(np.complex128).reshape(rows, cols)
    return raw_values(rows * cols, seed, mat, mode).reshape(rows, cols)


def walsh(K: int, M: int, scale: float = 1.0) -> np.ndarray:
    """Walsh columns A[k][m] = scale * (-1)^popcount(k & m) (structured input).

    For K a multiple of the next power of two >= M, the columns are mutually
    orthogonal, so A^T A = scale^2 * K * I exactly."""
    k = np.arange(K, dtype=np.uint64)[:, None]
    m = np.arange(M, dtype=np.uint64)[None, :]
    x = k & m
    par = np.zeros(x.shape, dtype=np.uint64)
    while np.any(x):
        par ^= x & np.uint64(1)
        x = x >> np.uint64(1)
    return np.where(par == 1, -scale, scale).astype(np.float64)
