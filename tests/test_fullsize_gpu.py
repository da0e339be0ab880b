"""Full-size parity of every tuned production plan (VERDICT r01 "next" item 1).

For every entry of the tuned table (`tune/b200.json`: all square widths
1..64, D and Z, both ops, plus the non-square shapes) the DEFAULT plan -- the
exact kernel and launch configuration `bench.py` times -- runs at the size it
was tuned and is timed at (K = 2^24; the configs[3] non-square shapes also at
K = 2^25), and sampled outputs are checked one by one against the CPU oracle
(definition PAPER.md:342-349 Listing 1 / PAPER.md:64-68):

* TSMTTSM: a 3 x 3 grid of C cells (rows {0, M-1, random}, columns {0, N-1,
  random}; every cell when M*N <= 9).  The oracle gets only the needed columns
  of A and B, regenerated on the host by tsminputs' generator (gen.c; SURVEY
  §8(c) streaming mode), and computes them with exactly the arithmetic it uses
  for the full matrices (each cell is an independent chunked sum over K).
* TSMM: rows {0, 1}, the last 640 rows (the ragged last chunk of every plan:
  R <= 512 rows per chunk), and 2048 random rows.

The device inputs are written by libtsm's own generator (tsm_fill, the same
counter-based generator implemented independently); every column / row the
oracle uses is first checked to be bit-identical on the device, so no oracle
input comes from the CUDA path.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import tsminputs as ti

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"tsmttsm": 1e-12, "tsmm": 1e-13}
K_TUNE = 1 << 24


def _entries():
    d = json.load(open(os.path.join(ROOT, "tune", "b200.json")))
    out = []
    for key in sorted(d["entries"], key=lambda k: (k.split("_")[1], k.split("_")[0],
                                                   int(k.split("_")[2]), int(k.split("_")[3]))):
        op, dt, M, N = key.split("_")
        out.append((op, dt, int(M), int(N), d["K"]))
    # configs[3]: the non-square shapes at K = 2^25 as well
    for dt in ("d", "z"):
        for op in ("tsmttsm", "tsmm"):
            for (M, N) in ((1, 64), (64, 1), (16, 48), (48, 16)):
                out.append((op, dt, M, N, 1 << 25))
    return out


ENTRIES = _entries()


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


class Buffers:
    """Flat device buffers filled once by tsm_fill; the leading K*w elements
    viewed as K x w are exactly tsminputs.matrix(K, w) (the generator value
    depends only on the flat index)."""

    def __init__(self, tsm):
        self.tsm = tsm
        self.cplx = None
        self.bufs = {}

    def get(self, cplx, mat, n):
        if cplx != self.cplx:  # one dtype resident at a time (Z K=2^25 x 64 is 34 GB)
            self.bufs.clear()
            torch.cuda.empty_cache()
            self.cplx = cplx
        t = self.bufs.get(mat)
        if t is None or t.numel() < n:
            self.bufs.pop(mat, None)
            torch.cuda.empty_cache()
            t = torch.empty(n, dtype=torch.complex128 if cplx else torch.float64, device="cuda")
            if mat != "O":
                self.tsm.fill(t, mat, ti.SEED_FP, "fp")
            self.bufs[mat] = t
        return t


@pytest.fixture(scope="module")
def bufs(tsm):
    b = Buffers(tsm)
    yield b
    b.bufs.clear()
    torch.cuda.empty_cache()


def _pick(w, rng):
    s = {0, w - 1}
    if w > 2:
        s.add(int(rng.integers(1, w - 1)))
    return sorted(s)


def _tsmttsm(tsm, bufs, M, N, K, cplx):
    dt = "z" if cplx else "d"
    A = bufs.get(cplx, "A", K * max(M, N, 64) if K == K_TUNE else K * M)[: K * M].view(K, M)
    B = bufs.get(cplx, "B", K * max(M, N, 64) if K == K_TUNE else K * N)[: K * N].view(K, N)
    plan = tsm.get_plan("tsmttsm", dt, M, N, 0)
    C = tsm.tsmttsm(A, B, plan=plan)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1000 * M + N + (7 if cplx else 0))
    ms, ns = _pick(M, rng), _pick(N, rng)
    a = ti.columns(K, M, ms, "A", complex_=cplx)
    b = ti.columns(K, N, ns, "B", complex_=cplx)
    assert np.array_equal(A[:, ms].cpu().numpy(), a), "device A columns differ from the host generator"
    assert np.array_equal(B[:, ns].cpu().numpy(), b), "device B columns differ from the host generator"
    ref, bound = oracle.tsmttsm(a, b)
    got = C.cpu().numpy()[np.ix_(ms, ns)]
    r, wi, ma = oracle.max_err_ratio(got, ref, bound)
    assert r <= TOL["tsmttsm"], (f"tsmttsm {dt} {M}x{N} K={K} plan {plan.describe(K)}: "
                                 f"max err/bound {r:.3e} at cell {(ms[wi // len(ns)], ns[wi % len(ns)])}")
    return r


def _tsmm(tsm, bufs, M, N, K, cplx):
    dt = "z" if cplx else "d"
    A = bufs.get(cplx, "A", K * max(M, N, 64) if K == K_TUNE else K * M)[: K * M].view(K, M)
    O = bufs.get(cplx, "O", K * max(M, N, 64) if K == K_TUNE else K * N)[: K * N].view(K, N)
    Cd = torch.empty(M, N, dtype=A.dtype, device="cuda")
    tsm.fill(Cd, "C", ti.SEED_FP, "fp")
    O.fill_(float("nan"))  # a row the kernel does not write fails the check
    plan = tsm.get_plan("tsmm", dt, M, N, 0)
    tsm.tsmm(A, Cd, out=O, plan=plan)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2000 * M + N + (7 if cplx else 0))
    rows = np.unique(np.concatenate([[0, 1], np.arange(max(0, K - 640), K), rng.integers(0, K, 2048)]))
    a = ti.rows(rows, M, "A", complex_=cplx)
    Cm = ti.matrix(M, N, "C", complex_=cplx)
    ridx = torch.from_numpy(rows).cuda()
    assert np.array_equal(A[ridx].cpu().numpy(), a), "device A rows differ from the host generator"
    assert np.array_equal(Cd.cpu().numpy(), Cm)
    ref, bound = oracle.tsmm(a, Cm)
    got = O[ridx].cpu().numpy()
    r, wi, _ = oracle.max_err_ratio(got, ref, bound)
    assert r <= TOL["tsmm"], (f"tsmm {dt} {M}x{N} K={K} plan {plan.describe(K)}: "
                              f"max err/bound {r:.3e} at row {rows[wi // N]}")
    return r


@pytest.mark.parametrize("op,dt,M,N,K", ENTRIES, ids=[f"{o}-{d}-{m}x{n}-K{k}" for o, d, m, n, k in ENTRIES])
def test_tuned_plan_full_size(tsm, bufs, op, dt, M, N, K):
    cplx = dt == "z"
    if op == "tsmttsm":
        _tsmttsm(tsm, bufs, M, N, K, cplx)
    else:
        _tsmm(tsm, bufs, M, N, K, cplx)
