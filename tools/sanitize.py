#!/usr/bin/env python3
"""compute-sanitizer driver (VERDICT r01 missing item 6).

Runs ONE representative launch configuration of every kernel family libtsm
ships -- every distinct kernel variant among the tuned default plans (all
square widths 1..64, D and Z, both ops, plus the non-square configs[3]
shapes), the explicit families of tools/gen_instances.candidates() the tuned
table does not pick, the TSMM update (beta = 1 reduce-add, beta = 2 scale),
the conjugate plans and the TMA strided views -- at K in {1, 2, 33, 4099},
and checks every result against the oracle (so a run under a sanitizer tool
is also a parity run).  Meant to be wrapped:

    compute-sanitizer --tool racecheck  python tools/sanitize.py
    compute-sanitizer --tool synccheck  python tools/sanitize.py
    compute-sanitizer --tool memcheck   python tools/sanitize.py
    compute-sanitizer --tool initcheck  python tools/sanitize.py

Prints one line per family and "SANITIZE_OK <n>" at the end.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import tsminputs as ti  # noqa: E402
from paper_1905_03136_b200 import binding as tsm  # noqa: E402

KS = [1, 2, 33, 4099]


def run_one(plan, op, z, M, N, K, conj=False, update=None, strided=False):
    A = ti.matrix(K, M, "A", complex_=z, seed=K + 11)
    dA = torch.from_numpy(A).cuda()
    if strided:  # a column subset of a wider block vector (ld = width + 8 elements)
        wideA = torch.zeros(K, M + 8, dtype=dA.dtype, device="cuda")
        oa = 3 if z else 2  # column offset: 16-byte aligned base (TMA / bulk copies)
        wideA[:, oa:oa + M] = dA
        dA = wideA[:, oa:oa + M]
    if op == "tsmttsm":
        B = ti.matrix(K, N, "B", complex_=z, seed=K + 12)
        dB = torch.from_numpy(B).cuda()
        if strided:
            wideB = torch.zeros(K, N + 8, dtype=dB.dtype, device="cuda")
            ob = 5 if z else 4
            wideB[:, ob:ob + N] = dB
            dB = wideB[:, ob:ob + N]
        got = tsm.tsmttsm(dA, dB, plan=plan, conj=conj)
        ref, bound = oracle.tsmttsm(A, B, conj=conj)
        tol = 1e-12
    else:
        Cm = ti.matrix(M, N, "C", complex_=z, seed=K + 13)
        dC = torch.from_numpy(Cm).cuda()
        if update is not None:
            B0 = ti.matrix(K, N, "B", complex_=z, seed=K + 14)
            dB = torch.from_numpy(B0).cuda()
            alpha, beta = update
            tsm.tsmm_update(dA, dC, dB, alpha=alpha, beta=beta, plan=plan, conj=conj)
            got = dB
            ref, bound = oracle.tsmm_update(A, Cm, B0, alpha, beta, conj=conj)
            tol = 1e-13 * 4
        else:
            out = None
            if strided:
                wideO = torch.zeros(K, N + 8, dtype=dA.dtype, device="cuda")
                oo = 1 if z else 2
                out = wideO[:, oo:oo + N]
            got = tsm.tsmm(dA, dC, plan=plan, out=out)
            ref, bound = oracle.tsmm(A, Cm)
            tol = 1e-13
    torch.cuda.synchronize()
    r, wi, _ = oracle.max_err_ratio(np.ascontiguousarray(got.cpu().numpy()), ref, bound)
    assert r <= tol, (op, z, M, N, K, r, wi, plan.describe(K))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="first 6 families only")
    ap.add_argument("--match", default="", help="comma list of kernel-name substrings: only those families")
    a = ap.parse_args()
    fams = {}
    shapes = [(w, w) for w in range(1, 65)] + [(1, 64), (64, 1), (16, 48), (48, 16)]
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for (M, N) in shapes:
                p = tsm.get_plan(op, dt, M, N, 0)
                d = p.describe(4099)
                key = (op, dt, d["kernel"], p.config()["kernel"] & 15)
                fams.setdefault(key, ("default", p, M, N))
    # explicit families the tuned table may not pick (autotuner search space);
    # only the first candidate of each (impl, flags) class is compiled
    import gen_instances as gi
    seen = set()
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for (M, N) in [(64, 64), (33, 17), (24, 24), (3, 5), (57, 57), (41, 41)]:
                for c in gi.candidates(op, M, N, dt == "z"):
                    cls = (op, dt, c.get("impl", 0), gi.flags(c) & ~64, c.get("WR", 1) % 2)
                    if cls in seen:
                        continue
                    seen.add(cls)
                    try:
                        p = tsm.Plan(op, dt, M, N, 0, config=gi.to_tsm_config(op, c, 3, 2))
                    except tsm.TsmError:
                        continue
                    key = (op, dt, p.describe(4099)["kernel"], p.config()["kernel"] & 15)
                    fams.setdefault(key, ("explicit", p, M, N))
    items = sorted(fams.items(), key=lambda kv: kv[0])
    if a.match:
        items = [it for it in items if any(m in it[0][2] for m in a.match.split(","))]
    if a.quick:
        items = items[:6]
    n = 0
    for (op, dt, kname, impl), (src, p, M, N) in items:
        z = dt == "z"
        for K in KS:
            run_one(p, op, z, M, N, K)
            n += 1
        print(f"{op:8s} {dt} impl {impl} {kname:55s} {src:8s} M={M} N={N}: ok", flush=True)
    # N1 update (beta = 1: bulk/TMA reduce-add; beta = 2: scale pass first), N2 conj, N4 strided
    extra = [("tsmm", "d", 63, 63), ("tsmm", "d", 64, 64), ("tsmm", "z", 24, 24), ("tsmm", "d", 5, 5)]
    for (op, dt, M, N) in extra:
        p = tsm.get_plan(op, dt, M, N, 0)
        for K in KS:
            run_one(p, op, dt == "z", M, N, K, update=(-1.0, 1.0))
            run_one(p, op, dt == "z", M, N, K, update=(0.5, 2.0))
            n += 2
        print(f"update   {dt} M={M} N={N} ({p.describe(99)['kernel']}): ok", flush=True)
    for (op, M, N) in [("tsmttsm", 32, 32), ("tsmttsm", 17, 17), ("tsmm", 24, 24), ("tsmm", 40, 40)]:
        p = tsm.get_plan(op, "z", M, N, 0, conj=True)
        for K in KS:
            if op == "tsmttsm":
                run_one(p, op, True, M, N, K, conj=True)
            else:
                run_one(p, op, True, M, N, K, update=(1.0, 0.0), conj=True)
            n += 1
        print(f"conj     z {op} M={M} N={N}: ok", flush=True)
    for (op, dt, M, N, g) in [("tsmttsm", "d", 32, 32, False), ("tsmm", "d", 16, 48, False),
                              ("tsmttsm", "z", 8, 8, False), ("tsmm", "z", 40, 40, False),
                              ("tsmttsm", "d", 33, 7, True), ("tsmm", "d", 57, 57, True),
                              ("tsmm", "z", 5, 3, True)]:
        p = tsm.get_plan(op, dt, M, N, 0, strided=not g, gather=g)
        for K in KS:
            run_one(p, op, dt == "z", M, N, K, strided=True)
            n += 1
        print(f"strided  {dt} {op} M={M} N={N}: ok", flush=True)
    print(f"SANITIZE_OK {n} launches, {len(items)} families", flush=True)


if __name__ == "__main__":
    main()
