#!/usr/bin/env python3
"""On-B200 autotuner for libtsm (the paper's exhaustive configuration search,
PAPER.md:748-749, 1021-1024, re-done on the target GPU).

For every requested (op, dtype, M, N):
  1. enumerate compile-time candidates (tools/gen_instances.candidates),
  2. JIT-compile them in parallel through tsm_plan_create_config (NVRTC,
     the same templates as the AOT build),
  3. time each with CUDA events at K rows (L2 flushed before every rep),
  4. re-time the best few over run-time parameters (pipeline stages, CTAs/SM),
  5. record the winner in tune/b200.json; tools/gen_instances.py then
     instantiates the winners ahead of time.
usage: autotune.py --ops tsmttsm,tsmm --dtypes d,z --widths 1-64 [--shapes 16x48,...]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import gen_instances as gi  # noqa: E402
from paper_1905_03136_b200 import binding as tsm  # noqa: E402

P_FP64 = 148 * 64 * 2 * 1.965e9


def parse_shapes(a):
    if a.shapes:
        return [tuple(map(int, s.split("x"))) for s in a.shapes.split(",")]
    if "-" in a.widths:
        lo, hi = map(int, a.widths.split("-"))
        return [(w, w) for w in range(lo, hi + 1)]
    return [(int(w), int(w)) for w in a.widths.split(",")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="tsmttsm,tsmm")
    ap.add_argument("--dtypes", default="d,z")
    ap.add_argument("--widths", default="1-64")
    ap.add_argument("--shapes", default="")
    ap.add_argument("--K", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--jobs", type=int, default=min(32, os.cpu_count() or 8))
    ap.add_argument("--out", default=os.path.join(ROOT, "tune", "b200.json"))
    ap.add_argument("--time-budget", type=float, default=0, help="stop after this many seconds")
    ap.add_argument("--filter", default="", help="python expression on a candidate dict c, e.g. "
                    "\"c.get('PAIR')\" -- only matching candidates are timed")
    ap.add_argument("--heat", type=int, default=0,
                    help="time every rep right after N launches of a heater (TSMM D 64 at K=2^22, about 1.1 ms "
                         "each) and a clean L2 flush, with no host sync in between: the power-capped SM clock "
                         "of bench.py's back-to-back sweep instead of the cool-GPU clock (HBM-bound kernels "
                         "whose SM side has no headroom lose 8-15 %% there, profiles/r02_order_run18.md)")
    ap.add_argument("--keep-better", action="store_true",
                    help="keep the stored entry when it is faster than this run's best")
    a = ap.parse_args()
    t_start = time.time()
    shapes = parse_shapes(a)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6.65e12
    db = {"entries": {}}
    if os.path.exists(a.out):
        db = json.load(open(a.out))
    db["gpu"] = torch.cuda.get_device_name(0)
    db["K"] = a.K
    K = a.K
    maxw = max(max(s) for s in shapes)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s_ptr = torch.cuda.current_stream().cuda_stream
    pool = cf.ThreadPoolExecutor(a.jobs)
    heat = None
    if a.heat:
        KH = 1 << 22
        hA = torch.empty(KH * 64, dtype=torch.float64, device="cuda")
        hB = torch.empty(KH * 64, dtype=torch.float64, device="cuda")
        hC = torch.empty(64 * 64, dtype=torch.float64, device="cuda")
        tsm.fill(hA, "A", 7)
        tsm.fill(hC, "C", 7)
        hplan = tsm.Plan("tsmm", "d", 64, 64, 0)

        def heat(n):
            for _ in range(n):
                tsm.tsmm_d(hplan.handle, KH, hA.data_ptr(), hC.data_ptr(), hB.data_ptr(), s_ptr)
            # clean L2 (the heater's dirty output lines are written back here, untimed)
            tsm.probe("read", flush.data_ptr(), flush.numel(), 1, s_ptr)
    for dt in a.dtypes.split(","):
        z = dt == "z"
        tdt = torch.complex128 if z else torch.float64
        Abuf = torch.empty(K * maxw, dtype=tdt, device="cuda")
        Bbuf = torch.empty(K * maxw, dtype=tdt, device="cuda")
        tsm.fill(Abuf, "A", 42)
        tsm.fill(Bbuf, "B", 42)
        Cmat = torch.empty(maxw * maxw, dtype=tdt, device="cuda")
        tsm.fill(Cmat, "C", 42)
        ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
        for op in a.ops.split(","):
            for (M, N) in shapes:
                if a.time_budget and time.time() - t_start > a.time_budget:
                    print("time budget reached", flush=True)
                    break
                key = f"{op}_{dt}_{M}_{N}"
                cands = gi.candidates(op, M, N, z)
                if a.filter:
                    cands = [c for c in cands if eval(a.filter, {}, {"c": c})]  # noqa: S307
                    if not cands:
                        continue
                A = Abuf[: K * M].view(K, M)
                if op == "tsmttsm":
                    B = Bbuf[: K * N].view(K, N)
                    O = torch.empty(M, N, dtype=tdt, device="cuda")
                    C = None
                else:
                    C = Cmat[: M * N].view(M, N)
                    O = Bbuf[: K * N].view(K, N)
                byts = (16 if z else 8) * (K * M + K * N + M * N)
                flops = (8 if z else 2) * M * N * K
                roof = max(byts / hbm, flops / P_FP64)

                def make(c, stages=4, ctas=4):
                    try:
                        return tsm.Plan(op, dt, M, N, 0, config=gi.to_tsm_config(op, c, stages, ctas))
                    except Exception as e:  # noqa: BLE001
                        return e

                def run(plan):
                    if op == "tsmttsm":
                        f = tsm.tsmttsm_z if z else tsm.tsmttsm_d
                        f(plan.handle, K, A.data_ptr(), B.data_ptr(), O.data_ptr(), ws.data_ptr(),
                          ws.numel(), s_ptr)
                    else:
                        f = tsm.tsmm_z if z else tsm.tsmm_d
                        f(plan.handle, K, A.data_ptr(), C.data_ptr(), O.data_ptr(), s_ptr)

                def timeit(plan):
                    if plan.workspace_bytes(K) > ws.numel():
                        return float("inf")
                    run(plan)
                    if heat:
                        heat(16)  # pre-roll: into the power-capped state
                        evs = []
                        for _ in range(a.reps):
                            heat(a.heat)
                            e0 = torch.cuda.Event(enable_timing=True)
                            e1 = torch.cuda.Event(enable_timing=True)
                            e0.record()
                            run(plan)
                            e1.record()
                            evs.append((e0, e1))
                        torch.cuda.synchronize()
                        ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
                        return ts[len(ts) // 2]
                    ts = []
                    for _ in range(a.reps):
                        tsm.tsm_l2_flush(flush.data_ptr(), flush.numel(), s_ptr)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        run(plan)
                        e1.record()
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    ts.sort()
                    return ts[len(ts) // 2]

                # the current default plan (tuned table entry), timed in this run
                try:
                    default_ms = timeit(tsm.Plan(op, dt, M, N, 0))
                except Exception:  # noqa: BLE001
                    default_ms = None
                t0 = time.time()
                plans = list(pool.map(make, cands))
                t_comp = time.time() - t0
                res = []
                for c, p in zip(cands, plans):
                    if isinstance(p, Exception):
                        continue
                    res.append((timeit(p), c, p.config()))
                if not res:
                    print(f"{key}: no valid candidate", flush=True)
                    continue
                res.sort(key=lambda r: r[0])
                # phase 2: run-time parameters for the best 3
                best = res[0]
                # (DMMA kernels: both consumer-warp orders, a launch argument)
                dmma = lambda c: c.get("impl", 0) >= 1  # noqa: E731
                for (_, c0, _) in res[:3]:
                    for c in ([c0, dict(c0, PLAIN=1)] if dmma(c0) else [c0]):
                        for stages in (2, 3, 4, 6):
                            for ctas in (1, 2, 3, 4):
                                p = make(c, stages, ctas)
                                if isinstance(p, Exception):
                                    continue
                                got = p.config()
                                if got["stages"] != stages or got["ctas_per_sm"] != ctas:
                                    continue  # clipped: same as another point
                                t = timeit(p)
                                if t < best[0]:
                                    best = (t, c, got)
                t, c, got = best
                cfg = dict(c)
                cfg["stages"] = got["stages"]
                cfg["ctas"] = got["ctas_per_sm"]
                prev = db["entries"].get(key)
                # keep-better: compare with the default plan timed in THIS run (same
                # clocks), else with the stored time
                ref_ms = default_ms if default_ms is not None else (prev["ms"] if prev else None)
                if a.keep_better and prev and ref_ms is not None and ref_ms <= t:
                    print(f"{key}: kept stored (default {ref_ms:.4f} ms this run; best candidate {t:.4f} ms "
                          f"{cfg})", flush=True)
                    continue
                db["entries"][key] = {"cfg": cfg, "ms": t, "frac": roof / (t * 1e-3),
                                      "candidates": len(res), "default_ms": default_ms}
                print(f"{key}: best {t:.4f} ms ({100 * roof / (t * 1e-3):.1f}% roof) "
                      f"{cfg} [{len(res)} cands, compile {t_comp:.1f}s]"
                      + (f" prev {prev['ms']:.4f}" if prev else ""), flush=True)
                os.makedirs(os.path.dirname(a.out), exist_ok=True)
                json.dump(db, open(a.out + ".tmp", "w"), indent=1, sort_keys=True)
                os.replace(a.out + ".tmp", a.out)
        del Abuf, Bbuf
        torch.cuda.empty_cache()
    pool.shutdown()


if __name__ == "__main__":
    main()
