#!/usr/bin/env python3
"""Per-kernel timing sweep (CUDA events, L2 flushed before every rep).

Prints one row per (op, dtype, M, N): median kernel time, algorithmic GB/s
and GFLOP/s, and % of the roofline min(BW * I, P_fp64) with BW the measured
HBM copy bandwidth (MEASURED_PEAKS.json) and P_fp64 = 148 SM x 64 FMA x 2 x
1.965 GHz = 37.2 TFLOP/s.
usage: quick_time.py [--ops tsmttsm,tsmm] [--dtypes d,z] [--widths 1,8,32,64] [--K 16777216]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1905_03136_b200 import binding as tsm  # noqa: E402

P_FP64 = 148 * 64 * 2 * 1.965e9


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
    except Exception:
        return 6.65e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="tsmttsm,tsmm")
    ap.add_argument("--dtypes", default="d")
    ap.add_argument("--widths", default="1,2,4,8,16,24,32,40,48,56,64")
    ap.add_argument("--shapes", default="")
    ap.add_argument("--K", type=int, default=1 << 24)
    ap.add_argument("--Ks", default="", help="comma list of K values (small-K study); overrides --K")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json", default="")
    ap.add_argument("--toggle-order", action="store_true",
                    help="time the default plan's configuration with the consumer-warp order flipped "
                         "(kernel ^ 1024, DMMA kernels)")
    a = ap.parse_args()

    def get_plan(op, dt, M, N):
        plan = tsm.get_plan(op, dt, M, N, 0)
        if a.toggle_order and plan.config()["kernel"] & 15:
            cfg = dict(plan.config())
            cfg["kernel"] ^= 1024
            plan = tsm.Plan(op, dt, M, N, 0, config=cfg)
        return plan
    bw = hbm_peak()
    shapes = [tuple(map(int, s.split("x"))) for s in a.shapes.split(",") if s] or \
        [(w, w) for w in map(int, a.widths.split(","))]
    maxw = max(max(s) for s in shapes)
    Ks = [int(float(x)) for x in a.Ks.split(",") if x] or [a.K]
    K = max(Ks)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rows = []
    for dt in a.dtypes.split(","):
        tdt = torch.complex128 if dt == "z" else torch.float64
        sz = 16 if dt == "z" else 8
        Abuf = torch.empty(K * maxw, dtype=tdt, device="cuda")
        Bbuf = torch.empty(K * maxw, dtype=tdt, device="cuda")
        tsm.fill(Abuf, "A", 42)
        tsm.fill(Bbuf, "B", 42)
        for op in a.ops.split(","):
          for K in Ks:
            for (M, N) in shapes:
                A = Abuf[: K * M].view(K, M)
                if op == "tsmttsm":
                    B = Bbuf[: K * N].view(K, N)
                    C = torch.empty(M, N, dtype=tdt, device="cuda")
                    plan = get_plan(op, dt, M, N)
                    fn = lambda: tsm.tsmttsm(A, B, out=C, plan=plan)  # noqa: E731
                    byts = sz * (K * M + K * N + M * N)
                else:
                    Cm = torch.empty(M, N, dtype=tdt, device="cuda")
                    tsm.fill(Cm, "C", 42)
                    B = Bbuf[: K * N].view(K, N)
                    plan = get_plan(op, dt, M, N)
                    fn = lambda: tsm.tsmm(A, Cm, out=B, plan=plan)  # noqa: E731
                    byts = sz * (K * M + K * N + M * N)
                flops = (8 if dt == "z" else 2) * M * N * K
                for _ in range(3):
                    fn()
                ts = []
                for _ in range(a.reps):
                    tsm.tsm_l2_flush(flush.data_ptr(), flush.numel(), s)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                ts.sort()
                t = ts[len(ts) // 2]
                roof_t = max(byts / bw, flops / P_FP64)
                row = dict(op=op, dtype=dt, M=M, N=N, K=K, ms=t * 1e3, gbs=byts / t / 1e9,
                           gflops=flops / t / 1e9, pct_roof=100 * roof_t / t,
                           bound="hbm" if byts / bw >= flops / P_FP64 else "fp64",
                           plan=plan.describe(K))
                rows.append(row)
                print(f"{op:8s} {dt} M={M:2d} N={N:2d} K={K}: {t*1e3:8.3f} ms {row['gbs']:7.0f} GB/s "
                      f"{row['gflops']:8.0f} GF/s  {row['pct_roof']:5.1f}% roof ({row['bound']})",
                      flush=True)
        del Abuf, Bbuf
        torch.cuda.empty_cache()
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
