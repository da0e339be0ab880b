#!/usr/bin/env python3
"""Small-K study in the paper's metric (Fig. "red_perf";
SURVEY.md §8(f) N3): TSMTTSM time with the fixed-order grid reduction
relative to the same plan WITHOUT the global reduction
(TSM_FLAG_NO_GRID_REDUCE: blocks write their partials only), for K from 10^4
to 10^8, plus the % of the roofline min(b_read * I, P_fp64) and, for
reference, a pure read of the same bytes (libtsm's read probe).
CUDA events, L2 flushed before every rep, median of --reps.
usage: smallk.py [--widths 4,8,32,64] [--Ks 1e4,...] [--json out.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1905_03136_b200 import binding as tsm  # noqa: E402

P_FP64 = 148 * 64 * 2 * 1.965e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", default="4,8,32,64")
    ap.add_argument("--Ks", default="1e4,3e4,1e5,3e5,1e6,3e6,1e7,1e8")
    ap.add_argument("--dtype", default="d")
    ap.add_argument("--reps", type=int, default=21)
    ap.add_argument("--json", default="")
    ap.add_argument("--flush", default="write", choices=["write", "read", "none"],
                    help="L2 flush before every rep: write 512 MB (leaves dirty lines that the timed "
                         "call must write back), read 512 MB (clean), or none")
    a = ap.parse_args()
    widths = [int(w) for w in a.widths.split(",")]
    Ks = [int(float(k)) for k in a.Ks.split(",")]
    z = a.dtype == "z"
    tdt = torch.complex128 if z else torch.float64
    s_ = 16 if z else 8
    Kmax, wmax = max(Ks), max(widths)
    Abuf = torch.empty(Kmax * wmax, dtype=tdt, device="cuda")
    Bbuf = torch.empty(Kmax * wmax, dtype=tdt, device="cuda")
    tsm.fill(Abuf, "A", 42)
    tsm.fill(Bbuf, "B", 42)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    s_ptr = torch.cuda.current_stream().cuda_stream

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(a.reps):
            if a.flush == "write":
                tsm.tsm_l2_flush(flush.data_ptr(), flush.numel(), s_ptr)
            elif a.flush == "read":
                tsm.probe("read", flush.data_ptr(), flush.numel(), 1, s_ptr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        ts.sort()
        return ts[len(ts) // 2]

    # read-only bandwidth at full size for the roofline
    big = Abuf.view(torch.uint8)
    nb = min(big.numel(), 4 << 30)
    bw = max(tsm.probe("read", big.data_ptr(), nb, 1, s_ptr) / timeit(
        lambda: tsm.probe("read", big.data_ptr(), nb, 1, s_ptr)) for _ in range(2))
    rows = []
    for M in widths:
        pl = tsm.Plan("tsmttsm", a.dtype, M, M, 0)
        nr = tsm.Plan("tsmttsm", a.dtype, M, M, 0, no_grid_reduce=True)
        f = tsm.tsmttsm_z if z else tsm.tsmttsm_d
        C = torch.empty(M, M, dtype=tdt, device="cuda")
        for K in Ks:
            A = Abuf[: K * M]
            B = Bbuf[: K * M]
            byts = s_ * (2 * K * M + M * M)
            t_red = timeit(lambda: f(pl.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(),
                                     ws.numel(), s_ptr))
            t_nor = timeit(lambda: f(nr.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(),
                                     ws.numel(), s_ptr))
            nrd = min(byts // 16 * 16, Abuf.numel() * s_)  # same bytes as the call (clamped to Abuf)
            t_rd = timeit(lambda: tsm.probe("read", Abuf.data_ptr(), nrd, 1, s_ptr))
            flops = (8 if z else 2) * M * M * K
            roof = max(byts / bw, flops / P_FP64)
            row = dict(M=M, N=M, K=K, dtype=a.dtype, us=t_red * 1e6, us_no_reduction=t_nor * 1e6,
                       reduction_overhead=t_red / t_nor - 1, pct_roof=100 * roof / t_red,
                       pct_roof_no_reduction=100 * roof / t_nor, us_read_probe=t_rd * 1e6,
                       plan=pl.describe(K))
            rows.append(row)
            print(f"D M=N={M:2d} K={K:>9d}: {t_red*1e6:9.1f} us  no-red {t_nor*1e6:9.1f} us  "
                  f"overhead {100*row['reduction_overhead']:6.1f}%  roof {row['pct_roof']:5.1f}%  "
                  f"grid {row['plan']['grid']} nfin {row['plan']['nfin']}", flush=True)
    if a.json:
        json.dump({"read_gbs": bw / 1e9, "flush": a.flush, "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
