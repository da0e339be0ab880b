#!/usr/bin/env python3
"""Does a short HBM-bound kernel run slower right after a long FP64-heavy one?
(bench.py times the sweep back to back: TSMTTSM M=1 of step s+1 follows TSMM
M=64 of step s.)  Times the light call (a) after an L2 flush only, (b) right
after the heavy call, (c) after the heavy call and a 2 ms host-side pause;
CUDA events around the light call only, median of --reps.
usage: order_probe.py [--dtype z] [--light tsmttsm:1] [--heavy tsmm:64]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1905_03136_b200 import binding as tsm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="z")
    ap.add_argument("--light", default="tsmttsm:1")
    ap.add_argument("--heavy", default="tsmm:64")
    ap.add_argument("--K", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=11)
    a = ap.parse_args()
    z = a.dtype == "z"
    tdt = torch.complex128 if z else torch.float64
    K = a.K
    A = torch.empty(K * 64, dtype=tdt, device="cuda")
    B = torch.empty(K * 64, dtype=tdt, device="cuda")
    O = torch.empty(K * 64, dtype=tdt, device="cuda")
    tsm.fill(A, "A", 42)
    tsm.fill(B, "B", 42)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def call(spec):
        op, w = spec.split(":")
        w = int(w)
        if op == "tsmttsm":
            C = torch.empty(w, w, dtype=tdt, device="cuda")
            return lambda: tsm.tsmttsm(A[: K * w].view(K, w), B[: K * w].view(K, w), out=C)
        C = torch.ones(w, w, dtype=tdt, device="cuda")
        return lambda: tsm.tsmm(A[: K * w].view(K, w), C, out=O[: K * w].view(K, w))

    light, heavy = call(a.light), call(a.heavy)
    light(), heavy()
    torch.cuda.synchronize()

    def timed(pre):
        ts = []
        for _ in range(a.reps):
            pre()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            light()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    def pause_after_heavy():
        heavy()
        torch.cuda.synchronize()
        time.sleep(0.002)

    res = {"after_flush": timed(lambda: tsm.tsm_l2_flush(flush.data_ptr(), flush.numel(), s)),
           "after_heavy": timed(heavy),
           "after_heavy_and_2ms_pause": timed(pause_after_heavy),
           "after_read_flush": timed(lambda: tsm.probe("read", flush.data_ptr(), flush.numel(), 1, s)),
           "after_itself": timed(light)}
    print({k: round(v, 4) for k, v in res.items()}, f"light {a.light} heavy {a.heavy} dtype {a.dtype}")


if __name__ == "__main__":
    main()
