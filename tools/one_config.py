#!/usr/bin/env python3
"""Time (or run once under ncu) ONE explicit configuration of one shape.
usage: one_config.py OP DT M N 'CFG_JSON' [--K 16777216] [--reps 5]
CFG_JSON is a gen_instances-style dict, e.g. '{"MT":1,"NTL":2,"NT":288,"R":32,"impl":1,
"AP":17,"BP":17,"EDGE":4,"G3":1,"stages":4,"ctas":2}'."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import gen_instances as gi  # noqa: E402
from paper_1905_03136_b200 import binding as tsm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op")
    ap.add_argument("dt")
    ap.add_argument("M", type=int)
    ap.add_argument("N", type=int)
    ap.add_argument("cfg")
    ap.add_argument("--K", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    c = json.loads(a.cfg)
    plan = tsm.Plan(a.op, a.dt, a.M, a.N, 0, config=gi.to_tsm_config(a.op, c, c.get("stages", 3), c.get("ctas", 1)))
    tdt = torch.complex128 if a.dt == "z" else torch.float64
    A = torch.empty(a.K, a.M, dtype=tdt, device="cuda")
    tsm.fill(A, "A", 42)
    if a.op == "tsmttsm":
        B = torch.empty(a.K, a.N, dtype=tdt, device="cuda")
        tsm.fill(B, "B", 42)
        fn = lambda: tsm.tsmttsm(A, B, plan=plan)  # noqa: E731
    else:
        C = torch.empty(a.M, a.N, dtype=tdt, device="cuda")
        tsm.fill(C, "C", 42)
        O = torch.empty(a.K, a.N, dtype=tdt, device="cuda")
        fn = lambda: tsm.tsmm(A, C, out=O, plan=plan)  # noqa: E731
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"op": a.op, "dt": a.dt, "M": a.M, "N": a.N, "ms": ts[len(ts) // 2],
                      "plan": plan.describe(a.K)}))


if __name__ == "__main__":
    main()
