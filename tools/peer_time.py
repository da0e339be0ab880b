#!/usr/bin/env python3
"""Small-K cost of the cross-GPU reduction at world 1 (NEXT N3): TSMTTSM
alone, TSMTTSM + NCCL allreduce of C (tsmttsm_allreduce_*), and the fused
peer-memory reduction (tsmttsm_peer_*), CUDA-event timed per call (median).
At world 1 the collectives move nothing, so the differences are the fixed
costs each path adds (NCCL launch vs. fence + atomic + rank-order pass).
usage: peer_time.py [--Ks 10000,100000,1000000] [--widths 8,32] [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1905_03136_b200 import binding as tsm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Ks", default="10000,100000,1000000,16777216")
    ap.add_argument("--widths", default="8,32,64")
    ap.add_argument("--dtypes", default="d,z")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = tsm.Comm(0, 1, 0)
    peer = tsm.PeerComm(0, 1, 0)
    s = torch.cuda.current_stream()
    rows = []
    for dt in a.dtypes.split(","):
        tdt = torch.complex128 if dt == "z" else torch.float64
        for K in map(int, a.Ks.split(",")):
            for M in map(int, a.widths.split(",")):
                A = torch.empty(K, M, dtype=tdt, device="cuda")
                B = torch.empty(K, M, dtype=tdt, device="cuda")
                tsm.fill(A, "A", 42)
                tsm.fill(B, "B", 42)
                C = torch.empty(M, M, dtype=tdt, device="cuda")
                fns = {"local": lambda: tsm.tsmttsm(A, B, out=C),
                       "nccl_allreduce": lambda: tsm.tsmttsm_allreduce(comm, A, B, out=C),
                       "fused_peer": lambda: tsm.tsmttsm_peer(peer, A, B, out=C)}
                row = dict(dtype=dt, K=K, M=M)
                for name, fn in fns.items():
                    for _ in range(3):
                        fn()
                    ts = []
                    for _ in range(a.reps):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        torch.cuda._sleep(20000)  # queue the launch behind a busy GPU (host overhead hidden)
                        e0.record(s)
                        fn()
                        e1.record(s)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    ts.sort()
                    row[name + "_us"] = ts[len(ts) // 2]
                assert peer.error() == 0
                rows.append(row)
                print(json.dumps(row), flush=True)
                del A, B
    comm.close()
    peer.close()
    dist.destroy_process_group()
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
