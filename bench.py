#!/usr/bin/env python3
"""libtsm benchmark (driver contract).

Workload (BASELINE.json metric "TSMTTSM/TSMM % of roofline and GB/s, M=N 1..64,
K>=2^24, D/Z"; configs[1]): one STEP = the whole hot path over the width sweep
    for M in 1..64:  C_M  = A_M^T B_M      (tsmttsm, K = 2^24 rows)
    for M in 1..64:  B'_M = A_M C_M        (tsmm)
with A_M / B_M the leading K x M block of two 2^24 x 64 device buffers filled
by libtsm's counter-based generator (synthetic, seed 42).  Every kernel reads
>= 268 MB (> 126 MB L2) and consecutive kernels' reuse window is long evicted,
so no L2 flush is needed between steps (config["l2"]).

value = algorithmic bytes of the step (sum over kernels of 8*(K*M + K*N + M*N)
for D) / device time of the step -> GB/s, whole job (sum over ranks).
With --gpus N > 1 (torchrun), every rank holds its own K = 2^24 row shard
(weak scaling): tsmttsm ends in an NCCL allreduce of C, tsmm starts with an
NCCL broadcast of C.  ``--impl reference`` times the CPU oracle instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TSMTTSM/TSMM % of roofline and GB/s, M=N 1..64, K>=2^24, D/Z, at 1/2/4/8 B200"
K_FULL = 1 << 24
P_FP64_NOMINAL = 148 * 64 * 2 * 1.965e9  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return d["hbm_gbs"] * 1e9, "measured"
    except Exception:
        return 6.65e12, "fallback"


def bench_config(args, widths, world):
    """The workload description shared by the libtsm arm and the reference arm."""
    z = args.dtype == "z"
    return {"workload": f"configs[1] sweep: {'Z' if z else 'D'} M=N {widths[0]}..{widths[-1]}, "
                        "tsmttsm then tsmm per step",
            "K_per_gpu": args.K, "widths": f"{widths[0]}..{widths[-1]}",
            "l2": "inputs > L2 (>=268 MB per kernel), no flush",
            "parallelism": f"K-sharded x{world}" if world > 1 else "single GPU",
            "collectives": ("fused peer-memory reduction (tsmttsm_peer)" if getattr(args, "peer", False)
                            else "allgather+rank-order sum" if args.deterministic else "nccl allreduce")
                           + " of C, nccl broadcast of C" if world > 1 else "none"}


def sizes(op, M, N, K, z):
    s = 16 if z else 8
    byts = s * (K * M + K * N + M * N)
    flops = (8 if z else 2) * M * N * K
    return byts, flops


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        def reader():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 3:
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                    except ValueError:
                        pass
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        loaded = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        mask = 0
        for s in loaded:
            mask |= s[2]
        return {"sm_mhz": statistics.median(s[0] for s in loaded),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": [n for b, n in REASONS.items() if mask & b and b != 0x1],
                "samples": len(loaded)}


# ----------------------------------------------------------------------------
# reference arm / cpu baseline: the CPU oracle as it stands
# ----------------------------------------------------------------------------
def oracle_sample(widths, K, dtype):
    """Time the oracle on the same sweep at K rows (compute only)."""
    import numpy as np

    import oracle
    import tsminputs as ti
    z = dtype == "z"
    maxw = max(widths)
    Abig = ti.matrix(K, maxw, "A", complex_=z)  # columns sliced per width below
    Bbig = ti.matrix(K, maxw, "B", complex_=z)
    total_bytes = 0
    t_total = 0.0
    Cs = {}
    for M in widths:
        A = np.ascontiguousarray(Abig[:, :M])
        B = np.ascontiguousarray(Bbig[:, :M])
        t0 = time.perf_counter()
        C, _ = oracle.tsmttsm(A, B)
        t_total += time.perf_counter() - t0
        Cs[M] = C
        total_bytes += sizes("tsmttsm", M, M, K, z)[0]
    for M in widths:
        A = np.ascontiguousarray(Abig[:, :M])
        t0 = time.perf_counter()
        oracle.tsmm(A, Cs[M])
        t_total += time.perf_counter() - t0
        total_bytes += sizes("tsmm", M, M, K, z)[0]
    return total_bytes, t_total, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    widths = list(range(1, 65))
    K = args.ref_k
    for _ in range(args.warmup):
        oracle_sample(widths, K, args.dtype)
    tb, tt = 0, 0.0
    cores = 1
    for _ in range(args.steps):
        b, t, cores = oracle_sample(widths, K, args.dtype)
        tb += b
        tt += t
    v = tb / tt / 1e9
    sample = f"full M=N 1..64 sweep of tsmttsm+tsmm at K={K} rows (K=2^24/{K_FULL // K}), per step"
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": bench_config(args, widths, world),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libtsm", choices=["libtsm", "reference"])
    ap.add_argument("--dtype", default="d", choices=["d", "z"])
    ap.add_argument("--K", type=int, default=K_FULL)
    ap.add_argument("--widths", default="1-64")
    ap.add_argument("--ref-k", type=int, default=1 << 19)
    ap.add_argument("--cpu-k", type=int, default=1 << 20)
    ap.add_argument("--e2e-widths", default="1,8,16,32")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--peer", action="store_true",
                    help="N>1: TSMTTSM with the grid reduction fused with the cross-GPU sum over "
                         "peer memory (NEXT N3, tsmttsm_peer_*) instead of tsmttsm + NCCL allreduce")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL process group + libtsm comm path even with one rank")
    ap.add_argument("--report", default="", help="write the per-kernel table (JSON) here")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        args.gpus = world
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1905_03136_b200 import binding as tsm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = world > 1 or args.force_comm
    if dist_on:
        if "RANK" not in os.environ:  # single process without torchrun (--force-comm)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        dist.init_process_group("nccl", device_id=dev)
        comm = tsm.Comm(rank, world, local, deterministic=args.deterministic)
    else:
        comm = None
    peer = tsm.PeerComm(rank, world, local) if (dist_on and args.peer) else None

    if "-" in args.widths:
        lo, hi = map(int, args.widths.split("-"))
        widths = list(range(lo, hi + 1))
    else:
        widths = [int(w) for w in args.widths.split(",")]
    z = args.dtype == "z"
    tdt = torch.complex128 if z else torch.float64
    K = args.K
    maxw = max(widths)
    hbm, peak_src = peaks()

    Abuf = torch.empty(K * maxw, dtype=tdt, device=dev)
    Bbuf = torch.empty(K * maxw, dtype=tdt, device=dev)
    Obuf = torch.empty(K * maxw, dtype=tdt, device=dev)
    # rank r holds rows [r*K, (r+1)*K) of the global (world*K) x 64 matrices:
    # generator offset r*K*64 (x2 complex) -- weak scaling, K rows per GPU
    seed = 42
    off = rank * K * maxw * (2 if z else 1)
    tsm.fill(Abuf, "A", seed, start=off)
    tsm.fill(Bbuf, "B", seed, start=off)
    Cs = {M: torch.empty(M, M, dtype=tdt, device=dev) for M in widths}
    plans = {(op, M): tsm.get_plan(op, args.dtype, M, M, local) for op in ("tsmttsm", "tsmm")
             for M in widths}
    stream = torch.cuda.current_stream(dev)
    s_ptr = stream.cuda_stream
    # one workspace big enough for every tsmttsm plan (+ deterministic gather)
    ws_need = max(p.workspace_bytes(K) for (op, _), p in plans.items() if op == "tsmttsm")
    ws_need += 4096 + (world * 64 * 64 * 2 * 8 if comm else 0)
    ws = torch.zeros(ws_need, dtype=torch.uint8, device=dev)

    kern = []  # (op, M) in launch order
    for M in widths:
        kern.append(("tsmttsm", M))
    for M in widths:
        kern.append(("tsmm", M))

    def launch(op, M):
        A = Abuf[: K * M].view(K, M)
        p = plans[(op, M)]
        if op == "tsmttsm":
            B = Bbuf[: K * M].view(K, M)
            C = Cs[M]
            if peer is not None:  # fused grid + cross-GPU reduction (NEXT N3)
                f = tsm.lib.tsmttsm_peer_z if z else tsm.lib.tsmttsm_peer_d
                tsm.check(f(p.handle, peer.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                            ws.data_ptr(), ws.numel(), s_ptr), "tsmttsm_peer")
            elif comm is None:
                f = tsm.tsmttsm_z if z else tsm.tsmttsm_d
                f(p.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel(), s_ptr)
            else:
                f = tsm.lib.tsmttsm_allreduce_z if z else tsm.lib.tsmttsm_allreduce_d
                tsm.check(f(p.handle, comm.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                            ws.data_ptr(), ws.numel(), s_ptr), "tsmttsm_allreduce")
        else:
            C = Cs[M]
            O = Obuf[: K * M].view(K, M)
            if comm is None:
                f = tsm.tsmm_z if z else tsm.tsmm_d
                f(p.handle, K, A.data_ptr(), C.data_ptr(), O.data_ptr(), s_ptr)
            else:
                f = tsm.lib.tsmm_bcast_z if z else tsm.lib.tsmm_bcast_d
                tsm.check(f(p.handle, comm.handle, 0, K, A.data_ptr(), C.data_ptr(), O.data_ptr(),
                            s_ptr), "tsmm_bcast")

    def step(evs=None):
        for i, (op, M) in enumerate(kern):
            if evs is not None:
                evs[i][0].record(stream)
            launch(op, M)
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in kern] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in range(args.steps):
        step(evs[s])
    t1.record(stream)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    if dist_on:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps

    # per-kernel table from the in-region events
    rows = []
    step_bytes = 0
    roof_sum = 0.0
    for i, (op, M) in enumerate(kern):
        ts = sorted(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps))
        t = ts[len(ts) // 2] * 1e-3
        b, f = sizes(op, M, M, K, z)
        step_bytes += b
        t_hbm, t_fp = b / hbm, f / P_FP64_NOMINAL
        roof = max(t_hbm, t_fp)
        roof_sum += roof
        rows.append({"op": op, "M": M, "N": M, "ms": t * 1e3, "gbs": b / t / 1e9,
                     "gflops": f / t / 1e9, "bound": "hbm" if t_hbm >= t_fp else "fp64",
                     "frac": roof / t, "share": 0.0})
    tot_k = sum(r["ms"] for r in rows)
    for r in rows:
        r["share"] = r["ms"] / tot_k
    dom = max(rows, key=lambda r: r["ms"])
    b, f = sizes(dom["op"], dom["M"], dom["N"], K, z)
    if dom["bound"] == "hbm":
        roofline = {"bound": "hbm", "achieved": b / (dom["ms"] * 1e-3) / 1e9, "peak": hbm / 1e9,
                    "unit": "GB/s", "peak_source": peak_src}
    else:
        roofline = {"bound": "alu", "achieved": f / (dom["ms"] * 1e-3) / 1e12,
                    "peak": P_FP64_NOMINAL / 1e12, "unit": "TFLOP/s",
                    "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz "
                                   "(probe: DFMA 36.9, DMMA 37.2 TFLOP/s, profiles/r01_probe.txt)"}
    roofline["frac"] = roofline["achieved"] / roofline["peak"]
    roofline["kernel"] = f"{dom['op']}_{args.dtype} M=N={dom['M']}"
    roofline["share_of_step"] = dom["share"]
    roofline["traffic"] = None
    tr_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_file):
        try:
            roofline["traffic"] = json.load(open(tr_file)).get(roofline["kernel"])
        except Exception:
            pass

    value = step_bytes * world / (ms_step * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(args, widths, world),
            "roofline": roofline,
            "roofline_step": {"frac": roof_sum / (tot_k * 1e-3),
                              "min_frac": min(r["frac"] for r in rows),
                              "note": "sum of per-kernel roofline times / sum of kernel times"},
            "gpu_launches": len(kern) * args.steps, "clocks": clk}

    # ---------------- e2e through host buffers (rank 0 section, every rank runs) -------------
    if not args.no_e2e:
        e2w = [int(w) for w in args.e2e_widths.split(",") if int(w) in widths]
        mw = max(e2w)
        hA = torch.empty(K * mw, dtype=tdt, pin_memory=True)
        hB = torch.empty(K * mw, dtype=tdt, pin_memory=True)
        hO = torch.empty(K * mw, dtype=tdt, pin_memory=True)
        hC = {M: torch.empty(M, M, dtype=tdt, pin_memory=True) for M in e2w}
        hA.copy_(Abuf[: K * mw])
        hB.copy_(Bbuf[: K * mw])
        torch.cuda.synchronize()
        h2d = d2h = e2e_bytes = 0
        for M in e2w:
            h2d += 2 * K * M * hA.element_size()
            d2h += (K * M + M * M) * hA.element_size()
            e2e_bytes += sizes("tsmttsm", M, M, K, z)[0] + sizes("tsmm", M, M, K, z)[0]

        # PCIe is full duplex: width i+1's H2D (s_in) overlaps width i's kernels
        # (compute stream) and width i-1's D2H (s_out); device buffers are
        # double-buffered (two halves of the K x 64 buffers) with events
        # guarding reuse.
        s_in = torch.cuda.Stream(dev)
        s_out = torch.cuda.Stream(dev)
        half = K * (maxw // 2) if 2 * mw <= maxw else 0
        nbuf = 2 if half else 1

        def e2e_step():
            ev_in, ev_comp, ev_out = {}, {}, {}
            s_in.wait_stream(stream)  # previous step's kernels are done with the buffers
            s_out.wait_stream(stream)
            for i, M in enumerate(e2w):
                off = (i % nbuf) * half
                dA = Abuf[off: off + K * M].view(K, M)
                dB = Bbuf[off: off + K * M].view(K, M)
                dO = Obuf[off: off + K * M].view(K, M)
                with torch.cuda.stream(s_in):
                    if i >= nbuf:  # the kernels of width i-nbuf have finished reading this buffer
                        s_in.wait_event(ev_comp[i - nbuf])
                    dA.copy_(hA[: K * M].view(K, M), non_blocking=True)
                    dB.copy_(hB[: K * M].view(K, M), non_blocking=True)
                    ev_in[i] = torch.cuda.Event()
                    ev_in[i].record(s_in)
                stream.wait_event(ev_in[i])
                if i >= nbuf:  # D2H of width i-nbuf has read this buffer of Obuf
                    stream.wait_event(ev_out[i - nbuf])
                C = tsm.tsmttsm(dA, dB, out=Cs[M], plan=plans[("tsmttsm", M)]) if comm is None \
                    else tsm.tsmttsm_allreduce(comm, dA, dB, out=Cs[M])
                O = tsm.tsmm(dA, C, out=dO, plan=plans[("tsmm", M)])
                ev_comp[i] = torch.cuda.Event()
                ev_comp[i].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_comp[i])
                    hC[M].copy_(C, non_blocking=True)
                    hO[: K * M].view(K, M).copy_(O, non_blocking=True)
                    ev_out[i] = torch.cuda.Event()
                    ev_out[i].record(s_out)
            stream.wait_stream(s_in)
            stream.wait_stream(s_out)

        e2e_step()
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.e2e_steps
        if dist_on:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        line["e2e"] = {"value": e2e_bytes * world / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "widths": e2w, "ms_per_step": e_ms,
                       "note": "pinned host A,B -> device, tsmttsm + tsmm via the public API, "
                               "C and B' -> pinned host; H2D / kernels / D2H of consecutive "
                               "widths overlap on three streams (PCIe full duplex); bytes "
                               "counted as the kernels' algorithmic bytes (same metric as value)"}
        del hA, hB, hO

    # ---------------- cpu baseline (rank 0, N=1 only) ----------------
    if rank == 0 and world == 1 and not args.no_cpu:
        tb, tt, cores = oracle_sample(widths, args.cpu_k, args.dtype)
        line["cpu_baseline"] = {"value": tb / tt / 1e9, "unit": "GB/s", "cores": cores,
                                "kind": "oracle",
                                "sample": f"same sweep at K={args.cpu_k} rows (1/{K // args.cpu_k} "
                                          f"of each matrix), compute time only ({tt:.1f} s)"}
    if args.report and rank == 0:
        json.dump({"line": line, "kernels": rows}, open(args.report, "w"), indent=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
