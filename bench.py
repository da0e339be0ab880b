#!/usr/bin/env python3
"""libtsm benchmark (driver contract).

Headline (BASELINE.json metric "TSMTTSM/TSMM % of roofline and GB/s, M=N 1..64,
K>=2^24, D/Z"; configs[1]): one STEP = the whole hot path over the width sweep
    for M in 1..64:  C_M  = A_M^T B_M      (tsmttsm, K = 2^24 rows)
    for M in 1..64:  B'_M = A_M C_M        (tsmm)
with A_M / B_M the leading K x M block of device buffers filled by libtsm's
counter-based generator (synthetic, seed 42).  Every kernel reads >= 268 MB
(> 126 MB L2), so no L2 flush is needed between kernels (config["l2"]).

value = algorithmic bytes of the step (sum over kernels of s*(K*M + K*N + M*N))
/ device time of the step -> GB/s, whole job (sum over ranks).  With --gpus
N > 1 (torchrun) every rank holds its own K = 2^24 row shard (weak scaling):
tsmttsm ends in an NCCL allreduce of C, tsmm starts with an NCCL broadcast.

Measured in the same run and added to the one JSON line:
  * roofline denominators: read-only and copy HBM bandwidth and the FP64
    (DMMA) peak from libtsm's probes; the FP64 peak used is the smaller of the
    probe and 148 SM x 64 FMA x 2 x the median SM clock under load (the
    sustained clock, not boost);
  * per-kernel % of min(b_s * I, P_fp64) (b_s read-only for tsmttsm, copy
    for tsmm) -> mean and MINIMUM over shapes;
  * sub-results (N = 1): the Z sweep (configs[2] extended to 64; paper-flop
    and executed-flop fractions for the 3M kernels), the configs[3]
    non-square shapes at K = 2^25, configs[0] (TSMTTSM D 8x8, K = 10^6, L2
    flushed before every call), and configs[4] (M=N=32, K = 2^28 in total:
    T_1 for D, per-shard sizes K/p for D and Z);
  * e2e: the same D sweep through the public API from pinned host buffers.
``--impl reference`` times the CPU oracle instead (bounded sample).
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
K_NONSQ = 1 << 25
K_CFG4 = 1 << 28
NONSQ = [(1, 64), (64, 1), (16, 48), (48, 16)]
SMS = 148
FMA_PER_CLK_SM = 64  # FP64 FMA / clock / SM (DFMA or DMMA)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_peaks_file():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return d.get("hbm_gbs")
    except Exception:
        return None


def bench_config(args, widths, world):
    """The workload description shared by the libtsm arm and the reference arm."""
    z = args.dtype == "z"
    return {"workload": f"configs[1] sweep: {'Z' if z else 'D'} M=N {widths[0]}..{widths[-1]}, "
                        "tsmttsm then tsmm per step",
            "K_per_gpu": args.K, "widths": f"{widths[0]}..{widths[-1]}",
            "l2": "inputs > L2 (>=268 MB per kernel), no flush between kernels; one L2 drain (a read of "
                  "2 x L2 of clean memory) at the end of each step, timed inside the step",
            "parallelism": f"K-sharded x{world}" if world > 1 else "single GPU",
            "collectives": ("fused peer-memory reduction (tsmttsm_peer)" if getattr(args, "peer", False)
                            else "allgather+rank-order sum" if args.deterministic else "nccl allreduce")
                           + " of C, nccl broadcast of C" if world > 1 else "none"}


def sizes(op, M, N, K, z):
    """Algorithmic bytes and paper flops of one call."""
    s = 16 if z else 8
    byts = s * (K * M + K * N + M * N)
    flops = (8 if z else 2) * M * N * K
    return byts, flops


def parse_widths(spec):
    if "-" in spec:
        lo, hi = map(int, spec.split("-"))
        return list(range(lo, hi + 1))
    return [int(w) for w in spec.split(",")]


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self

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
        return self

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


def dtype_label(z):
    return "c128 (f64 complex)" if z else "f64"


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    widths = parse_widths(args.widths)
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
    sample = (f"full M=N {widths[0]}..{widths[-1]} sweep of tsmttsm+tsmm at K={K} rows per step "
              f"(1/{K_FULL // K} of the workload's K={args.K}; GB/s counts the sample's own bytes)")
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(args.dtype == "z"),
            "data": "synthetic", "impl": "reference",
            "config": bench_config(args, widths, world),
            "sample": {"K_timed": K, "K_workload": args.K, "fraction": K / args.K},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
class Ctx:
    """Per-process state shared by the timed sections."""

    def __init__(self, args, rank, world, local):
        import torch
        import torch.distributed as dist

        from paper_1905_03136_b200 import binding as tsm
        self.torch, self.dist, self.tsm = torch, dist, tsm
        self.args, self.rank, self.world, self.local = args, rank, world, local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.dist_on = world > 1 or args.force_comm
        if self.dist_on:
            if "RANK" not in os.environ:  # single process without torchrun (--force-comm)
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29517")
                os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
            dist.init_process_group("nccl", device_id=self.dev)
            self.comm = tsm.Comm(rank, world, local, deterministic=args.deterministic)
        else:
            self.comm = None
        self.peer = tsm.PeerComm(rank, world, local) if (self.dist_on and args.peer) else None
        self.stream = torch.cuda.current_stream(self.dev)
        self.s_ptr = self.stream.cuda_stream
        self.ws = torch.zeros(1 << 20, dtype=torch.uint8, device=self.dev)
        self.plans = {}
        self.peaks = None

    # -- helpers ---------------------------------------------------------------
    def plan(self, op, dt, M, N):
        key = (op, dt, M, N)
        p = self.plans.get(key)
        if p is None:
            p = self.tsm.get_plan(op, dt, M, N, self.local)
            self.plans[key] = p
        return p

    def need_ws(self, nbytes):
        if self.ws.numel() < nbytes:
            self.ws = self.torch.zeros(nbytes + (1 << 20), dtype=self.torch.uint8, device=self.dev)

    def barrier(self):
        if self.dist_on:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if not self.dist_on:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def view(self, raw, z, rows, cols):
        """rows x cols float64/complex128 view of the leading bytes of a raw buffer."""
        t = raw.view(self.torch.complex128 if z else self.torch.float64)
        return t[: rows * cols].view(rows, cols)

    def fill(self, raw, z, mat, n_elems, start_elem=0):
        t = raw.view(self.torch.complex128 if z else self.torch.float64)[:n_elems]
        self.tsm.fill(t, mat, 42, "fp", start=start_elem * (2 if z else 1))

    # -- one call through the C ABI (collectives when a communicator exists) ----
    def launch(self, op, z, M, N, K, A, B, C, use_comm=True):
        p = self.plan(op, "z" if z else "d", M, N)
        tsm, s = self.tsm, self.s_ptr
        comm = self.comm if use_comm else None
        peer = self.peer if use_comm else None
        if op == "tsmttsm":
            if peer is not None:  # fused grid + cross-GPU reduction (NEXT N3)
                f = tsm.lib.tsmttsm_peer_z if z else tsm.lib.tsmttsm_peer_d
                tsm.check(f(p.handle, peer.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                            self.ws.data_ptr(), self.ws.numel(), s), "tsmttsm_peer")
            elif comm is None:
                f = tsm.tsmttsm_z if z else tsm.tsmttsm_d
                f(p.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), self.ws.data_ptr(), self.ws.numel(), s)
            else:
                f = tsm.lib.tsmttsm_allreduce_z if z else tsm.lib.tsmttsm_allreduce_d
                tsm.check(f(p.handle, comm.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                            self.ws.data_ptr(), self.ws.numel(), s), "tsmttsm_allreduce")
        else:  # B = A C  (here: A, C in; B out)
            if comm is None:
                f = tsm.tsmm_z if z else tsm.tsmm_d
                f(p.handle, K, A.data_ptr(), C.data_ptr(), B.data_ptr(), s)
            else:
                f = tsm.lib.tsmm_bcast_z if z else tsm.lib.tsmm_bcast_d
                tsm.check(f(p.handle, comm.handle, 0, K, A.data_ptr(), C.data_ptr(), B.data_ptr(), s),
                          "tsmm_bcast")

    def ws_for(self, items):
        need = 4096
        for (op, z, M, N, K) in items:
            if op == "tsmttsm":
                p = self.plan(op, "z" if z else "d", M, N)
                need = max(need, p.workspace_bytes(K) + 4096 + (self.world * 64 * 64 * 16 if self.comm else 0))
        self.need_ws(need)

    # -- timing ------------------------------------------------------------------
    def timed(self, calls, steps, warmup, flush=None):
        """calls: list of zero-argument callables (one kernel launch each, maybe
        followed by its collective).  W untimed warm-up passes, then `steps`
        timed passes bracketed by barrier + synchronize, events around every
        call on the launching stream.  Returns (per-call median ms, step ms
        (max over ranks), per-step totals)."""
        torch = self.torch
        for _ in range(max(3, warmup)):
            for c in calls:
                if flush:
                    flush()
                c()
        torch.cuda.synchronize()
        evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in calls] for _ in range(steps)]
        self.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(self.stream)
        for s in range(steps):
            for i, c in enumerate(calls):
                if flush:
                    flush()
                evs[s][i][0].record(self.stream)
                c()
                evs[s][i][1].record(self.stream)
        t1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        per = []
        for i in range(len(calls)):
            ts = sorted(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(steps))
            per.append(ts[len(ts) // 2])
        total = t0.elapsed_time(t1) / steps
        if flush:  # flush kernels are inside the bracket: report the sum of the calls
            total = sum(sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for i in range(len(calls)))
                        for s in range(steps)) / steps
        return per, self.max_over_ranks(total)

    # -- roofline denominators ---------------------------------------------------
    def measure_peaks(self, raw):
        torch, tsm = self.torch, self.tsm
        nbytes = min(raw.numel(), 4 << 30)

        def best(kind, iters=1, reps=8):
            ts, work = [], 0.0
            for r in range(reps + 2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                work = tsm.probe(kind, raw.data_ptr(), nbytes, iters, self.s_ptr)
                e1.record(self.stream)
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            return work / min(ts), work / statistics.median(ts)

        read_best, read_med = best("read")
        copy_best, copy_med = best("copy")
        dmma_best, dmma_med = best("dmma", iters=20000, reps=4)
        return {"read_gbs": read_best / 1e9, "copy_gbs": copy_best / 1e9, "dmma_tflops": dmma_best / 1e12,
                "fp64_tflops": dmma_best / 1e12, "fp64_source": "probe",
                "read_gbs_median": read_med / 1e9, "copy_gbs_median": copy_med / 1e9,
                "dmma_tflops_median": dmma_med / 1e12,
                "how": "libtsm tsm_probe, in this run: read-only and copy over 4 GiB (best of 8), "
                       "DMMA m8n8k4 chains 8 blocks x 4 warps per SM (best of 4)"}

    def set_fp64_peak(self, sm_mhz):
        """P_fp64 = min(probe, 148 SM x 64 FMA x 2 x median SM clock under load)."""
        pk = self.peaks
        probe = pk["dmma_tflops"] * 1e12
        if sm_mhz:
            at_clock = SMS * FMA_PER_CLK_SM * 2 * sm_mhz * 1e6
            pk["fp64_at_clock_tflops"] = at_clock / 1e12
            pk["fp64_sm_mhz"] = sm_mhz
            pk["fp64_tflops"] = min(probe, at_clock) / 1e12
            pk["fp64_source"] = ("clock" if at_clock < probe else "probe")
        else:
            pk["fp64_tflops"] = probe / 1e12
            pk["fp64_source"] = "probe"

    def row(self, op, z, M, N, K, ms, kname="", mhz=None):
        """Per-kernel roofline row: % of min(b_s * I, P_fp64)."""
        pk = self.peaks
        b, f = sizes(op, M, N, K, z)
        t = ms * 1e-3
        bw = (pk["read_gbs"] if op == "tsmttsm" else pk["copy_gbs"]) * 1e9
        P = pk["fp64_tflops"] * 1e12
        t_hbm, t_fp = b / bw, f / P
        roof = max(t_hbm, t_fp)
        r = {"op": op, "dtype": "z" if z else "d", "M": M, "N": N, "K": K, "ms": ms, "gbs": b / t / 1e9,
             "gflops": f / t / 1e9, "bound": "hbm" if t_hbm >= t_fp else "fp64", "frac": roof / t,
             "kernel": kname}
        if mhz:  # the FP64 roof at the clock measured right after this kernel (sweep rows)
            Pk = min(pk["dmma_tflops"] * 1e12, SMS * FMA_PER_CLK_SM * 2 * mhz * 1e6)
            fexec = f * (0.75 if (z and "3m" in kname) else 1.0)
            r["frac_at_kernel_clock"] = max(t_hbm, fexec / Pk) / t
            r["sm_mhz_after"] = mhz
            # the same roofline with the work the kernel executes (tile padding
            # included): how close the kernel runs to what its tiling allows
            tw = tile_work(op, M, N, z, kname)
            r["tile_work"] = tw
            r["frac_of_executed"] = max(t_hbm, tw * fexec / Pk) / t
        if z and "3m" in kname:  # 3M / Gauss: 6 executed real flops per complex MAC (R12)
            r["frac_exec"] = max(t_hbm, 0.75 * t_fp) / t
            r["bound_exec"] = "hbm" if t_hbm >= 0.75 * t_fp else "fp64"
        return r


def tile_work(op, M, N, z, kname):
    """Multiply-adds the kernel executes per row, padding included, over the
    useful M*N (the 'tile ceiling' of DESIGN.md §5b: DMMA works on 8 x 8 blocks
    of C (TSMTTSM) / 4-deep k-steps x 8-column blocks (TSMM); the DFMA edge
    cells are useful work on the same FP64 pipe).  1.0 for the DFMA kernels."""
    if "dmma" not in kname:
        return 1.0
    if "complex-as-real" in kname:
        M, N = 2 * M, 2 * N  # the real kernel on the interleaved view (4 real MACs per complex one)
    cd = lambda a, b: -(-a // b)  # noqa: E731
    if op == "tsmttsm":
        MC, NC = 8 * (M // 8), 8 * (N // 8)
        if "l-blocks" in kname:
            er, ec = M - MC, N - NC
            nl = max(cd(MC, 8 - er), cd(NC, 8 - ec))
            work = 64 * ((MC // 8) * (NC // 8) + nl)
        elif "edge" in kname:  # DFMA edge warps / inline edge: the edge cells unpadded
            work = MC * NC + (M * N - MC * NC)
        else:
            work = 64 * cd(M, 8) * cd(N, 8)
    else:
        ec = N % 8 if "edge-columns" in kname else 0
        work = 4 * cd(M, 4) * 8 * cd(N - ec, 8) + M * ec
    return work / (M * N)


def summarize(rows):
    fr = [r.get("frac_exec", r["frac"]) for r in rows]
    fp = [r["frac"] for r in rows]
    worst = min(rows, key=lambda r: r.get("frac_exec", r["frac"]))
    fc = [r["frac_at_kernel_clock"] for r in rows if "frac_at_kernel_clock" in r]
    fe = [r["frac_of_executed"] for r in rows if "frac_of_executed" in r]
    extra = {"mean_frac_at_kernel_clock": sum(fc) / len(fc), "min_frac_at_kernel_clock": min(fc),
             "mean_frac_of_executed": sum(fe) / len(fe), "min_frac_of_executed": min(fe),
             "sm_mhz_after_kernels_min": min(r["sm_mhz_after"] for r in rows if "sm_mhz_after" in r)} if fc else {}
    return {**extra, "shapes": len(rows), "mean_frac": sum(fr) / len(fr), "min_frac": min(fr),
            "n_ge_90": sum(1 for x in fr if x >= 0.9),
            "mean_frac_paper_flops": sum(fp) / len(fp), "min_frac_paper_flops": min(fp),
            "worst": f"{worst['op']}_{worst['dtype']} {worst['M']}x{worst['N']} K={worst['K']} "
                     f"({worst.get('frac_exec', worst['frac']):.3f})",
            "note": "frac = roofline time / measured time; for 3M Z kernels the roofline of the executed "
                    "6-flop algorithm (frac_paper_flops counts the paper's 8, DESIGN.md R3/R12)"}


def sweep(ctx, raw, z, widths, K, steps, warmup):
    """The configs[1]/[2] sweep: tsmttsm for every width, then tsmm."""
    A, B, O = raw
    n = K * max(widths)
    ctx.fill(A, z, "A", n, ctx.rank * n)
    ctx.fill(B, z, "B", n, ctx.rank * n)
    dt = "z" if z else "d"
    Cs = {M: ctx.torch.empty(M, M, dtype=ctx.torch.complex128 if z else ctx.torch.float64, device=ctx.dev)
          for M in widths}
    items = [("tsmttsm", z, M, M, K) for M in widths] + [("tsmm", z, M, M, K) for M in widths]
    ctx.ws_for(items)
    calls = []
    for (op, _, M, N, _) in items:
        a = ctx.view(A, z, K, M)
        if op == "tsmttsm":
            calls.append(lambda a=a, M=M: ctx.launch("tsmttsm", z, M, M, K, a, ctx.view(B, z, K, M), Cs[M]))
        else:
            calls.append(lambda a=a, M=M: ctx.launch("tsmm", z, M, M, K, a, ctx.view(O, z, K, M), Cs[M]))
    # L2 drain at the end of the step (timed inside the step, not a kernel row):
    # the last TSMM leaves ~L2-size of dirty B lines, whose write-back the next
    # step's first TSMTTSMs would otherwise pay (order probe run 23: TSMTTSM D 1 /
    # 2 / 4 take 6-16 us longer right after TSMM D 64 than after a clean L2).
    # A read of 2 x L2 of clean memory (the tail of the A buffer, which the first
    # kernels of the next step do not read) absorbs it, so each kernel row
    # carries its own cost; the step time still includes it.
    l2 = ctx.torch.cuda.get_device_properties(ctx.dev).L2_cache_size
    nb = ((2 * l2) // 4096) * 4096
    drain_ptr = A.data_ptr() + A.numel() - nb
    assert A.numel() - nb >= K * min(widths) * (16 if z else 8) * 4, "drain overlaps the first kernels' inputs"
    calls.append(lambda: ctx.tsm.probe("read", drain_ptr, nb, 1, ctx.s_ptr))
    per, step_ms = ctx.timed(calls, steps, warmup)
    drain_ms = per.pop()
    calls.pop()
    # untimed pass: the SM clock right after every kernel of the step (a 1-thread
    # probe counting cycles over 2 us of globaltimer) -- the clock the FP64-bound
    # kernels actually ran at under the power cap
    for _ in range(2):
        clk = ctx.torch.zeros(2 * len(calls), dtype=ctx.torch.float64, device=ctx.dev)
        for i, c in enumerate(calls):
            c()
            ctx.tsm.probe("clock", clk[2 * i:].data_ptr(), 16, 2000, ctx.s_ptr)
        ctx.torch.cuda.synchronize()
    mhzs = clk[0::2].cpu().tolist()
    rows = [ctx.row(op, z, M, N, K, ms, ctx.plan(op, dt, M, N).describe(K).get("kernel", ""), mhz)
            for (op, _, M, N, _), ms, mhz in zip(items, per, mhzs)]
    byts = sum(sizes(op, M, N, K, z)[0] for (op, _, M, N, _) in items)
    ctx.l2_drain_ms = drain_ms
    return rows, step_ms, byts, Cs


def nonsquare(ctx, raw, steps, warmup):
    A, B, O = raw
    K = K_NONSQ
    rows = []
    for z in (False, True):
        n = K * 64
        ctx.fill(A, z, "A", n)
        ctx.fill(B, z, "B", n)
        items = [(op, z, M, N, K) for op in ("tsmttsm", "tsmm") for (M, N) in NONSQ]
        ctx.ws_for(items)
        calls = []
        Cs = {}
        for (op, _, M, N, _) in items:
            C = Cs.setdefault((M, N), ctx.torch.empty(M, N, dtype=ctx.torch.complex128 if z else ctx.torch.float64,
                                                      device=ctx.dev))
            a = ctx.view(A, z, K, M)
            if op == "tsmttsm":
                calls.append(lambda a=a, M=M, N=N, C=C: ctx.launch("tsmttsm", z, M, N, K, a, ctx.view(B, z, K, N), C,
                                                                   use_comm=False))
            else:
                calls.append(lambda a=a, M=M, N=N, C=C: ctx.launch("tsmm", z, M, N, K, a, ctx.view(O, z, K, N), C,
                                                                   use_comm=False))
        per, _ = ctx.timed(calls, steps, warmup)
        dt = "z" if z else "d"
        rows += [ctx.row(op, z, M, N, K, ms, ctx.plan(op, dt, M, N).describe(K).get("kernel", ""))
                 for (op, _, M, N, _), ms in zip(items, per)]
    return rows


def config0(ctx, raw, reps):
    """configs[0]: TSMTTSM D M=N=8, K=10^6 (128 MB, about the L2 size): the L2
    is flushed before every timed call, two ways:
      * "clean" (the row's ms / frac): write 2 x L2 of scratch, then read its
        first L2 bytes, so L2 ends up full of CLEAN lines that hold none of
        the kernel's inputs;
      * "dirty" (ms_dirty_flush / frac_dirty_flush): the 2 x L2 write only.
        The timed call then also pays the write-back of ~L2 bytes of the
        flush kernel's dirty lines as its reads evict them -- a cost of the
        flush, not of the TSMTTSM (libtsm's read probe over the same 128 MB
        shows the same ~15 us, profiles/r02_smallk_run3.md)."""
    A, B, O = raw
    K, M = 10 ** 6, 8
    ctx.fill(A, False, "A", K * M)
    ctx.fill(B, False, "B", K * M)
    C = ctx.torch.empty(M, M, dtype=ctx.torch.float64, device=ctx.dev)
    ctx.ws_for([("tsmttsm", False, M, M, K)])
    l2 = ctx.torch.cuda.get_device_properties(ctx.dev).L2_cache_size
    scratch = O.view(ctx.torch.float64)[: 2 * l2 // 8]

    def flush_dirty():
        ctx.tsm.tsm_l2_flush(scratch.data_ptr(), scratch.numel() * 8, ctx.s_ptr)

    def flush_clean():
        flush_dirty()
        ctx.tsm.probe("read", scratch.data_ptr(), (l2 // 4096) * 4096, 1, ctx.s_ptr)
    calls = [lambda: ctx.launch("tsmttsm", False, M, M, K, ctx.view(A, False, K, M), ctx.view(B, False, K, M), C,
                                use_comm=False)]
    kname = ctx.plan("tsmttsm", "d", M, M).describe(K).get("kernel", "")
    per, _ = ctx.timed(calls, reps, 3, flush=flush_clean)
    r = ctx.row("tsmttsm", False, M, M, K, per[0], kname)
    per_d, _ = ctx.timed(calls, reps, 3, flush=flush_dirty)
    rd = ctx.row("tsmttsm", False, M, M, K, per_d[0], kname)
    r["ms_dirty_flush"], r["frac_dirty_flush"] = rd["ms"], rd["frac"]
    # the floor of one cold launch over these bytes: libtsm's read-only probe
    # over 128 MB (the bytes of A and B) after the same clean flush
    nb = 2 * K * M * 8
    per_p, _ = ctx.timed([lambda: ctx.tsm.probe("read", A.data_ptr(), nb, 1, ctx.s_ptr)], reps, 3,
                         flush=flush_clean)
    r["read_probe_ms"] = per_p[0]
    r["frac_of_read_probe"] = per_p[0] / r["ms"]
    r["l2"] = "flushed before every call: 2 x L2 write + 1 x L2 read (clean lines); *_dirty_flush: write only"
    return r


def configs4(ctx, steps, warmup, sizes_list):
    """configs[4]: M=N=32, K = 2^28 rows in total, K-sharded over the ranks.
    A step = tsmttsm (+ sum of C over ranks) then tsmm (+ broadcast of C); the
    tsmm output goes to a 2^25-row scratch in pieces (the full K x 32 output
    does not fit next to A and B: 3 x 68.7 GB), every row computed and
    written once.  Returns one entry per (dtype, K_local)."""
    torch = ctx.torch
    M = 32
    out = []
    piece = 1 << 25
    maxK = max(K for (_, K) in sizes_list)
    maxbytes = max(K * M * (16 if z else 8) for (z, K) in sizes_list)
    A = torch.empty(maxbytes, dtype=torch.uint8, device=ctx.dev)
    B = torch.empty(maxbytes, dtype=torch.uint8, device=ctx.dev)
    O = torch.empty(min(maxK, piece) * M * 16, dtype=torch.uint8, device=ctx.dev)
    for (z, K) in sizes_list:
        start = ctx.rank * K * M  # this rank's rows of the global matrices
        ctx.fill(A, z, "A", K * M, start)
        ctx.fill(B, z, "B", K * M, start)
        C = torch.empty(M, M, dtype=torch.complex128 if z else torch.float64, device=ctx.dev)
        ctx.ws_for([("tsmttsm", z, M, M, K)])
        a, b = ctx.view(A, z, K, M), ctx.view(B, z, K, M)
        s = 16 if z else 8

        def tsmm_pieces(a=a, K=K, z=z, C=C):
            for k0 in range(0, K, piece):
                k = min(piece, K - k0)
                ctx.launch("tsmm", z, M, M, k, a[k0:k0 + k], ctx.view(O, z, k, M), C)
        entry = {"dtype": "z" if z else "d", "M": M, "N": M, "K_local": K, "K_total": K * ctx.world,
                 "ranks": ctx.world}
        for label, use_comm in (("", True), ("_local", False)):
            if use_comm is False and ctx.world == 1:
                continue
            calls = [lambda a=a, b=b, C=C, K=K, z=z, u=use_comm: ctx.launch("tsmttsm", z, M, M, K, a, b, C, use_comm=u)]
            if use_comm:
                calls.append(tsmm_pieces)
            else:
                calls.append(lambda a=a, K=K, z=z, C=C: [ctx.launch("tsmm", z, M, M, min(piece, K - k0),
                                                                    a[k0:k0 + min(piece, K - k0)],
                                                                    ctx.view(O, z, min(piece, K - k0), M), C,
                                                                    use_comm=False)
                                                         for k0 in range(0, K, piece)])
            per, step_ms = ctx.timed(calls, steps, warmup)
            entry["ms_step" + label] = step_ms
            entry["ms_tsmttsm" + label] = per[0]
            entry["ms_tsmm" + label] = per[1]
        byts = sizes("tsmttsm", M, M, K, z)[0] + sizes("tsmm", M, M, K, z)[0]
        entry["gbs_per_gpu"] = byts / (entry["ms_step"] * 1e-3) / 1e9
        entry["tsmm_launches"] = (K + piece - 1) // piece
        entry["bytes_per_gpu"] = byts
        _ = s
        out.append(entry)
    del A, B, O
    torch.cuda.empty_cache()
    return out


def e2e(ctx, raw, widths, K, z, steps):
    """The headline sweep through the public API from pinned host buffers:
    per width, H2D of A and B, tsmttsm (+allreduce) and tsmm, D2H of C and B'.
    PCIe is full duplex: width i+1's H2D (s_in) overlaps width i's kernels and
    width i-1's D2H (s_out); device buffers are double-buffered (two halves)."""
    torch, tsm = ctx.torch, ctx.tsm
    A, B, O = raw
    tdt = torch.complex128 if z else torch.float64
    mw = max(widths)
    Ad = A.view(tdt)
    Bd = B.view(tdt)
    Od = O.view(tdt)
    hA = torch.empty(K * mw, dtype=tdt, pin_memory=True)
    hB = torch.empty(K * mw, dtype=tdt, pin_memory=True)
    hO = torch.empty(K * mw, dtype=tdt, pin_memory=True)
    hC = {M: torch.empty(M, M, dtype=tdt, pin_memory=True) for M in widths}
    n = K * mw
    ctx.fill(A, z, "A", n, ctx.rank * n)
    ctx.fill(B, z, "B", n, ctx.rank * n)
    hA.copy_(Ad[:n])
    hB.copy_(Bd[:n])
    torch.cuda.synchronize()
    h2d = d2h = e2e_bytes = 0
    es = hA.element_size()
    for M in widths:
        h2d += 2 * K * M * es
        d2h += (K * M + M * M) * es
        e2e_bytes += sizes("tsmttsm", M, M, K, z)[0] + sizes("tsmm", M, M, K, z)[0]
    Cs = {M: torch.empty(M, M, dtype=tdt, device=ctx.dev) for M in widths}
    s_in = torch.cuda.Stream(ctx.dev)
    s_out = torch.cuda.Stream(ctx.dev)
    stream = ctx.stream
    half = Ad.numel() // 2  # two device halves, each >= K * mw elements
    assert half >= K * mw

    def step():
        ev_in, ev_comp, ev_out = {}, {}, {}
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        for i, M in enumerate(widths):
            off = (i % 2) * half
            dA = Ad[off: off + K * M].view(K, M)
            dB = Bd[off: off + K * M].view(K, M)
            dO = Od[off: off + K * M].view(K, M)
            with torch.cuda.stream(s_in):
                if i >= 2:  # the kernels of width i-2 have finished reading this half
                    s_in.wait_event(ev_comp[i - 2])
                dA.copy_(hA[: K * M].view(K, M), non_blocking=True)
                dB.copy_(hB[: K * M].view(K, M), non_blocking=True)
                ev_in[i] = torch.cuda.Event()
                ev_in[i].record(s_in)
            stream.wait_event(ev_in[i])
            if i >= 2:  # the D2H of width i-2 has read this half of O
                stream.wait_event(ev_out[i - 2])
            C = tsm.tsmttsm(dA, dB, out=Cs[M], plan=ctx.plan("tsmttsm", "z" if z else "d", M, M)) \
                if ctx.comm is None else tsm.tsmttsm_allreduce(ctx.comm, dA, dB, out=Cs[M])
            Ob = tsm.tsmm(dA, C, out=dO, plan=ctx.plan("tsmm", "z" if z else "d", M, M))
            ev_comp[i] = torch.cuda.Event()
            ev_comp[i].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[i])
                hC[M].copy_(C, non_blocking=True)
                hO[: K * M].view(K, M).copy_(Ob, non_blocking=True)
                ev_out[i] = torch.cuda.Event()
                ev_out[i].record(s_out)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)

    step()
    torch.cuda.synchronize()
    ctx.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = ctx.max_over_ranks(e0.elapsed_time(e1) / steps)
    del hA, hB, hO
    return {"value": e2e_bytes * ctx.world / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "widths": f"{widths[0]}..{widths[-1]}", "ms_per_step": e_ms, "steps": steps,
            "note": "pinned host A,B -> device, tsmttsm + tsmm via the public API, C and B' -> pinned "
                    "host, every width of the headline sweep; H2D / kernels / D2H of consecutive widths "
                    "overlap on three streams (PCIe full duplex); bytes counted as the kernels' "
                    "algorithmic bytes (same metric as value)"}


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
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-results (Z sweep, configs[0,3,4])")
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--peer", action="store_true",
                    help="N>1: TSMTTSM with the grid reduction fused with the cross-GPU sum over "
                         "peer memory (NEXT N3, tsmttsm_peer_*) instead of tsmttsm + NCCL allreduce")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL process group + libtsm comm path even with one rank")
    ap.add_argument("--report", default="", help="write the per-kernel tables (JSON) here")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        args.gpus = world
    if args.impl == "reference":
        return run_reference(args, rank, world)

    ctx = Ctx(args, rank, world, local)
    torch = ctx.torch
    widths = parse_widths(args.widths)
    z = args.dtype == "z"
    K = args.K
    sub = not args.no_sub and world == 1 and K == K_FULL
    # raw buffers shared by the sweeps and configs[0]/[3]: 3 x (K x 64 complex), or
    # 3 x (2^25 x 64 complex) when the non-square shapes run (103 GB)
    # (e2e double-buffers: two halves of K x max(widths))
    elems = max(K * max(widths) * (2 if z else 1) * (1 if args.no_e2e else 2),
                (K_NONSQ * 64 * 2) if sub else 0, (K * max(widths) * 2) if sub else 0)
    raw = [torch.empty(elems * 8, dtype=torch.uint8, device=ctx.dev) for _ in range(3)]

    ctx.peaks = ctx.measure_peaks(raw[0])
    allclk = ClockSampler(local).start()

    # ---------------- headline: the configs[1] sweep ----------------
    clocks = ClockSampler(local).start()
    time.sleep(0.3)
    rows, ms_step, step_bytes, _ = sweep(ctx, raw, z, widths, K, args.steps, args.warmup)
    clk = clocks.stop()
    ctx.set_fp64_peak(clk.get("sm_mhz"))
    # rows were computed before the clock was known: recompute with the final peak
    rows = [ctx.row(r["op"], z, r["M"], r["N"], r["K"], r["ms"], r["kernel"], r.get("sm_mhz_after")) for r in rows]
    tot_k = sum(r["ms"] for r in rows)
    for r in rows:
        r["share"] = r["ms"] / tot_k
    dom = max(rows, key=lambda r: r["ms"])
    b, f = sizes(dom["op"], dom["M"], dom["N"], K, z)
    pk = ctx.peaks
    if dom["bound"] == "hbm":
        bw = pk["read_gbs"] if dom["op"] == "tsmttsm" else pk["copy_gbs"]
        roofline = {"bound": "hbm", "achieved": b / (dom["ms"] * 1e-3) / 1e9, "peak": bw, "unit": "GB/s",
                    "peak_source": f"in-run probe ({'read-only' if dom['op'] == 'tsmttsm' else 'copy'})"}
    else:
        fexec = f * (0.75 if "3m" in dom["kernel"] else 1.0)
        # DMMA (mma.sync m8n8k4 f64) is the FP64 tensor-core contraction: the
        # peak is its own dtype's, the in-run DMMA probe at the timed clock
        roofline = {"bound": "tensor", "achieved": fexec / (dom["ms"] * 1e-3) / 1e12, "peak": pk["fp64_tflops"],
                    "unit": "TFLOP/s",
                    "peak_source": (f"FP64 (DMMA) peak = min(in-run probe {pk['dmma_tflops']:.2f} TFLOP/s, "
                                    f"148 SM x 64 FMA/clk x 2 x {pk.get('fp64_sm_mhz')} MHz median SM clock "
                                    f"in the timed region = {pk.get('fp64_at_clock_tflops', 0):.2f}) -> "
                                    f"{pk['fp64_source']}")}
    roofline["frac"] = roofline["achieved"] / roofline["peak"]
    # context: the executed work of that kernel's tiling (8 x 8 DMMA blocks,
    # bench.tile_work) and its fraction of that work's roofline at its own clock
    if "tile_work" in dom:
        roofline["tile_work"] = dom["tile_work"]
        roofline["frac_of_executed_at_kernel_clock"] = dom["frac_of_executed"]
    roofline["kernel"] = f"{dom['op']}_{args.dtype} M=N={dom['M']} ({dom['kernel']})"
    roofline["share_of_step"] = dom["share"]
    roofline["traffic"] = None
    tr_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_file):
        try:
            roofline["traffic"] = json.load(open(tr_file)).get(f"{dom['op']}_{args.dtype} M=N={dom['M']}")
        except Exception:
            pass

    value = step_bytes * world / (ms_step * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(z),
            "data": "synthetic",
            "config": bench_config(args, widths, world),
            "roofline": roofline,
            "roofline_step": dict(summarize(rows), frac=sum(r["ms"] * r["frac"] for r in rows) / tot_k),
            "peaks": dict(pk, measured_peaks_json_hbm_gbs=measured_peaks_file()),
            "gpu_launches": (len(rows) + 1) * args.steps, "clocks": clk,
            "l2_drain_ms_per_step": getattr(ctx, "l2_drain_ms", None)}
    report = {"sweep": rows}

    # ---------------- sub-results (single GPU) ----------------
    subs = {}
    if sub:
        if not z:
            # (as many steps as the headline: the first kernel of the first timed step
            # follows the host-side sync and runs on a ramping clock; the median drops it)
            zrows, zms, zbytes, _ = sweep(ctx, raw, True, widths, K, max(3, args.steps), args.warmup)
            report["z_sweep"] = zrows
            subs["z_sweep"] = dict(summarize(zrows), ms_per_step=zms,
                                   gbs=zbytes / (zms * 1e-3) / 1e9, K=K)
        nrows = nonsquare(ctx, raw, args.steps, args.warmup)
        report["nonsquare"] = nrows
        subs["configs3_nonsquare"] = dict(summarize(nrows), shapes_list=[f"{r['op']}_{r['dtype']} {r['M']}x{r['N']}: "
                                                                         f"{r.get('frac_exec', r['frac']):.3f}"
                                                                         for r in nrows])
        c0 = config0(ctx, raw, 20)
        report["config0"] = c0
        subs["configs0"] = {k: c0[k] for k in ("ms", "gbs", "frac", "bound", "kernel", "l2", "ms_dirty_flush",
                                                 "frac_dirty_flush", "read_probe_ms", "frac_of_read_probe")}
    if args.report and rank == 0:
        json.dump({"line": line, "kernels": report}, open(args.report, "w"), indent=1)

    # ---------------- e2e through host buffers ----------------
    if not args.no_e2e:
        line["e2e"] = e2e(ctx, raw, widths, K, z, args.e2e_steps)

    # ---------------- configs[4]: M=N=32, K = 2^28 in total ----------------
    if not args.no_sub and K == K_FULL:
        del raw
        torch.cuda.empty_cache()
        if world == 1:  # T_1 (D, all of K) and the per-shard sizes K/p, p = 2, 4, 8
            todo = [(False, K_CFG4)] + [(zz, K_CFG4 // p) for p in (2, 4, 8) for zz in (False, True)]
        else:
            todo = [(False, K_CFG4 // world), (True, K_CFG4 // world)]
        c4 = configs4(ctx, args.steps, args.warmup, todo)
        subs["configs4"] = {"entries": c4,
                            "note": "M=N=32, K=2^28 rows in total, K-sharded; step = tsmttsm (+sum of C over ranks) "
                                    "+ tsmm (+broadcast of C), tsmm output in 2^25-row pieces.  At N=1: T_1 for D "
                                    "(all 2^28 rows on one GPU) and the per-shard sizes K/p (Z at 2^28 = 275 GB does "
                                    "not fit one GPU).  At N>1 ms_step includes the collectives, ms_step_local is "
                                    "the same shard without them.  E_p(D, strong) = T_1(2^28) / (p * T_p); "
                                    "per shard E_p = T_1(2^28/p) / T_p (SURVEY.md §8(e))."}
    if subs:
        line["sub_results"] = subs
    line["clocks_all_sections"] = allclk.stop()

    # ---------------- cpu baseline (rank 0, N=1 only) ----------------
    if rank == 0 and world == 1 and not args.no_cpu:
        tb, tt, cores = oracle_sample(widths, args.cpu_k, args.dtype)
        line["cpu_baseline"] = {"value": tb / tt / 1e9, "unit": "GB/s", "cores": cores,
                                "kind": "oracle", "cpu_model": cpu_model(),
                                "sample": f"same sweep at K={args.cpu_k} rows (1/{K // args.cpu_k} "
                                          f"of each matrix), compute time only ({tt:.1f} s)"}
    if args.report and rank == 0:
        json.dump({"line": line, "kernels": report}, open(args.report, "w"), indent=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ctx.comm is not None:
        ctx.comm.close()
        ctx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
