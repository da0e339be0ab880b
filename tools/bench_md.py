#!/usr/bin/env python3
"""Render a bench.py --report JSON as the per-shape markdown table committed
under profiles/ (every kernel of the timed D sweep, the Z sweep, the
non-square shapes and configs[0]; fractions against the in-run denominators).
usage: bench_md.py report.json out.md"""
import json
import sys


def table(rows, title):
    out = [f"## {title}", "", "| op | dtype | M | N | K | ms | GB/s | GFLOP/s | bound | % roofline | "
           "% exec. roofline | SM MHz after | % at that clock | tile work | % of executed | kernel |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        fe = r.get("frac_exec")
        mz, fk = r.get("sm_mhz_after"), r.get("frac_at_kernel_clock")
        tw, fx = r.get("tile_work"), r.get("frac_of_executed")
        out.append(f"| {r['op']} | {r['dtype'].upper()} | {r['M']} | {r['N']} | 2^{int(r['K']).bit_length() - 1} "
                   f"| {r['ms']:.3f} | {r['gbs']:.0f} | {r['gflops']:.0f} | {r['bound']} | {100 * r['frac']:.1f} | "
                   f"{'' if fe is None else f'{100 * fe:.1f}'} | {'' if mz is None else f'{mz:.0f}'} | "
                   f"{'' if fk is None else f'{100 * fk:.1f}'} | {'' if tw is None else f'{tw:.3f}'} | "
                   f"{'' if fx is None else f'{100 * fx:.1f}'} | {r['kernel']} |")
    return out


def bands(rows):
    out = ["| op | dtype | 1-8 | 9-16 | 17-32 | 33-48 | 49-64 | mean | min |", "|---|---|---|---|---|---|---|---|---|"]
    by = {}
    for r in rows:
        by.setdefault((r["op"], r["dtype"]), []).append(r)
    for (op, dt), rs in sorted(by.items()):
        cells = []
        for lo, hi in ((1, 8), (9, 16), (17, 32), (33, 48), (49, 64)):
            v = [r.get("frac_exec", r["frac"]) for r in rs if lo <= r["M"] <= hi]
            cells.append(f"{100 * min(v):.0f} / {100 * sum(v) / len(v):.0f}" if v else "")
        allv = [r.get("frac_exec", r["frac"]) for r in rs]
        out.append(f"| {op} | {dt.upper()} | " + " | ".join(cells) +
                   f" | {100 * sum(allv) / len(allv):.1f} | {100 * min(allv):.1f} |")
    return out


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    d = json.load(open(rep))
    line, k = d["line"], d["kernels"]
    pk = line.get("peaks", {})
    hdr = [f"# bench.py per-kernel table ({rep.split('/')[-1]})", "",
           f"value {line['value']:.0f} GB/s, step {line['ms_per_step']:.1f} ms, roofline_step "
           f"{line['roofline_step']['frac']:.3f} (mean {line['roofline_step']['mean_frac']:.3f}, min "
           f"{line['roofline_step']['min_frac']:.3f}); clocks {line.get('clocks')}",
           f"denominators (in-run): read {pk.get('read_gbs', 0):.0f} GB/s, copy {pk.get('copy_gbs', 0):.0f} GB/s, "
           f"FP64 {pk.get('fp64_tflops', 0):.2f} TFLOP/s ({pk.get('fp64_source')}; DMMA probe "
           f"{pk.get('dmma_tflops', 0):.2f}, at the median clock {pk.get('fp64_at_clock_tflops', 0):.2f})", "",
           "% roofline = min(b * I, P_fp64) time / measured time (b: read-only bandwidth for tsmttsm, copy for "
           "tsmm); % exec. roofline: 3M kernels against their executed 6 flops per complex MAC (DESIGN.md R12). "
           "Per-kernel times are the median over the timed steps of back-to-back kernels (no flush between "
           "kernels; configs[0] flushed). 'SM MHz after': the clock a 1-thread probe measured right after the "
           "kernel in an untimed pass of the same sequence; '% at that clock': the roofline with the FP64 peak "
           "at that clock; 'tile work': multiply-adds executed per useful one (8 x 8 DMMA blocks / 4-deep k-steps, "
           "padding included; bench.py tile_work); '% of executed': the roofline at that clock with the executed "
           "work -- how close the kernel runs to what its tiling allows.", "", "band minimum / mean (% of roofline; 3M: executed):", ""]
    allrows = list(k.get("sweep", [])) + list(k.get("z_sweep", []))
    body = bands(allrows) + [""]
    body += table(k.get("sweep", []), "D sweep (headline step)") + [""]
    if k.get("z_sweep"):
        body += table(k["z_sweep"], "Z sweep (sub-result)") + [""]
    if k.get("nonsquare"):
        body += table(k["nonsquare"], "configs[3] non-square, K = 2^25 (sub-result)") + [""]
    if k.get("config0"):
        body += table([k["config0"]], "configs[0] (L2 flushed before every call)") + [""]
    open(dst, "w").write("\n".join(hdr + body) + "\n")
    print("\n".join(hdr[:4] + bands(allrows)))


if __name__ == "__main__":
    main()
