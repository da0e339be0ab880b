#!/usr/bin/env python3
"""Format tools/quick_time.py --json outputs as the per-shape roofline table
committed under profiles/ (north-star metric: % of min(HBM BW x I, FP64 peak)).

usage: report_md.py out.md in1.json [in2.json ...]
"""
import json
import sys


def main():
    out, ins = sys.argv[1], sys.argv[2:]
    rows = []
    for f in ins:
        rows += json.load(open(f))
    lines = ["| op | dtype | M | N | K | ms | GB/s | GFLOP/s | bound | % roofline | kernel |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        k = r.get("plan", {}).get("kernel", "")
        lines.append(f"| {r['op']} | {r['dtype'].upper()} | {r['M']} | {r['N']} | 2^{r['K'].bit_length() - 1} | "
                     f"{r['ms']:.3f} | {r['gbs']:.0f} | {r['gflops']:.0f} | {r['bound']} | "
                     f"{r['pct_roof']:.1f} | {k} |")
    by = {}
    for r in rows:
        by.setdefault((r["op"], r["dtype"]), []).append(r["pct_roof"])
    summ = ["", "| op | dtype | shapes | min % | mean % | >= 90 % |", "|---|---|---|---|---|---|"]
    for (op, dt), v in sorted(by.items()):
        summ.append(f"| {op} | {dt.upper()} | {len(v)} | {min(v):.1f} | {sum(v) / len(v):.1f} | "
                    f"{sum(1 for x in v if x >= 90)} |")
    note = ["", "% roofline counts the paper's flops (8 real flops per complex multiply-add, DESIGN.md R3); "
            "kernels marked +3m execute 6 (3M / Gauss products, R12), so compute-bound Z shapes can exceed "
            "100 %; for FP64-bound shapes their executed-flop fraction of the FP64 peak is 3/4 of the printed value."]
    open(out, "w").write("\n".join(summ[1:] + note + [""] + lines) + "\n")
    print("\n".join(summ))


if __name__ == "__main__":
    main()
