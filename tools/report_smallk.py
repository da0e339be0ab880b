#!/usr/bin/env python3
"""Small-K table: per (op,
dtype, M=N, K) the kernel time, its roofline time, the fixed overhead
t - t_roof (launch ramp, grid reduction, tail) and % of roofline, from
tools/quick_time.py --Ks ... --json.

usage: report_smallk.py out.md in.json
"""
import json
import sys


def main():
    out, inp = sys.argv[1], sys.argv[2]
    rows = json.load(open(inp))
    lines = ["| op | dtype | M=N | K | time µs | roofline µs | overhead µs | % roofline | grid | nfin |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        t = r["ms"] * 1e3
        roof = t * r["pct_roof"] / 100
        pl = r.get("plan", {})
        lines.append(f"| {r['op']} | {r['dtype'].upper()} | {r['M']} | {r['K']:.0e} | {t:.1f} | {roof:.1f} | "
                     f"{t - roof:.1f} | {r['pct_roof']:.1f} | {pl.get('grid', '')} | {pl.get('nfin', '')} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
