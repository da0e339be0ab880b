#!/usr/bin/env python3
"""Hot SASS instructions of an ncu --set full capture (--import-source on):
per instruction the stall samples, executed count and shared-memory
wavefronts (ideal vs actual), and the totals per stall reason.
usage: ncu_sass_hot.py <rep.ncu-rep> [--top 40]"""
import argparse
import csv
import io
import subprocess
import collections


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr, data = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}

    def num(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError, IndexError):
            return 0.0
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in data:
        for s in stalls:
            tot[s] += num(r, s)
    S = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"total samples {S:.0f}")
    for s, v in tot.most_common(12):
        print(f"  {s:28s} {100 * v / max(S, 1):5.1f} %")
    wf = sum(num(r, "L1 Wavefronts Shared") for r in data)
    wfi = sum(num(r, "L1 Wavefronts Shared Ideal") for r in data)
    print(f"shared wavefronts {wf:.3e} (ideal {wfi:.3e})")
    print("hot instructions (samples, executed, shared wavefronts / ideal, top stalls):")
    data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
    for r in data[:a.top]:
        top = sorted(((num(r, s), s[6:]) for s in stalls), reverse=True)[:3]
        print(f"{num(r, 'Warp Stall Sampling (All Samples)'):7.0f} {num(r, 'Instructions Executed'):10.0f} "
              f"{num(r, 'L1 Wavefronts Shared'):10.0f}/{num(r, 'L1 Wavefronts Shared Ideal'):<10.0f} "
              f"{r[ix['Source']].strip()[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in top if v))


if __name__ == "__main__":
    main()
