#!/usr/bin/env python3
"""Stall samples of an ncu --set full capture (--import-source on) per CUDA
source line of tsm_kernels.cuh: which lines of the kernel the warps wait on,
and why.  NVRTC kernels name their source "<repo>/tsm_kernels.cuh"; if that
path does not exist here a temporary symlink to the package header is made
for ncu's source resolution (the header must be the one the kernel was built
from).
usage: ncu_lines.py <rep.ncu-rep> [--top 25]"""
import argparse
import csv
import io
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1905_03136_b200", "csrc", "tsm_kernels.cuh")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    link = os.path.join(ROOT, "tsm_kernels.cuh")
    made = False
    if not os.path.exists(link):
        os.symlink(HDR, link)
        made = True
    try:
        out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                             capture_output=True, text=True).stdout
    finally:
        if made:
            os.remove(link)
    rows = list(csv.reader(io.StringIO(out)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    per = {}
    cur = None
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        if r[0]:
            cur = (int(r[0]), r[1].strip())
            per.setdefault(cur, {"samples": 0.0, **{s: 0.0 for s in stalls}})
            continue
        if cur is None:
            continue

        def num(k):
            try:
                return float(r[ix[k]])
            except (ValueError, KeyError):
                return 0.0
        d = per[cur]
        d["samples"] += num("Warp Stall Sampling (All Samples)")
        for s in stalls:
            d[s] += num(s)
    tot = sum(d["samples"] for d in per.values()) or 1.0
    print(f"total samples {tot:.0f}")
    for (ln, src), d in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[: a.top]:
        top = sorted(((d[s], s[6:]) for s in stalls), reverse=True)[:3]
        why = " ".join(f"{n}:{100 * v / max(d['samples'], 1):.0f}%" for v, n in top if v > 0)
        print(f"{100 * d['samples'] / tot:5.1f} %  L{ln:<5d} {src[:70]:70s} {why}")


if __name__ == "__main__":
    main()
