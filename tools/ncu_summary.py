#!/usr/bin/env python3
"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  ncu_summary.py full <rep.ncu-rep> [--name KEY] [--traffic profiles/ncu_traffic.json]
      key metrics of a `--set full` capture (per launch); with --traffic, also
      records dram read+write bytes per launch under KEY for bench.py's
      roofline.traffic.
  ncu_summary.py launches <launches.csv> [--out profiles/...json]
      per-kernel totals / shares from a `--metrics gpu__time_duration.sum` list.
  ncu_summary.py traffic <rep.ncu-rep> --traffic profiles/ncu_traffic.json
      a `--metrics dram__bytes_read.sum,dram__bytes_write.sum,...` capture over
      many shapes (tools/quick_time.py): dram read+write bytes per launch,
      keyed like bench.py's roofline.kernel ("tsmm_d M=N=58"; median over the
      launches of a shape), parsed from the template arguments in the names.
"""
import re
import argparse
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum" ,
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def full(a):
    hdr, units, rows = raw_rows(a.rep)
    res = []
    for r in rows:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        d["traffic_bytes"] = to_bytes(r[i_r], units[i_r]) + to_bytes(r[i_w], units[i_w])
        res.append(d)
    print(json.dumps(res, indent=1))
    if a.traffic and a.name:
        db = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
        db[a.name] = sum(x["traffic_bytes"] for x in res) / len(res)
        json.dump(db, open(a.traffic, "w"), indent=1, sort_keys=True)


def kernel_key(name: str):
    """bench.py key of a libtsm kernel name (None for other kernels)."""
    m = re.search(r"(tsmttsm|tsmm)\w*<\s*tsm::(\w+)Cfg<([^>]*)>", name) or \
        re.search(r"(tsmttsm|tsmm)\w*<(\w+)Cfg<([^>]*)>", name)
    if not m:
        return None
    op, fam, args = m.group(1), m.group(2), [x.strip() for x in m.group(3).split(",")]
    M, N = int(args[0]), int(args[1])
    z = args[2] in ("1", "true")
    zr = (fam == "TsmttsmMma" and len(args) >= 13 and args[12] in ("1", "true")) or \
         (fam == "TsmmCst" and len(args) >= 8 and args[7] in ("1", "true"))
    if zr:
        M, N, z = M // 2, N // 2, True
    if M != N:
        return f"{op}_{'z' if z else 'd'} M={M},N={N}"
    return f"{op}_{'z' if z else 'd'} M=N={M}"


def traffic(a):
    hdr, units, rows = raw_rows(a.rep)
    ik = hdr.index("Kernel Name")
    i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    per = {}
    for r in rows:
        key = kernel_key(r[ik])
        if key is None:
            continue
        per.setdefault(key, []).append(to_bytes(r[i_r], units[i_r]) + to_bytes(r[i_w], units[i_w]))
    db = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
    for k, v in per.items():
        v.sort()
        db[k] = v[len(v) // 2]
    json.dump(db, open(a.traffic, "w"), indent=1, sort_keys=True)
    print(f"{len(per)} kernels -> {a.traffic}")


def launches(a):
    rows = list(csv.reader(open(a.csv)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = {}
    for r in rows[start + 1:]:
        if len(r) <= iv or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[iu], 1.0)
        name = r[ik].split("(")[0][:120]
        t = tot.setdefault(name, [0, 0.0])
        t[0] += 1
        t[1] += v
    all_us = sum(t[1] for t in tot.values())
    summ = sorted(([n, c, us, us / all_us] for n, (c, us) in tot.items()), key=lambda x: -x[2])
    out = {"total_us": all_us, "kernels": [{"name": n, "launches": c, "us": us, "share": s}
                                           for n, c, us, s in summ]}
    js = json.dumps(out, indent=1)
    if a.out:
        open(a.out, "w").write(js)
    print(js[:3000])


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("full")
    f.add_argument("rep")
    f.add_argument("--name", default="")
    f.add_argument("--traffic", default="")
    t = sub.add_parser("traffic")
    t.add_argument("rep")
    t.add_argument("--traffic", required=True)
    l = sub.add_parser("launches")
    l.add_argument("csv")
    l.add_argument("--out", default="")
    a = ap.parse_args()
    {"full": full, "launches": launches, "traffic": traffic}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
