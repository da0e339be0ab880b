#!/usr/bin/env python3
"""SASS opcode summary of the kernels the tuned plans load (the NVRTC cubins
in paper_1905_03136_b200/kcache, the code that runs): per kernel family, the
static count of the instructions that prove the data path -- DMMA (FP64
tensor pipe, mma.sync m8n8k4 f64), DFMA (FP64 FMA pipe), UTMALDG / UTMASTG /
UTMAREDG (TMA tensor copies), UBLKCP / UBLKRED (cp.async.bulk copies /
reduce-add), SYNCS (mbarrier), LDS / STS (shared memory).
usage: sass_summary.py [--out profiles/sass_summary.md]"""
import argparse
import collections
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["DMMA", "DFMA", "DMUL", "DADD", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "UBLKRED", "SYNCS", "LDS",
       "STS", "LDG", "STG", "SHFL"]


def family(name):
    m = re.search(r"tsm(\d+)?(\w+?)_kernel", name)
    base = re.search(r"(tsmttsm_mma_kernel|tsmttsm_kernel|tsmm_cstb_kernel|tsmm_cst_kernel|tsmm_mma_kernel|"
                     r"tsmm_kernel)", name)
    fam = base.group(1) if base else (m.group(0) if m else name)
    if fam in ("tsmttsm_mma_kernel", "tsmm_mma_kernel"):
        args = re.search(r"Cfg(ILi.*)EEEE", name)
        # the TMA template flag: 10th parameter of TsmttsmMmaCfg / 9th of TsmmMmaCfg
        bools = re.findall(r"Lb([01])E", name)
        if bools:
            tma = bools[1] if fam == "tsmttsm_mma_kernel" and len(bools) > 1 else bools[-1]
            fam += "+tma" if tma == "1" else "+bulk"
        _ = args
    return fam


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_summary.md"))
    a = ap.parse_args()
    cubins = sorted(glob.glob(os.path.join(ROOT, "paper_1905_03136_b200", "kcache", "*", "*.cubin")))
    fams = collections.defaultdict(lambda: collections.Counter())
    nk = collections.Counter()
    for c in cubins:
        out = subprocess.run(["cuobjdump", "-sass", c], capture_output=True, text=True).stdout
        cur = None
        for line in out.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                cur = family(m.group(1))
                nk[cur] += 1
                continue
            if cur is None:
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                op = m.group(2).split(".")[0]
                if op in OPS:
                    fams[cur][op] += 1
    lines = [f"# SASS opcode summary of the precompiled (NVRTC, sm_100a) kernels in kcache ({len(cubins)} cubins)",
             "", "Static instruction counts summed over the kernels of each family (tools/sass_summary.py).", "",
             "| family | kernels | " + " | ".join(OPS) + " |", "|---|---|" + "---|" * len(OPS)]
    for f in sorted(fams):
        lines.append(f"| {f} | {nk[f]} | " + " | ".join(str(fams[f][o]) for o in OPS) + " |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
