"""Build step: compile the tuned kernels with NVRTC into libtsm's kernel cache
(<package>/kcache, see include/libtsm.h tsm_jit_precompile).

Plans load these cubins instead of compiling at plan time.  torch is imported
first so that the NVRTC bound here is the one a torch process binds at run
time (the autotuner measured that code).  Runs on the CPU box: NVRTC needs no
device.  Stale kernel-source versions are pruned.
"""
from __future__ import annotations

import concurrent.futures as cf
import ctypes
import os
import shutil
import sys
import time

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
KCACHE = os.path.join(PKG, "kcache")


def main() -> int:
    import torch  # noqa: F401  (binds torch's NVRTC, as at run time)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_instances as gi
    lib = ctypes.CDLL(os.path.join(PKG, "libtsm.so"))
    lib.tsm_jit_precompile.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_uint]
    lib.tsm_jit_precompile.restype = ctypes.c_int
    lib.tsm_last_error_detail.restype = ctypes.c_char_p
    jobs = []
    for op in (0, 1):
        for dt in (0, 1):
            for (M, N) in gi.SHAPES:
                jobs.append((op, dt, M, N, 0))
                jobs.append((op, dt, M, N, 2))  # TSM_FLAG_STRIDED default (skipped if none)
                jobs.append((op, dt, M, N, 8))  # TSM_FLAG_GATHER default
    t0 = time.time()

    def one(j):
        op, dt, M, N, fl = j
        st = lib.tsm_jit_precompile(op, dt, M, N, None, fl)
        return j, st

    bad = []
    with cf.ThreadPoolExecutor(min(32, os.cpu_count() or 4)) as ex:
        for j, st in ex.map(one, jobs):
            if st not in (0, 2):  # 2: no strided kernel for this shape
                bad.append((j, st))
    # prune kernel caches of other source versions (the current one was just written / read)
    if os.path.isdir(KCACHE):
        subs = [os.path.join(KCACHE, d) for d in os.listdir(KCACHE) if d.startswith("src_")]
        if subs:
            cur = max(subs, key=os.path.getmtime)
            for d in subs:
                if d != cur:
                    shutil.rmtree(d, ignore_errors=True)
    print(f"precompiled {len(jobs) - len(bad)} of {len(jobs)} kernels into {KCACHE} in {time.time() - t0:.0f} s")
    if bad:
        print("failures:", bad[:5])
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
