"""Build libtsm.so in-tree (nvcc, sm_100a) -- used by __graft_entry__.build().

Steps: regenerate the AOT instance files (tools/gen_instances.py), compile
every translation unit with nvcc in parallel (incremental: an object is
rebuilt when its source, the shared headers or the flags change), link
``paper_1905_03136_b200/libtsm.so`` with a static CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libtsm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
HEADERS = ["tsm_kernels.cuh", "tsm_registry.h", "tsm_internal.h", "gen/kernel_source.inc"]


def _sources():
    srcs = [os.path.join(CSRC, f) for f in ("tsm_api.cu", "tsm_comm.cu", "tsm_peer.cu", "tsm_registry.cpp",
                                            "tsm_jit.cpp")]
    gen = os.path.join(CSRC, "gen")
    srcs += sorted(os.path.join(gen, f) for f in os.listdir(gen)
                   if f.endswith(".cu") or f.endswith(".cpp"))
    return srcs


def _digest(src: str) -> str:
    h = hashlib.sha1()
    for p in [src] + [os.path.join(CSRC, x) for x in HEADERS] + \
            [os.path.join(ROOT, "include", "libtsm.h")]:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src: str) -> str:
    base = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(OBJ, base + "." + _digest(src) + ".o")
    if os.path.exists(obj):
        return obj
    lang = ["-x", "cu"] if src.endswith(".cpp") else []
    tmp = obj + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *lang, "-I", CSRC, "-I", os.path.join(ROOT, "include"),
           "-c", src, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if "spill" in r.stderr and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)
    os.replace(tmp, obj)
    return obj


def build(jobs: int | None = None, verbose: bool = True) -> str:
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_instances  # noqa: E402
    gen_instances.main()
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(_compile, srcs))
    keep = set(os.path.basename(o) for o in objs)
    for f in os.listdir(OBJ):  # drop stale objects of earlier source versions
        if f.endswith(".o") and f not in keep:
            os.remove(os.path.join(OBJ, f))
    stamp = hashlib.sha1("".join(objs).encode()).hexdigest()[:16]
    stamp_file = os.path.join(OBJ, "libtsm.stamp")
    if os.path.exists(LIB) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        precompile()
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "-o", tmp, *objs,
           "-L/usr/local/cuda/lib64", "-lnvrtc", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
           "-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp_file, "w") as f:
        f.write(stamp)
    if verbose:
        print(f"built {LIB} from {len(srcs)} translation units")
    precompile()
    return LIB


def precompile() -> None:
    """NVRTC-compile the tuned kernels into <package>/kcache (precompile.py,
    in a fresh interpreter so torch's NVRTC is the one bound)."""
    r = subprocess.run([sys.executable, os.path.join(PKG, "precompile.py")], capture_output=True, text=True)
    sys.stdout.write(r.stdout)
    if r.returncode != 0:
        raise RuntimeError(f"kernel precompile failed:\n{r.stdout[-2000:]}{r.stderr[-2000:]}")


if __name__ == "__main__":
    build()
