"""C-ABI library checks that need no GPU (-m "not gpu").

* libtsm.so loads and exports every function include/libtsm.h declares;
* argument validation happens before any CUDA call (so it is testable here);
* the AOT instantiation set covers the benchmark shapes;
* the binding fails loudly instead of falling back to CPU.
"""
import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libtsm.h")
LIB = os.path.join(ROOT, "paper_1905_03136_b200", "libtsm.so")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith("tsm")))


@pytest.fixture(scope="module")
def tsm():
    from paper_1905_03136_b200 import binding as libtsm
    return libtsm


def test_library_exists():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"


def test_exports_every_header_symbol(tsm):
    declared = header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if " T " in line)
    missing = [n for n in declared if n not in exported]
    assert not missing, missing
    assert sorted(tsm.EXPORTS) == declared


def test_no_torch_types_in_header():
    src = open(HEADER).read()
    assert "torch" not in re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    assert "#include <cuda" not in src  # plain C: no CUDA header dependency


def test_status_strings(tsm):
    for code, name in tsm.STATUS.items():
        assert tsm.lib.tsm_status_string(code).decode() == name


def _create(tsm, op, dt, M, N, dev=0):
    h = ctypes.c_void_p()
    return tsm.lib.tsm_plan_create(ctypes.byref(h), op, dt, M, N, dev), h


@pytest.mark.parametrize("M,N", [(0, 5), (5, 0), (65, 1), (1, 65), (-1, 3)])
def test_plan_rejects_bad_shapes(tsm, M, N):
    st, h = _create(tsm, 0, 0, M, N)
    assert st == 1 and not h.value  # TSM_ERR_INVALID_VALUE
    assert b"[1, 64]" in tsm.lib.tsm_last_error_detail()


def test_plan_rejects_bad_enums(tsm):
    assert _create(tsm, 7, 0, 4, 4)[0] == 1
    assert _create(tsm, 0, 9, 4, 4)[0] == 1
    assert tsm.lib.tsm_plan_create(None, 0, 0, 4, 4, 0) == 1


def test_null_plan_calls(tsm):
    assert tsm.lib.tsmttsm_d(None, 10, 16, 16, 16, 16, 1024, None) == 1
    assert tsm.lib.tsmm_z(None, 10, 16, 16, 16, None) == 1
    n = ctypes.c_size_t()
    assert tsm.lib.tsm_plan_workspace_bytes(None, 10, ctypes.byref(n)) == 1


def test_fill_validation(tsm):
    assert tsm.lib.tsm_fill(None, -1, 0, 1, 0, 0, None) == 1
    assert tsm.lib.tsm_fill(None, 10, 0, 1, 5, 0, None) == 1
    assert tsm.lib.tsm_fill(None, 0, 0, 1, 0, 0, None) == 0  # empty fill is a no-op


def test_plan_needs_a_gpu_here(tsm):
    # No GPU in this container: a valid plan request must fail with a CUDA
    # error, never silently succeed on a CPU path.
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, h = _create(tsm, 0, 0, 8, 8)
    assert st == 5 and not h.value


def test_build_info_covers_benchmark_shapes(tsm):
    info = json.loads(tsm.tsm_build_info())
    shapes = {tuple(s) for s in info["aot_shapes"]}
    for w in range(1, 65):
        assert (w, w) in shapes
    for s in [(1, 64), (64, 1), (16, 48)]:
        assert s in shapes
    assert info["instances"] == 4 * len(shapes)


def test_binding_refuses_cpu_tensors(tsm):
    import torch
    A = torch.zeros(4, 2, dtype=torch.float64)
    with pytest.raises(ValueError):
        tsm.tsmttsm(A, A)
    with pytest.raises(TypeError):
        tsm._dtype_code(torch.zeros(2, dtype=torch.float32))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1905_03136_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.c" not in src and "liboracle" not in src, f


def test_generator_consistency_host():
    # the values_at/column/rows helpers agree with the dense generator
    import tsminputs as ti
    A = ti.matrix(50, 7, "A")
    assert np.array_equal(ti.column(50, 7, 3, "A"), A[:, 3])
    assert np.array_equal(ti.rows(np.array([0, 17, 49]), 7, "A"), A[[0, 17, 49]])
    Z = ti.matrix(20, 3, "B", complex_=True, mode="int")
    assert np.array_equal(ti.column(20, 3, 2, "B", complex_=True, mode="int"), Z[:, 2])


def test_jit_precompile_without_device(tmp_path):
    """tsm_jit_precompile (build tooling) compiles a kernel with NVRTC into the
    cache without a GPU; bad shapes / configs are rejected (fresh process so
    TSM_JIT_CACHE_DIR applies)."""
    code = r'''
import ctypes, os, sys
from paper_1905_03136_b200 import binding as tsm
f = tsm.lib.tsm_jit_precompile
assert f(0, 0, 24, 24, None, 0) == 0, tsm.lib.tsm_last_error_detail()
assert f(1, 1, 17, 17, None, 0) == 0
assert f(0, 0, 65, 1, None, 0) == 1          # M out of range
assert f(0, 0, 33, 33, None, 2) == 0         # odd D widths: the strided default is the gather kernel
assert f(1, 0, 7, 1, None, 8) == 0           # TSM_FLAG_GATHER default exists for every shape
assert f(0, 1, 64, 64, None, 8) == 0
cfg = tsm.TsmConfig(threads=288, rows_per_chunk=30, p0=1, p1=1, p2=0, stages=3, ctas_per_sm=1, kernel=0, p3=0)
assert f(0, 0, 8, 8, ctypes.byref(cfg), 0) == 0
bad = tsm.TsmConfig(threads=100, rows_per_chunk=30, p0=1, p1=1, p2=0, stages=3, ctas_per_sm=1, kernel=0, p3=0)
assert f(0, 0, 8, 8, ctypes.byref(bad), 0) == 1
print("ok")
'''
    env = dict(os.environ, TSM_JIT_CACHE_DIR=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    cubins = [p for p in tmp_path.rglob("*.cubin")]
    assert len(cubins) >= 3


def test_flag_validation_without_device(tmp_path):
    """The 3M flag (kernel | 512) and the warp-order flag (kernel | 1024) are
    validated before any compilation: 3M needs dtype Z, a DMMA TSMTTSM kernel
    1/2 or the C-stationary TSMM kernel 3, and excludes complex-as-real; valid
    3M configurations compile with NVRTC on this CPU box (no device)."""
    code = r'''
import ctypes
from paper_1905_03136_b200 import binding as tsm
f = tsm.lib.tsm_jit_precompile
def cfg(**k):
    d = dict(threads=160, rows_per_chunk=32, p0=2, p1=2, p2=32, stages=3, ctas_per_sm=1, kernel=2, p3=32)
    d.update(k)
    return ctypes.byref(tsm.TsmConfig(**d))
assert f(0, 1, 32, 32, cfg(kernel=2 | 512), 0) == 0, tsm.lib.tsm_last_error_detail()      # Z TSMTTSM 3M (TMA)
assert f(0, 1, 32, 32, cfg(kernel=2 | 512 | 1024), 0) == 0                                # + plain warp order
assert f(0, 0, 32, 32, cfg(kernel=2 | 512), 0) == 1                                       # 3M needs Z
assert f(0, 1, 16, 16, cfg(kernel=2 | 512 | 256, p2=32, p3=32), 0) == 1                   # 3M excludes ZR
assert f(1, 1, 32, 32, cfg(threads=160, rows_per_chunk=64, p0=2, p1=2, p2=0, p3=0, kernel=3 | 512), 0) == 0
assert f(1, 1, 32, 32, cfg(threads=160, rows_per_chunk=64, p0=2, p1=2, p2=0, p3=0, kernel=4 | 512), 0) == 1
print("ok")
'''
    env = dict(os.environ, TSM_JIT_CACHE_DIR=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
