"""Thin ctypes binding of libtsm (include/libtsm.h).

Argument marshalling only: every step of TSMTTSM / TSMM runs in libtsm.so's
CUDA kernels.  The raw functions keep the C names (``tsmttsm_d`` ...) and take
integer device pointers; the ``tsmttsm`` / ``tsmm`` helpers accept torch CUDA
tensors (PyTorch supplies device memory and the current stream only).

There is deliberately no CPU fallback: if libtsm.so is missing or cannot be
loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSM_LIB", os.path.join(PKG, "libtsm.so"))

TSM_SUCCESS = 0
STATUS = {0: "TSM_SUCCESS", 1: "TSM_ERR_INVALID_VALUE", 2: "TSM_ERR_UNSUPPORTED",
          3: "TSM_ERR_MISALIGNED", 4: "TSM_ERR_WORKSPACE", 5: "TSM_ERR_CUDA",
          6: "TSM_ERR_NCCL", 7: "TSM_ERR_INTERNAL"}
OP = {"tsmttsm": 0, "tsmm": 1}
DTYPE = {"d": 0, "z": 1}
TSM_COMM_DETERMINISTIC = 1
TSM_FLAG_CONJ = 1
TSM_FLAG_STRIDED = 2
TSM_FLAG_NO_GRID_REDUCE = 4  # measurement only: TSMTTSM without T4, C not written
TSM_FLAG_GATHER = 8  # gather-capable kernel: any row stride, 8-byte D bases (N4)
MAT_ID = {"A": 1, "B": 2, "C": 3}

# exported symbols declared in include/libtsm.h (checked by tests/test_abi.py)
EXPORTS = [
    "tsm_plan_create", "tsm_plan_create_config", "tsm_plan_get_config", "tsm_plan_workspace_bytes", "tsm_workspace_init", "tsm_plan_describe",
    "tsm_plan_destroy", "tsm_status_string", "tsm_last_error_detail",
    "tsmttsm_d", "tsmttsm_z", "tsmm_d", "tsmm_z", "tsm_fill", "tsm_l2_flush",
    "tsm_comm_unique_id", "tsm_comm_init", "tsm_comm_destroy", "tsm_comm_workspace_extra_bytes",
    "tsmttsm_allreduce_d", "tsmttsm_allreduce_z", "tsmm_bcast_d", "tsmm_bcast_z",
    "tsm_build_info", "tsm_plan_create_ex", "tsm_plan_get_flags", "tsmm_update_d", "tsmm_update_z",
    "tsm_cgs_step_d", "tsm_cgs_step_z", "tsmttsm_ld_d", "tsmttsm_ld_z", "tsmm_ld_d", "tsmm_ld_z",
    "tsm_jit_precompile", "tsm_peer_create", "tsm_peer_export", "tsm_peer_open", "tsm_peer_destroy",
    "tsm_peer_error", "tsmttsm_peer_d", "tsmttsm_peer_z", "tsm_peer_set_timeout", "tsm_peer_reset",
    "tsm_probe",
]


class ZComplex(ctypes.Structure):
    """tsm_zcomplex (include/libtsm.h), passed by value."""
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class TsmConfig(ctypes.Structure):
    """tsm_config (include/libtsm.h)."""
    _fields_ = [("threads", ctypes.c_int), ("rows_per_chunk", ctypes.c_int), ("p0", ctypes.c_int),
                ("p1", ctypes.c_int), ("p2", ctypes.c_int), ("stages", ctypes.c_int),
                ("ctas_per_sm", ctypes.c_int), ("kernel", ctypes.c_int), ("p3", ctypes.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class TsmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}" + (f" ({detail})" if detail else ""))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtsm.so not found at {LIB_PATH}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, I, I64, SZ, VP = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
    sig = {
        "tsm_plan_create": [ctypes.POINTER(P), I, I, I, I, I],
        "tsm_plan_create_config": [ctypes.POINTER(P), I, I, I, I, I, ctypes.POINTER(TsmConfig)],
        "tsm_plan_get_config": [P, ctypes.POINTER(TsmConfig)],
        "tsm_plan_workspace_bytes": [P, I64, ctypes.POINTER(SZ)],
        "tsm_workspace_init": [VP, SZ, VP],
        "tsm_plan_describe": [P, I64, ctypes.c_char_p, SZ],
        "tsm_plan_destroy": [P],
        "tsm_status_string": [I],
        "tsm_last_error_detail": [],
        "tsmttsm_d": [P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmttsm_z": [P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmm_d": [P, I64, VP, VP, VP, VP],
        "tsmm_z": [P, I64, VP, VP, VP, VP],
        "tsm_fill": [VP, I64, ctypes.c_uint64, I, I, I64, VP],
        "tsm_l2_flush": [VP, SZ, VP],
        "tsm_comm_unique_id": [VP],
        "tsm_comm_init": [ctypes.POINTER(P), VP, I, I, I, I],
        "tsm_comm_destroy": [P],
        "tsm_comm_workspace_extra_bytes": [P, P, ctypes.POINTER(SZ)],
        "tsmttsm_allreduce_d": [P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmttsm_allreduce_z": [P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmm_bcast_d": [P, P, I, I64, VP, VP, VP, VP],
        "tsmm_bcast_z": [P, P, I, I64, VP, VP, VP, VP],
        "tsm_build_info": [],
        "tsm_plan_create_ex": [ctypes.POINTER(P), I, I, I, I, I, ctypes.POINTER(TsmConfig), ctypes.c_uint],
        "tsm_plan_get_flags": [P, ctypes.POINTER(ctypes.c_uint)],
        "tsmm_update_d": [P, I64, ctypes.c_double, VP, VP, ctypes.c_double, VP, VP],
        "tsmm_update_z": [P, I64, ZComplex, VP, VP, ZComplex, VP, VP],
        "tsm_cgs_step_d": [P, P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsm_cgs_step_z": [P, P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmttsm_ld_d": [P, I64, VP, I64, VP, I64, VP, VP, SZ, VP],
        "tsmttsm_ld_z": [P, I64, VP, I64, VP, I64, VP, VP, SZ, VP],
        "tsmm_ld_d": [P, I64, VP, I64, VP, VP, I64, VP],
        "tsmm_ld_z": [P, I64, VP, I64, VP, VP, I64, VP],
        "tsm_jit_precompile": [I, I, I, I, ctypes.POINTER(TsmConfig), ctypes.c_uint],
        "tsm_peer_create": [ctypes.POINTER(P), I, I, I],
        "tsm_peer_export": [P, VP],
        "tsm_peer_open": [P, VP],
        "tsm_peer_destroy": [P],
        "tsm_peer_error": [P, ctypes.POINTER(I)],
        "tsm_peer_set_timeout": [P, ctypes.c_uint64],
        "tsm_peer_reset": [P, VP],
        "tsmttsm_peer_d": [P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsmttsm_peer_z": [P, P, I64, VP, VP, VP, VP, SZ, VP],
        "tsm_probe": [I, VP, SZ, I64, VP, ctypes.POINTER(ctypes.c_double)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_char_p if name in ("tsm_status_string", "tsm_last_error_detail",
                                               "tsm_build_info") else ctypes.c_int
    return lib


lib = _load()


def check(status: int, where: str) -> None:
    if status != TSM_SUCCESS:
        raise TsmError(status, where, lib.tsm_last_error_detail().decode(errors="replace"))


# ---------------------------------------------------------------------------
# Raw C-ABI functions (same names as include/libtsm.h; pointers as ints)
# ---------------------------------------------------------------------------
def tsm_plan_create(op: str, dtype: str, M: int, N: int, device: int) -> int:
    h = ctypes.c_void_p()
    check(lib.tsm_plan_create(ctypes.byref(h), OP[op], DTYPE[dtype], M, N, device),
          f"tsm_plan_create({op},{dtype},{M},{N})")
    return h.value


def tsm_plan_create_config(op: str, dtype: str, M: int, N: int, device: int, cfg: dict) -> int:
    h = ctypes.c_void_p()
    c = TsmConfig(**cfg)
    check(lib.tsm_plan_create_config(ctypes.byref(h), OP[op], DTYPE[dtype], M, N, device,
                                     ctypes.byref(c)), f"tsm_plan_create_config({op},{dtype},{M},{N})")
    return h.value


def tsm_plan_create_ex(op: str, dtype: str, M: int, N: int, device: int, cfg: dict | None,
                       flags: int) -> int:
    h = ctypes.c_void_p()
    c = TsmConfig(**cfg) if cfg is not None else None
    check(lib.tsm_plan_create_ex(ctypes.byref(h), OP[op], DTYPE[dtype], M, N, device,
                                 ctypes.byref(c) if c is not None else None, flags),
          f"tsm_plan_create_ex({op},{dtype},{M},{N},flags={flags})")
    return h.value


def tsm_plan_get_flags(plan: int) -> int:
    f = ctypes.c_uint()
    check(lib.tsm_plan_get_flags(plan, ctypes.byref(f)), "tsm_plan_get_flags")
    return f.value


def tsmm_update_d(plan, K, alpha, A, C, beta, B, stream):
    check(lib.tsmm_update_d(plan, K, float(alpha), A, C, float(beta), B, stream), "tsmm_update_d")


def tsmm_update_z(plan, K, alpha, A, C, beta, B, stream):
    a, b = complex(alpha), complex(beta)
    check(lib.tsmm_update_z(plan, K, ZComplex(a.real, a.imag), A, C, ZComplex(b.real, b.imag), B, stream),
          "tsmm_update_z")


def tsm_cgs_step_d(p_tt, p_mm, comm, K, A, B, C, ws, ws_bytes, stream):
    check(lib.tsm_cgs_step_d(p_tt, p_mm, comm, K, A, B, C, ws, ws_bytes, stream), "tsm_cgs_step_d")


def tsm_cgs_step_z(p_tt, p_mm, comm, K, A, B, C, ws, ws_bytes, stream):
    check(lib.tsm_cgs_step_z(p_tt, p_mm, comm, K, A, B, C, ws, ws_bytes, stream), "tsm_cgs_step_z")


def tsm_plan_get_config(plan: int) -> dict:
    c = TsmConfig()
    check(lib.tsm_plan_get_config(plan, ctypes.byref(c)), "tsm_plan_get_config")
    return c.as_dict()


def tsm_plan_destroy(plan: int) -> None:
    check(lib.tsm_plan_destroy(plan), "tsm_plan_destroy")


def tsm_plan_workspace_bytes(plan: int, K: int) -> int:
    n = ctypes.c_size_t()
    check(lib.tsm_plan_workspace_bytes(plan, K, ctypes.byref(n)), "tsm_plan_workspace_bytes")
    return n.value


def tsm_plan_describe(plan: int, K: int) -> str:
    buf = ctypes.create_string_buffer(1024)
    check(lib.tsm_plan_describe(plan, K, buf, 1024), "tsm_plan_describe")
    return buf.value.decode()


def tsm_workspace_init(ws: int, nbytes: int, stream: int) -> None:
    check(lib.tsm_workspace_init(ws, nbytes, stream), "tsm_workspace_init")


def tsmttsm_d(plan, K, A, B, C, ws, ws_bytes, stream):
    check(lib.tsmttsm_d(plan, K, A, B, C, ws, ws_bytes, stream), "tsmttsm_d")


def tsmttsm_z(plan, K, A, B, C, ws, ws_bytes, stream):
    check(lib.tsmttsm_z(plan, K, A, B, C, ws, ws_bytes, stream), "tsmttsm_z")


def tsmm_d(plan, K, A, C, B, stream):
    check(lib.tsmm_d(plan, K, A, C, B, stream), "tsmm_d")


def tsmm_z(plan, K, A, C, B, stream):
    check(lib.tsmm_z(plan, K, A, C, B, stream), "tsmm_z")


def tsm_fill(dst, n, seed, mat_id, mode, start, stream):
    check(lib.tsm_fill(dst, n, seed, mat_id, mode, start, stream), "tsm_fill")


def tsm_l2_flush(scratch, nbytes, stream):
    check(lib.tsm_l2_flush(scratch, nbytes, stream), "tsm_l2_flush")


PROBE = {"read": 0, "copy": 1, "dmma": 2, "clock": 3}


def probe(kind: str, buf, nbytes: int, iters: int, stream) -> float:
    """Launch one roofline-denominator probe (measurement only); returns the
    launch's work (bytes or FP64 flops) -- the caller times it with events."""
    w = ctypes.c_double()
    check(lib.tsm_probe(PROBE[kind], buf, nbytes, iters, stream, ctypes.byref(w)), "tsm_probe")
    return w.value


def tsm_build_info() -> str:
    return lib.tsm_build_info().decode()


# ---------------------------------------------------------------------------
# torch-tensor convenience layer (device memory + current stream from torch)
# ---------------------------------------------------------------------------
_plans: dict = {}
_ws: dict = {}
_mu = threading.Lock()


class Plan:
    """Owning wrapper of a tsm_plan handle."""

    def __init__(self, op: str, dtype: str, M: int, N: int, device: int = 0,
                 config: dict | None = None, conj: bool = False, strided: bool = False,
                 no_grid_reduce: bool = False, gather: bool = False):
        """conj=True (Z only, TSM_FLAG_CONJ): TSMTTSM C = A^H B, TSMM B = A conj(C).
        strided=True (TSM_FLAG_STRIDED): a kernel that takes strided row views.
        no_grid_reduce=True (TSM_FLAG_NO_GRID_REDUCE): MEASUREMENT ONLY, the
        reduction-overhead baseline; C is not written.
        gather=True (TSM_FLAG_GATHER): a kernel for strided views of any row
        stride and 8-byte aligned D bases."""
        self.op, self.dtype, self.M, self.N, self.device = op, dtype, M, N, device
        self.conj, self.strided, self.gather = conj, strided, gather
        self.handle = None
        if conj or strided or no_grid_reduce or gather:
            flags = (TSM_FLAG_CONJ if conj else 0) | (TSM_FLAG_STRIDED if strided else 0) | \
                (TSM_FLAG_NO_GRID_REDUCE if no_grid_reduce else 0) | (TSM_FLAG_GATHER if gather else 0)
            self.handle = tsm_plan_create_ex(op, dtype, M, N, device, config, flags)
        elif config is None:
            self.handle = tsm_plan_create(op, dtype, M, N, device)
        else:
            self.handle = tsm_plan_create_config(op, dtype, M, N, device, config)

    def config(self) -> dict:
        return tsm_plan_get_config(self.handle)

    def workspace_bytes(self, K: int) -> int:
        return tsm_plan_workspace_bytes(self.handle, K)

    def describe(self, K: int = 1 << 24) -> dict:
        import json
        return json.loads(tsm_plan_describe(self.handle, K))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:
            lib.tsm_plan_destroy(h)
            self.handle = None


def get_plan(op: str, dtype: str, M: int, N: int, device: int, conj: bool = False,
             strided: bool = False, gather: bool = False) -> Plan:
    key = (op, dtype, M, N, device, conj, strided, gather)
    with _mu:
        p = _plans.get(key)
        if p is None:
            p = Plan(op, dtype, M, N, device, conj=conj, strided=strided, gather=gather)
            _plans[key] = p
    return p


def _torch():
    import torch
    return torch


def _dtype_code(t) -> str:
    torch = _torch()
    if t.dtype == torch.float64:
        return "d"
    if t.dtype == torch.complex128:
        return "z"
    raise TypeError(f"libtsm supports float64 (D) and complex128 (Z), got {t.dtype}")


def _check_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("libtsm needs CUDA tensors (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError("libtsm needs contiguous row-major tensors")


def _check_rows(*ts):
    """CUDA 2-D tensors with unit column stride (row-strided views allowed, N4)."""
    for t in ts:
        if not t.is_cuda:
            raise ValueError("libtsm needs CUDA tensors (there is no CPU path)")
        if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1) or t.stride(0) < t.shape[1]:
            raise ValueError("libtsm needs row-major tensors with unit column stride")


def _ld(t) -> int:
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


def _view_mode(dt: str, views) -> str:
    """Plan kind for a call on (tensor, ld, width) views: "dense" (contiguous,
    16-byte aligned), "strided" (16-byte row strides and bases: TMA kernel when
    the shape has one), else "gather" (any stride, 8-byte D bases)."""
    S = 2 if dt == "z" else 1
    aligned = all(t.data_ptr() % 16 == 0 for t, _, _ in views)
    if aligned and all(ld == w for _, ld, w in views):
        return "dense"
    if aligned and all((ld * S) % 2 == 0 for _, ld, _ in views):
        return "strided"
    return "gather"


def _check_out(out, shape, like, name="out"):
    """A caller-supplied output must have exactly the shape, dtype and device
    the call writes (the C ABI cannot see buffer sizes)."""
    if out is None:
        return
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.dtype != like.dtype:
        raise ValueError(f"{name} has dtype {out.dtype}, expected {like.dtype}")
    if out.device != like.device:
        raise ValueError(f"{name} is on {out.device}, expected {like.device}")


def _check_plan(plan, op: str, dt: str, M: int, N: int, device: int):
    """An explicit plan must match the call's op, dtype, widths and device."""
    if plan is None:
        return
    if (plan.op, plan.dtype, plan.M, plan.N) != (op, dt, M, N):
        raise ValueError(f"plan is ({plan.op}, {plan.dtype}, M={plan.M}, N={plan.N}), "
                         f"the call is ({op}, {dt}, M={M}, N={N})")
    if plan.device != device:
        raise ValueError(f"plan is for device {plan.device}, tensors are on device {device}")


def _same(A, *ts):
    for t in ts:
        if t.dtype != A.dtype:
            raise ValueError(f"dtype mismatch: {t.dtype} vs {A.dtype}")
        if t.device != A.device:
            raise ValueError(f"device mismatch: {t.device} vs {A.device}")


def workspace(plan: Plan, K: int, stream: int, min_bytes: int = 0):
    """Cached, counter-zeroed workspace for (device, stream); grows as needed."""
    torch = _torch()
    need = max(plan.workspace_bytes(K), min_bytes, 256)
    key = (plan.device, stream)
    with _mu:
        buf = _ws.get(key)
        if buf is None or buf.numel() < need:
            buf = torch.zeros(need + (1 << 20), dtype=torch.uint8, device=f"cuda:{plan.device}")
            _ws[key] = buf
    return buf


def tsmttsm(A, B, out=None, plan: Plan | None = None, conj: bool | None = None):
    """C = A^T B (plain transpose; conj=True: A^H B, Z only) for torch CUDA
    tensors A (K x M), B (K x N).  Row-strided views (e.g. column subsets of a
    wider block vector) go through tsmttsm_ld_* with a TSM_FLAG_STRIDED plan.
    conj=None takes the plan's TSM_FLAG_CONJ (False without a plan); an
    explicit value must match the plan's."""
    torch = _torch()
    _check_rows(A, B)
    dt = _dtype_code(A)
    if B.dtype != A.dtype or A.dim() != 2 or B.dim() != 2 or A.shape[0] != B.shape[0]:
        raise ValueError("A and B must be 2-D, same dtype, same row count")
    K, M = A.shape
    N = B.shape[1]
    dev = A.device.index
    _same(A, B)
    lda, ldb = _ld(A), _ld(B)
    mode = _view_mode(dt, [(A, lda, M), (B, ldb, N)])
    dense = mode == "dense"
    _check_plan(plan, "tsmttsm", dt, M, N, dev)
    if conj is None:
        conj = plan.conj if plan is not None else False
    if plan is not None and plan.conj != conj:
        raise ValueError("conj does not match the plan's TSM_FLAG_CONJ")
    plan = plan or get_plan("tsmttsm", dt, M, N, dev, conj, strided=mode == "strided", gather=mode == "gather")
    _check_out(out, (M, N), A)
    C = out if out is not None else torch.empty((M, N), dtype=A.dtype, device=A.device)
    _check_cuda(C)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    ws = workspace(plan, K, stream)
    if dense:
        f = tsmttsm_z if dt == "z" else tsmttsm_d
        f(plan.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    else:
        f = lib.tsmttsm_ld_z if dt == "z" else lib.tsmttsm_ld_d
        check(f(plan.handle, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ws.data_ptr(), ws.numel(),
                stream), "tsmttsm_ld")
    return C


def tsmm(A, C, out=None, plan: Plan | None = None):
    """B = A C for torch CUDA tensors A (K x M), C (M x N); A and `out` may be
    row-strided views (TSM_FLAG_STRIDED plan, tsmm_ld_*)."""
    torch = _torch()
    _check_rows(A)
    _check_cuda(C)
    dt = _dtype_code(A)
    if C.dtype != A.dtype or A.dim() != 2 or C.dim() != 2 or A.shape[1] != C.shape[0]:
        raise ValueError("A (K x M) and C (M x N) must be 2-D with matching M and dtype")
    K, M = A.shape
    N = C.shape[1]
    dev = A.device.index
    _same(A, C)
    _check_out(out, (K, N), A)
    B = out if out is not None else torch.empty((K, N), dtype=A.dtype, device=A.device)
    _check_rows(B)
    lda, ldb = _ld(A), _ld(B)
    mode = _view_mode(dt, [(A, lda, M), (B, ldb, N)])
    dense = mode == "dense"
    _check_plan(plan, "tsmm", dt, M, N, dev)
    plan = plan or get_plan("tsmm", dt, M, N, dev, strided=mode == "strided", gather=mode == "gather")
    stream = torch.cuda.current_stream(A.device).cuda_stream
    if dense:
        f = tsmm_z if dt == "z" else tsmm_d
        f(plan.handle, K, A.data_ptr(), C.data_ptr(), B.data_ptr(), stream)
    else:
        f = lib.tsmm_ld_z if dt == "z" else lib.tsmm_ld_d
        check(f(plan.handle, K, A.data_ptr(), lda, C.data_ptr(), B.data_ptr(), ldb, stream), "tsmm_ld")
    return B


def tsmm_update(A, C, B, alpha=1.0, beta=0.0, plan: Plan | None = None, conj: bool | None = None):
    """In place B <- alpha * A C + beta * B (NEXT N1; conj: A conj(C), Z only;
    conj=None takes the plan's TSM_FLAG_CONJ).  Returns B."""
    torch = _torch()
    _check_cuda(A, C, B)
    dt = _dtype_code(A)
    if C.dtype != A.dtype or B.dtype != A.dtype or A.dim() != 2 or C.dim() != 2 or B.dim() != 2 \
            or A.shape[1] != C.shape[0] or B.shape != (A.shape[0], C.shape[1]):
        raise ValueError("A (K x M), C (M x N), B (K x N): shapes / dtypes do not match")
    K, M = A.shape
    N = C.shape[1]
    _same(A, C, B)
    _check_plan(plan, "tsmm", dt, M, N, A.device.index)
    if conj is None:
        conj = plan.conj if plan is not None else False
    if plan is not None and plan.conj != conj:
        raise ValueError("conj does not match the plan's TSM_FLAG_CONJ")
    plan = plan or get_plan("tsmm", dt, M, N, A.device.index, conj)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    f = tsmm_update_z if dt == "z" else tsmm_update_d
    f(plan.handle, K, alpha, A.data_ptr(), C.data_ptr(), beta, B.data_ptr(), stream)
    return B


def cgs_step(A, B, C=None, p_tt: Plan | None = None, p_mm: Plan | None = None, comm=None):
    """One block classical Gram-Schmidt projection of B (K x N) against the
    basis A (K x M), in place: C = A^T B (A^H B for Z), then
    B <- B - A C.  comm: a Comm (K = this rank's rows; C summed over ranks).
    Returns C."""
    torch = _torch()
    _check_cuda(A, B)
    dt = _dtype_code(A)
    if A.dim() != 2 or B.dim() != 2 or A.shape[0] != B.shape[0]:
        raise ValueError("A (K x M) and B (K x N) must be 2-D with the same row count")
    _same(A, B)
    K, M = A.shape
    N = B.shape[1]
    dev = A.device.index
    _check_plan(p_tt, "tsmttsm", dt, M, N, dev)
    _check_plan(p_mm, "tsmm", dt, M, N, dev)
    p_tt = p_tt or get_plan("tsmttsm", dt, M, N, dev, dt == "z")
    p_mm = p_mm or get_plan("tsmm", dt, M, N, dev)
    _check_out(C, (M, N), A, "C")
    C = C if C is not None else torch.empty((M, N), dtype=A.dtype, device=A.device)
    _check_cuda(C)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    extra = 0
    if comm is not None:
        n = ctypes.c_size_t()
        check(lib.tsm_comm_workspace_extra_bytes(comm.handle, p_tt.handle, ctypes.byref(n)),
              "tsm_comm_workspace_extra_bytes")
        extra = n.value
    ws = workspace(p_tt, K, stream, p_tt.workspace_bytes(K) + extra)
    f = tsm_cgs_step_z if dt == "z" else tsm_cgs_step_d
    f(p_tt.handle, p_mm.handle, comm.handle if comm is not None else None, K, A.data_ptr(), B.data_ptr(),
      C.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    return C


def fill(t, mat: str, seed: int, mode: str = "fp", start: int = 0):
    """Fill a float64/complex128 CUDA tensor with the counter-based generator
    (the same values tsminputs.matrix() produces on the host).  `start` is the
    flat real-value index of t[0] in the generator stream (a rank's shard of a
    global matrix starts at row_offset * width (* 2 for complex))."""
    torch = _torch()
    _check_cuda(t)
    n = t.numel() * (2 if t.dtype == torch.complex128 else 1)
    if t.dtype not in (torch.float64, torch.complex128):
        raise TypeError("fill expects float64 or complex128")
    stream = torch.cuda.current_stream(t.device).cuda_stream
    tsm_fill(t.data_ptr(), n, seed, MAT_ID[mat], 0 if mode == "fp" else 1, start, stream)
    return t


# ---------------------------------------------------------------------------
# multi-GPU (one process per GPU; NCCL id exchanged through torch.distributed)
# ---------------------------------------------------------------------------
class Comm:
    def __init__(self, rank: int, world: int, device: int, deterministic: bool = False,
                 group=None):
        import torch.distributed as dist
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            check(lib.tsm_comm_unique_id(uid), "tsm_comm_unique_id")
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        flags = TSM_COMM_DETERMINISTIC if deterministic else 0
        check(lib.tsm_comm_init(ctypes.byref(h), uid, world, rank, device, flags), "tsm_comm_init")
        self.handle = h.value
        self.rank, self.world, self.device, self.deterministic = rank, world, device, deterministic

    def extra_bytes(self, plan: Plan) -> int:
        n = ctypes.c_size_t()
        check(lib.tsm_comm_workspace_extra_bytes(self.handle, plan.handle, ctypes.byref(n)),
              "tsm_comm_workspace_extra_bytes")
        return n.value

    def close(self):
        if self.handle:
            check(lib.tsm_comm_destroy(self.handle), "tsm_comm_destroy")
            self.handle = None


def tsmttsm_allreduce(comm: Comm, A, B, out=None):
    torch = _torch()
    _check_cuda(A, B)
    dt = _dtype_code(A)
    if A.dim() != 2 or B.dim() != 2 or A.shape[0] != B.shape[0]:
        raise ValueError("A (K x M) and B (K x N) must be 2-D with the same row count")
    _same(A, B)
    K, M = A.shape
    N = B.shape[1]
    plan = get_plan("tsmttsm", dt, M, N, A.device.index)
    _check_out(out, (M, N), A)
    C = out if out is not None else torch.empty((M, N), dtype=A.dtype, device=A.device)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    need = plan.workspace_bytes(K) + 256 + comm.extra_bytes(plan)
    ws = workspace(plan, K, stream, need)
    f = lib.tsmttsm_allreduce_z if dt == "z" else lib.tsmttsm_allreduce_d
    check(f(plan.handle, comm.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(),
            ws.numel(), stream), "tsmttsm_allreduce")
    return C


def tsmm_bcast(comm: Comm, A, C, root: int = 0, out=None):
    torch = _torch()
    _check_cuda(A, C)
    dt = _dtype_code(A)
    if A.dim() != 2 or C.dim() != 2 or A.shape[1] != C.shape[0]:
        raise ValueError("A (K x M) and C (M x N) must be 2-D with matching M")
    _same(A, C)
    K, M = A.shape
    N = C.shape[1]
    plan = get_plan("tsmm", dt, M, N, A.device.index)
    _check_out(out, (K, N), A)
    B = out if out is not None else torch.empty((K, N), dtype=A.dtype, device=A.device)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    f = lib.tsmm_bcast_z if dt == "z" else lib.tsmm_bcast_d
    check(f(plan.handle, comm.handle, root, K, A.data_ptr(), C.data_ptr(), B.data_ptr(), stream),
          "tsmm_bcast")
    return B


# ---------------------------------------------------------------------------
# NEXT N3: TSMTTSM with the grid reduction fused with the cross-GPU sum over
# peer memory (CUDA IPC + NVLink P2P; include/libtsm.h tsm_peer_*)
# ---------------------------------------------------------------------------
class PeerComm:
    """One per rank.  The 64-byte IPC handles of the slot buffers are exchanged
    with torch.distributed.all_gather_object (any backend, e.g. gloo)."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist
        h = ctypes.c_void_p()
        check(lib.tsm_peer_create(ctypes.byref(h), world, rank, device), "tsm_peer_create")
        self.handle = h.value
        self.rank, self.world, self.device = rank, world, device
        mine = ctypes.create_string_buffer(64)
        check(lib.tsm_peer_export(self.handle, mine), "tsm_peer_export")
        if world > 1:
            got = [None] * world
            dist.all_gather_object(got, bytes(mine.raw), group=group)
        else:
            got = [bytes(mine.raw)]
        allh = ctypes.create_string_buffer(b"".join(got), 64 * world)
        check(lib.tsm_peer_open(self.handle, allh), "tsm_peer_open")

    def error(self) -> int:
        v = ctypes.c_int()
        check(lib.tsm_peer_error(self.handle, ctypes.byref(v)), "tsm_peer_error")
        return v.value

    def set_timeout(self, seconds: float) -> None:
        check(lib.tsm_peer_set_timeout(self.handle, int(seconds * 1e9)), "tsm_peer_set_timeout")

    def reset(self) -> None:
        """Collective: every rank resets, then barriers (include/libtsm.h)."""
        import torch
        import torch.distributed as dist
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(lib.tsm_peer_reset(self.handle, stream), "tsm_peer_reset")
        if self.world > 1:
            dist.barrier()

    def close(self):
        if self.handle:
            check(lib.tsm_peer_destroy(self.handle), "tsm_peer_destroy")
            self.handle = None


def tsmttsm_peer(peer: PeerComm, A, B, out=None, plan: Plan | None = None):
    """C = sum over ranks of A_r^T B_r, replicated, with the grid reduction
    fused with the cross-GPU rank-order sum (no NCCL call).  A, B: this rank's
    K_local x M / K_local x N rows (K_local may be 0)."""
    torch = _torch()
    _check_cuda(A, B)
    dt = _dtype_code(A)
    if A.dim() != 2 or B.dim() != 2 or A.shape[0] != B.shape[0]:
        raise ValueError("A (K x M) and B (K x N) must be 2-D with the same row count")
    _same(A, B)
    K, M = A.shape
    N = B.shape[1]
    _check_plan(plan, "tsmttsm", dt, M, N, A.device.index)
    plan = plan or get_plan("tsmttsm", dt, M, N, A.device.index)
    _check_out(out, (M, N), A)
    C = out if out is not None else torch.empty((M, N), dtype=A.dtype, device=A.device)
    stream = torch.cuda.current_stream(A.device).cuda_stream
    ws = workspace(plan, K, stream)
    f = lib.tsmttsm_peer_z if dt == "z" else lib.tsmttsm_peer_d
    check(f(plan.handle, peer.handle, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(),
            ws.numel(), stream), "tsmttsm_peer")
    return C
