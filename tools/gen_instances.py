#!/usr/bin/env python3
"""Emit the AOT instantiation set of libtsm's width-specialised kernels.

For every (op, dtype, M, N) in the AOT shape set this writes one explicit
template instantiation (C++ templates, csrc/tsm_kernels.cuh) plus a registry
entry carrying its launch parameters.  Tile / launch parameters come from
``tune/b200.json`` (autotuned on the B200, tools/autotune.py) when present,
otherwise from the heuristics below.

Output: paper_1905_03136_b200/csrc/gen/{inst_*.cu, registry_gen.cpp}
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GEN = os.path.join(ROOT, "paper_1905_03136_b200", "csrc", "gen")
TUNE = os.path.join(ROOT, "tune", "b200.json")

# shapes instantiated ahead of time (both ops, both dtypes)
SQUARE = [(w, w) for w in range(1, 65)]
NONSQUARE = [(1, 64), (64, 1), (16, 48), (48, 16),             # BASELINE configs[3]
             (1, 2), (2, 1), (3, 5), (5, 3), (7, 2), (13, 29), (29, 13),
             (33, 17), (17, 33), (5, 64), (64, 5), (1, 7), (9, 1), (63, 64), (64, 63)]
SHAPES = SQUARE + [s for s in NONSQUARE if s[0] != s[1]]


def pow2ceil(x: int) -> int:
    p = 1
    while p < x:
        p <<= 1
    return p


def pow2floor(x: int) -> int:
    p = 1
    while p * 2 <= x:
        p <<= 1
    return p


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def tsmttsm_default(M: int, N: int, z: bool) -> dict:
    """Register-tile choice: big tiles for FMA/load, but at
    least 32 threads per row (a warp shares one row -> broadcast smem reads)
    whenever the row has >= 32 cells."""
    tmax_m, tmax_n = (4, 8) if z else (8, 8)
    MT = 1
    while cdiv(M, MT) > tmax_m and MT * 2 <= M:
        MT *= 2
    NTL = 1
    while cdiv(N, NTL) > tmax_n and NTL * 2 <= N:
        NTL *= 2
    tpr_min = min(32, pow2floor(M) * pow2floor(N))
    while MT * NTL < tpr_min:
        TM, TN = cdiv(M, MT), cdiv(N, NTL)
        can_m, can_n = MT * 2 <= M, NTL * 2 <= N
        if can_n and (TN >= TM or not can_m):
            NTL *= 2
        elif can_m:
            MT *= 2
        else:
            break
    NT = 256
    RB = NT // (MT * NTL)
    S = 2 if z else 1
    row_bytes = (M + N) * 8 * S
    R = max(2, (16384 // row_bytes))
    step = max(2, RB) if RB % 2 == 0 or RB == 1 else 2 * RB
    R = max(step, (R // step) * step)
    return dict(MT=MT, NTL=NTL, NT=NT, R=R, stages=4, ctas=4, impl=0)


def use_mma(M: int, N: int, z: bool) -> bool:
    """DMMA where the FP64 work per byte is high (PAPER.md:126-143 intensity
    I = f*M*N / (s*(M+N))): at I >= ~2 flop/B the FP64 pipe must run at >= ~40 %
    of peak just to keep up with HBM, where the register-tile kernel becomes
    issue-bound (ncu r01)."""
    f, s = (8, 16) if z else (2, 8)
    return f * M * N / (s * (M + N)) >= 2.0 and min(M, N) >= 8


def tsmttsm_mma_default(M: int, N: int, z: bool) -> dict:
    """DMMA kernel: WM x WN 8x8 accumulator blocks per warp (<= 32 accumulator
    doubles per lane), NW consumer warps (a multiple of the warp tiles) + 1
    producer warp, ~24 KB stages."""
    MB, NB = cdiv(M, 8), cdiv(N, 8)
    wmax = 8 if z else 16  # WM*WN blocks per warp
    best = None
    for WM in range(1, min(MB, 8) + 1):
        for WN in range(1, min(NB, 8) + 1):
            if WM * WN > wmax:
                continue
            if cdiv(MB, WM) * cdiv(NB, WN) > 16:
                continue
            # load balance (padded / useful blocks) x fragment loads per DMMA
            bal = cdiv(MB, WM) * WM * cdiv(NB, WN) * WN / (MB * NB)
            key = (bal * (1 + 0.5 * (WM + WN) / (WM * WN)), abs(WM - WN))
            if best is None or key < best[0]:
                best = (key, WM, WN)
    _, WM, WN = best
    WT = cdiv(MB, WM) * cdiv(NB, WN)
    NW = WT * max(1, 8 // WT)
    RS = NW // WT
    S = 2 if z else 1
    row_bytes = (M + N) * 8 * S
    if tma_ok(M, N, z):
        # 2-D TMA boxes of 16 doubles, 128B swizzle (conflict-free fragments)
        tb = (cdiv(M * S, 16) + cdiv(N * S, 16)) * 128
        step = max(8, 4 * RS)
        step = step if step % 8 == 0 else 2 * step
        R = min(256, max(step, (24576 // tb) // step * step))
        return dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=R, stages=4, ctas=2, impl=2, AP=M, BP=N)
    step = 4 * RS
    R = max(step, (24576 // row_bytes) // step * step)
    return dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=R, stages=4, ctas=2, impl=1,
                AP=pick_stride(M, z, "t"), BP=pick_stride(N, z, "t"))


def edge_candidates(M: int, N: int, z: bool) -> list:
    """DMMA on the 8-aligned core + one DFMA edge warp (EDGE=1), for widths
    just above a multiple of 8 (M % 8 or N % 8 in 1..3)."""
    if M < 8 or N < 8 or (M % 8 not in (1, 2, 3, 4) and N % 8 not in (1, 2, 3, 4)):
        return []
    S = 2 if z else 1
    MC, NC = (M // 8) * 8, (N // 8) * 8
    if ((M - MC) * cdiv(N, 32) + cdiv(MC, 32) * (N - NC)) * S > 64:  # edge-strip accumulators per lane
        return []
    MB, NB = M // 8, N // 8
    wmax = 8 if z else 16
    wt = []
    for WM in range(1, min(MB, 8) + 1):
        for WN in range(1, min(NB, 8) + 1):
            if WM * WN > wmax or cdiv(MB, WM) * cdiv(NB, WN) > 16:
                continue
            bal = cdiv(MB, WM) * WM * cdiv(NB, WN) * WN / (MB * NB)
            wt.append((bal * (1 + 0.5 * (WM + WN) / (WM * WN)), WM, WN))
    wt.sort()
    out = []
    row = (M + N) * 8 * S
    for (_, WM, WN) in wt[:3]:
        WT = cdiv(MB, WM) * cdiv(NB, WN)
        for k in (1, 2, 4):
            NW = WT * k
            if NW > 16 or NW < 2:
                continue
            for ne in (1, 2, 4):  # edge warps split the rows of a chunk
                if NW + ne + 1 > 32:
                    continue
                for tgt in (16384, 32768):
                    Rd = _rows(16 * k, row, tgt)  # whole k-step atoms for any row spacing
                    out.append(dict(MT=WM, NTL=WN, NT=(NW + ne + 1) * 32, R=Rd, impl=1,
                                    AP=M, BP=N, EDGE=ne))
                    if tma_ok(M, N, z):
                        tb = (cdiv(M * S, 16) + cdiv(N * S, 16)) * 128
                        step = 4 * k if (4 * k) % 8 == 0 else 8 * k
                        Rt = min(256 // step * step, max(step, (tgt // tb) // step * step))
                        out.append(dict(MT=WM, NTL=WN, NT=(NW + ne + 1) * 32, R=Rt, impl=2, AP=M, BP=N,
                                        EDGE=ne))
    # paired core fragments (TMA) + edge warps: the best even warp tiles
    if not z and tma_ok(M, N, z):
        tb = (cdiv(M, 16) + cdiv(N, 16)) * 128
        for (_, WM, WN) in [t for t in wt if t[1] % 2 == 0 and t[2] % 2 == 0][:2]:
            WT = cdiv(MB, WM) * cdiv(NB, WN)
            for k in (1, 2, 4):
                NW = WT * k
                if NW > 16 or NW < 2:
                    continue
                for ne in (1, 2, 4):
                    if NW + ne + 1 > 32:
                        continue
                    for tgt in (16384, 32768):
                        step = 4 * k if (4 * k) % 8 == 0 else 8 * k
                        Rt = min(256 // step * step, max(step, (tgt // tb) // step * step))
                        out.append(dict(MT=WM, NTL=WN, NT=(NW + ne + 1) * 32, R=Rt, impl=2, AP=M, BP=N,
                                        EDGE=ne, PAIR=1))
    return out


def lblock_candidates(M: int, N: int, z: bool) -> list:
    """LB=1: the core tilings of the inline-edge search with the edge
    strips on L-blocks (tsm_kernels.cuh LB) -- only where they need fewer MMA
    blocks than the padded tiling."""
    if M < 8 or N < 8 or not (1 <= M % 8 <= 6 and 1 <= N % 8 <= 6):
        return []
    MR, NR = M % 8, N % 8
    MC, NC = M - MR, N - NR
    nl = max(cdiv(MC, 8 - MR), cdiv(NC, 8 - NR))
    if (MC // 8) * (NC // 8) + nl >= cdiv(M, 8) * cdiv(N, 8):
        return []
    out, seen = [], set()
    for c in inline_edge_candidates(M, N, z):
        c = dict(c)
        c.pop("EI", None)
        c["LB"] = 1
        k = tuple(sorted(c.items()))
        if k not in seen:
            seen.add(k)
            out.append(c)
    return out


def inline_edge_candidates(M: int, N: int, z: bool) -> list:
    """EI=1: the edge candidates without edge warps -- the consumer warps
    compute the edge strips between their DMMAs (<= 16 strip accumulators
    per lane)."""
    S = 2 if z else 1
    if M < 8 or N < 8 or (M % 8 == 0 and N % 8 == 0):
        return []
    MC, NC = (M // 8) * 8, (N // 8) * 8
    if ((M - MC) * cdiv(N, 32) + cdiv(MC, 32) * (N - NC)) * S > 16:
        return []
    out, seen = [], set()

    def add(c):
        k = tuple(sorted(c.items()))
        if k not in seen:
            seen.add(k)
            out.append(c)

    for c in edge_candidates(M, N, z):
        ne = c.pop("EDGE")
        add(dict(c, NT=c["NT"] - 32 * ne, EI=1))
    # a wider search of the core tiling: more warp tiles, more row slots (the
    # consumer warps carry the edge work, so more of them share it)
    MB, NB = M // 8, N // 8
    wmax = 8 if z else 16
    row = (M + N) * 8 * S
    wt = []
    for WM in range(1, min(MB, 8) + 1):
        for WN in range(1, min(NB, 8) + 1):
            if WM * WN > wmax or cdiv(MB, WM) * cdiv(NB, WN) > 16:
                continue
            bal = cdiv(MB, WM) * WM * cdiv(NB, WN) * WN / (MB * NB)
            wt.append((bal * (1 + 0.5 * (WM + WN) / (WM * WN)), WM, WN))
    wt.sort()
    for (_, WM, WN) in wt[:6]:
        WT = cdiv(MB, WM) * cdiv(NB, WN)
        for k in (1, 2, 4, 8):
            NW = WT * k
            if NW > 16 or NW < 2:
                continue
            for tgt in (16384, 32768, 65536):
                add(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=_rows(16 * k, row, tgt), impl=1, AP=M, BP=N, EI=1))
                if tma_ok(M, N, z):
                    tb = (cdiv(M * S, 16) + cdiv(N * S, 16)) * 128
                    step = 4 * k if (4 * k) % 8 == 0 else 8 * k
                    Rt = min(256 // step * step, max(step, (tgt // tb) // step * step))
                    add(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=Rt, impl=2, AP=M, BP=N, EI=1))
    return out


def pair_stride(w: int) -> int:
    """Smallest even smem stride >= w whose 4 fragment rows start 32 bytes
    apart modulo 128: the 8 lanes of each LDS.128 phase then read 8 distinct
    16-byte granules (conflict-free paired loads without the swizzle)."""
    st = w
    while st % 16 not in (4, 12):
        st += 1
    return st


def pair_candidates(M: int, N: int, z: bool) -> list:
    """Real DMMA TSMTTSM with paired fragment loads (PAIR=1): each lane loads
    rows (m, m+1) with one 16-byte LDS feeding two 8x8 blocks, halving the
    fragment load instructions per DMMA.  Needs even WM, WN."""
    if z or M < 16 or N < 16:
        return []
    MB, NB = cdiv(M, 8), cdiv(N, 8)  # an odd last block is loaded single
    wt = []
    for WM in range(2, min(MB, 8) + 1, 2):
        for WN in range(2, min(NB, 8) + 1, 2):
            if WM * WN > 16 or cdiv(MB, WM) * cdiv(NB, WN) > 16:
                continue
            bal = cdiv(MB, WM) * WM * cdiv(NB, WN) * WN / (MB * NB)
            wt.append((bal * (1 + 0.5 * (WM + WN) / (WM * WN)), WM, WN))
    wt.sort()
    out = []
    row = (M + N) * 8
    for (_, WM, WN) in wt[:3]:
        WT = cdiv(MB, WM) * cdiv(NB, WN)
        for k in (1, 2, 4, 8):
            NW = WT * k
            if NW > 16:
                break
            if NW < 4 and WT * k * 2 <= 16:
                continue
            for tgt in (16384, 32768, 65536):
                if M % 2 == 0 and N % 2 == 0:  # conflict-free strides (row copies if padded)
                    Rp = _rows(16 * k, row, tgt)  # whole 16-row k-step atoms (kernel KD <= 4)
                    out.append(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=Rp, impl=1,
                                    AP=pair_stride(M), BP=pair_stride(N), PAIR=1))
                    if M % 8 and N % 8 and (M % 4 == N % 4):  # dense rows, spaced k-steps
                        out.append(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=Rp, impl=1,
                                        AP=M, BP=N, PAIR=1))
                if tma_ok(M, N, z):
                    tb = (cdiv(M, 16) + cdiv(N, 16)) * 128
                    step = 4 * k if (4 * k) % 8 == 0 else 8 * k
                    Rt = min(256 // step * step, max(step, (tgt // tb) // step * step))
                    out.append(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=Rt, impl=2, AP=M, BP=N, PAIR=1))
    return out


def tma_ok(M: int, N: int, z: bool) -> bool:
    """2-D tensor maps need 16-byte global row strides; boxes are 16 doubles."""
    S = 2 if z else 1
    return (M * S) % 2 == 0 and (N * S) % 2 == 0 and M * S >= 16 and N * S >= 16


def tsmttsm_pick(M: int, N: int, z: bool) -> dict:
    return tsmttsm_mma_default(M, N, z) if use_mma(M, N, z) else tsmttsm_default(M, N, z)


def tsmm_default(M: int, N: int, z: bool) -> dict:
    """C in smem; TN interleaved columns x U rows per thread
    (PAPER.md:661-714); MSPLIT lanes share an output so a warp reads one row
    group of A (broadcast)."""
    # lanes along n first (coalesced outputs, broadcast A reads), then MSPLIT
    # lanes split the m-sum to fill the warp (one butterfly per output).
    S = 2 if z else 1
    NTL = min(32, pow2floor(N))
    TN = cdiv(N, NTL)
    MSPLIT = 1
    while NTL * MSPLIT * 2 <= 32 and MSPLIT * 2 <= M:
        MSPLIT *= 2
    GS = NTL * MSPLIT
    acc_max = 16 if z else 32  # accumulator doubles per thread: U*TN*S <= 32
    U = max(1, min(16, acc_max // TN))
    NT = 256
    # staging buffers (A chunk, output pass) of at most ~16 KB, 32 KB when
    # the shape is FMA-heavy (big U amortises the C loads)
    T = 32768 if M * N >= 1024 else 16384
    rows_cap = max(2, T // (max(M, N) * S * 8))
    while (NT // GS) * U > rows_cap:
        if NT > 128:
            NT //= 2
        elif U > 4:
            U //= 2
        elif NT > 32:
            NT //= 2
        elif U > 1:
            U //= 2
        else:
            break
    rpp = (NT // GS) * U
    if rpp % 2:
        U *= 2
        rpp *= 2
    R = rpp * max(1, round(T / (rpp * M * 8 * S)))
    return dict(NTL=NTL, MSPLIT=MSPLIT, U=U, NT=NT, R=R, stages=4, ctas=4, impl=0)


def _tsmm_p(c: dict) -> tuple:
    if c.get("impl", 0) in (3, 4):
        return (c["NBW"], c["WR"], 0)
    if c.get("impl", 0) >= 1:
        return (c["WR"], c["AP"], c["NOP"])
    return (c["NTL"], c["MSPLIT"], c["U"])


def load_tune() -> dict:
    if os.path.exists(TUNE):
        with open(TUNE) as f:
            return json.load(f).get("entries", {})
    return {}


def entries():
    tune = load_tune()
    out = []
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for (M, N) in SHAPES:
                key = f"{op}_{dt}_{M}_{N}"
                out.append((op, dt, M, N, resolve(op, M, N, dt == "z", tune.get(key, {}).get("cfg"))))
    return out


def resolve(op: str, M: int, N: int, z: bool, tuned: dict | None) -> dict:
    """Default config, overridden by a tuned one; DMMA TSMTTSM configs tuned
    before padded strides existed get the conflict-free strides."""
    cfg = (tsmttsm_pick if op == "tsmttsm" else tsmm_pick)(M, N, z)
    if tuned:
        if tuned.get("impl", 0) != cfg.get("impl", 0):
            cfg = {k: v for k, v in cfg.items() if k in ("stages", "ctas")}
        cfg.update(tuned)
    if op == "tsmttsm" and cfg.get("impl", 0) >= 1 and "AP" not in cfg:
        cfg["AP"], cfg["BP"] = pick_stride(M, z, "t"), pick_stride(N, z, "t")
    return cfg


def cfg_type(op, dt, M, N, c) -> str:
    zr = "true" if c.get("ZR", 0) else "false"
    if c.get("ZR", 0):  # complex-as-real: the real kernel on the interleaved 2M x 2N view
        M, N, dt = 2 * M, 2 * N, "d"
    z = "true" if dt == "z" else "false"
    if op == "tsmttsm" and c.get("impl", 0) >= 1:
        tma = "true" if c["impl"] == 2 else "false"
        edge = c.get("EDGE", 0)
        pair = "true" if c.get("PAIR", 0) else "false"
        return (f"tsm::TsmttsmMmaCfg<{M}, {N}, {z}, {c['MT']}, {c['NTL']}, {c['NT'] // 32 - 1 - edge}, "
                f"{c['R']}, {c.get('AP', M)}, {c.get('BP', N)}, {tma}, {edge}, {pair}, {zr}, "
                f"{'true' if c.get('G3', 0) else 'false'}, {'true' if c.get('EI', 0) else 'false'}, "
                f"{'true' if c.get('LB', 0) else 'false'}, {'true' if c.get('GA', 0) else 'false'}>")
    if op == "tsmttsm":
        return f"tsm::TsmttsmCfg<{M}, {N}, {z}, {c['MT']}, {c['NTL']}, {c['NT']}, {c['R']}>"
    if c.get("impl", 0) == 4:
        ec = N % 8 if c.get("EDGE", 0) else 0
        return (f"tsm::TsmmCstbCfg<{M}, {N}, {z}, {c['NBW']}, {c['WR']}, {c['NT'] // 32 - 1}, {c['R']}, {ec}, "
                f"{'true' if c.get('GA', 0) else 'false'}>")
    if c.get("impl", 0) == 3:
        ec = N % 8 if c.get("EDGE", 0) else 0
        return (f"tsm::TsmmCstCfg<{M}, {N}, {z}, {c['NBW']}, {c['WR']}, {c['NT'] // 32 - 1}, {c['R']}, {zr}, "
                f"{ec}, {'true' if c.get('G3', 0) else 'false'}>")
    if c.get("impl", 0) >= 1:
        tma = "true" if c["impl"] == 2 else "false"
        return (f"tsm::TsmmMmaCfg<{M}, {N}, {z}, {c['WR']}, {c['NT'] // 32 - 1}, {c['R']}, "
                f"{c['AP']}, {c['NOP']}, {tma}>")
    return f"tsm::TsmmCfg<{M}, {N}, {z}, {c['NTL']}, {c['MSPLIT']}, {c['U']}, {c['NT']}, {c['R']}>"


def entry_init(op, dt, M, N, c) -> str:
    t = cfg_type(op, dt, M, N, c)
    if op == "tsmttsm":
        kn = "tsmttsm_mma_kernel" if c.get("impl", 0) >= 1 else "tsmttsm_kernel"
        fn = f"(const void*)&tsm::{kn}<{t}>"
        kind = "tsm::KIND_TSMTTSM"
    else:
        kn = {4: "tsmm_cstb_kernel", 3: "tsmm_cst_kernel", 2: "tsmm_mma_kernel", 1: "tsmm_mma_kernel"}.get(
            c.get("impl", 0), "tsmm_kernel")
        fn = f"(const void*)&tsm::{kn}<{t}>"
        kind = "tsm::KIND_TSMM"
    p = params4(op, M, N, c)
    return (f"  {{{kind}, {1 if dt == 'z' else 0}, {M}, {N}, {fn}, {c['NT']}, {c['R']}, "
            f"{p[0]}, {p[1]}, {p[2]}, {p[3]}, {c['stages']}, {c['ctas']}, {c.get('impl', 0)}, "
            f"{flags(c)}}},")


def flags(c: dict) -> int:
    """KernelEntry.edge / tsm_config.kernel >> 4: bit 0 DFMA edge warps, bit 1
    paired 16-byte fragment loads, bits 2-3 edge warps - 1 (EDGE = edge warp count),
    bit 4 complex-as-real (ZR), bit 5 3M / Gauss complex products (G3), bit 6
    plain consumer-warp order (PLAIN; a launch argument of the DMMA kernels),
    bit 7 inline edge (EI: consumer warps compute the edge strips), bit 8
    L-blocks (LB: edge strips by MMA blocks pairing edge rows with core
    columns and core rows with edge columns), bit 9 gather-capable
    instantiation (GA, strided views)."""
    e = c.get("EDGE", 0)
    return ((1 if e else 0) | (c.get("PAIR", 0) << 1) | (((e - 1) & 3) << 2 if e else 0)
            | (c.get("ZR", 0) << 4) | (c.get("G3", 0) << 5) | (c.get("PLAIN", 0) << 6)
            | (c.get("EI", 0) << 7) | (c.get("LB", 0) << 8) | (c.get("GA", 0) << 9))


def params4(op: str, M: int, N: int, c: dict) -> tuple:
    """(p0, p1, p2, p3) of the registry entry / tsm_config for a gen-style cfg."""
    if c.get("ZR", 0):
        M, N = 2 * M, 2 * N
    if op == "tsmttsm":
        if c.get("impl", 0) >= 1:
            return (c["MT"], c["NTL"], c.get("AP", M), c.get("BP", N))
        return (c["MT"], c["NTL"], 0, 0)
    return _tsmm_p(c) + (0,)


def main(per_file: int = 12) -> int:
    os.makedirs(GEN, exist_ok=True)
    ents = entries()
    files = []
    for i in range(0, len(ents), per_file):
        batch = ents[i:i + per_file]
        idx = i // per_file
        name = f"inst_{idx:03d}.cu"
        lines = ["// GENERATED by tools/gen_instances.py -- do not edit.",
                 '#include "../tsm_kernels.cuh"', '#include "../tsm_registry.h"', "",
                 f"extern const tsm::KernelEntry tsm_gen_table_{idx:03d}[] = {{"]
        lines += [entry_init(*e) for e in batch]
        lines += ["};", f"extern const int tsm_gen_count_{idx:03d} = {len(batch)};", ""]
        src = "\n".join(lines)
        path = os.path.join(GEN, name)
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        files.append(idx)
    # drop stale batch files
    for fn in os.listdir(GEN):
        if fn.startswith("inst_") and fn.endswith(".cu") and int(fn[5:8]) not in files:
            os.remove(os.path.join(GEN, fn))
    reg = ["// GENERATED by tools/gen_instances.py -- do not edit.", '#include "../tsm_registry.h"', ""]
    for idx in files:
        reg.append(f"extern const tsm::KernelEntry tsm_gen_table_{idx:03d}[];")
        reg.append(f"extern const int tsm_gen_count_{idx:03d};")
    reg.append("")
    reg.append("namespace tsm {")
    reg.append("extern const KernelTable g_gen_tables[] = {")
    for idx in files:
        reg.append(f"  {{tsm_gen_table_{idx:03d}, tsm_gen_count_{idx:03d}}},")
    reg.append("};")
    reg.append(f"extern const int g_gen_ntables = {len(files)};")
    shapes = ",".join(f"[{M},{N}]" for (M, N) in SHAPES)
    reg.append(f'const char* g_gen_info = "{{\\"aot_shapes\\":[{shapes}],\\"instances\\":{len(ents)}}}";')
    reg.append("}  // namespace tsm")
    src = "\n".join(reg) + "\n"
    _write(os.path.join(GEN, "registry_gen.cpp"), src)

    # default launch parameters for EVERY (op, dtype, M, N): the JIT path
    # instantiates these for shapes outside the AOT set.  Index:
    # ((op*2 + dt)*64 + (M-1))*64 + (N-1).
    tune = load_tune()
    lines = ["// GENERATED by tools/gen_instances.py -- do not edit.", '#include "../tsm_registry.h"',
             "", "namespace tsm {", "extern const KernelEntry g_param_table[] = {"]
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for M in range(1, 65):
                for N in range(1, 65):
                    c = resolve(op, M, N, dt == "z", tune.get(f"{op}_{dt}_{M}_{N}", {}).get("cfg"))
                    p = params4(op, M, N, c)
                    lines.append(f"  {{{0 if op == 'tsmttsm' else 1}, {1 if dt == 'z' else 0}, {M}, {N}, "
                                 f"nullptr, {c['NT']}, {c['R']}, {p[0]}, {p[1]}, {p[2]}, {p[3]}, "
                                 f"{c['stages']}, {c['ctas']}, {c.get('impl', 0)}, "
                                 f"{flags(c)}}},")
    lines += ["};", ""]
    # strided-view defaults (TSM_FLAG_STRIDED, NEXT N4): a TMA kernel, whose
    # tensor maps take any 16-byte row stride; impl -1 = no such kernel.
    lines += ["extern const KernelEntry g_param_table_strided[] = {"]
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for M in range(1, 65):
                for N in range(1, 65):
                    c = strided_default(op, M, N, dt == "z",
                                        tune.get(f"{op}_{dt}_{M}_{N}", {}).get("cfg"))
                    if c is None:
                        lines.append(f"  {{{0 if op == 'tsmttsm' else 1}, {1 if dt == 'z' else 0}, {M}, {N}, "
                                     f"nullptr, 32, 2, 0, 0, 0, 0, 2, 1, -1, 0}},")
                        continue
                    p = params4(op, M, N, c)
                    lines.append(f"  {{{0 if op == 'tsmttsm' else 1}, {1 if dt == 'z' else 0}, {M}, {N}, "
                                 f"nullptr, {c['NT']}, {c['R']}, {p[0]}, {p[1]}, {p[2]}, {p[3]}, "
                                 f"{c['stages']}, {c['ctas']}, {c.get('impl', 0)}, "
                                 f"{flags(c)}}},")
    lines += ["};", ""]
    # gather-capable defaults (TSM_FLAG_GATHER, NEXT N4): TSMTTSM kernel 1 /
    # TSMM kernel 4, any row stride
    lines += ["extern const KernelEntry g_param_table_gather[] = {"]
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for M in range(1, 65):
                for N in range(1, 65):
                    c = gather_default(op, M, N, dt == "z", tune.get(f"{op}_{dt}_{M}_{N}", {}).get("cfg"))
                    p = params4(op, M, N, c)
                    lines.append(f"  {{{0 if op == 'tsmttsm' else 1}, {1 if dt == 'z' else 0}, {M}, {N}, "
                                 f"nullptr, {c['NT']}, {c['R']}, {p[0]}, {p[1]}, {p[2]}, {p[3]}, "
                                 f"{c['stages']}, {c['ctas']}, {c.get('impl', 0)}, "
                                 f"{flags(c)}}},")
    lines += ["};", "}  // namespace tsm", ""]
    _write(os.path.join(GEN, "params_gen.cpp"), "\n".join(lines))

    # the kernel template source, embedded for NVRTC
    ksrc = open(os.path.join(os.path.dirname(GEN), "tsm_kernels.cuh")).read()
    assert ")TSMSRC\"" not in ksrc
    _write(os.path.join(GEN, "kernel_source.inc"),
           "// GENERATED by tools/gen_instances.py from csrc/tsm_kernels.cuh -- do not edit.\n"
           f"static const char* kTsmKernelSource = R\"TSMSRC({ksrc})TSMSRC\";\n")
    print(f"{len(ents)} instances in {len(files)} files")
    return 0


def _write(path: str, src: str) -> None:
    if not os.path.exists(path) or open(path).read() != src:
        with open(path, "w") as f:
            f.write(src)



# ---------------------------------------------------------------------------
# Autotuning search space (tools/autotune.py measures these on the B200).
# Compile-time parameters only; stages / ctas are run-time and swept there.
# ---------------------------------------------------------------------------
def _rows(step: int, row_bytes: int, target: int) -> int:
    return max(step, (target // row_bytes) // step * step)


def candidates(op: str, M: int, N: int, z: bool) -> list:
    S = 2 if z else 1
    row = (M + N) * 8 * S
    out = []
    if op == "tsmttsm":
        amax = 32 if z else 64
        tiles = []
        MT = 1
        while MT <= M:
            NTL = 1
            while NTL <= N:
                TM, TN = cdiv(M, MT), cdiv(N, NTL)
                TPR = MT * NTL
                if TM * TN <= amax and TPR <= 256:
                    waste = MT * TM * NTL * TN / (M * N)
                    lds = (TM + TN) / (TM * TN)
                    conflict = 0 if TPR >= 16 or TPR >= pow2floor(M) * pow2floor(N) else 1
                    tiles.append((conflict, waste * (1 + lds), MT, NTL))
                NTL *= 2
            MT *= 2
        tiles.sort()
        for (_, _, MT, NTL) in tiles[:5]:
            for NT in (128, 256):
                if NT % (MT * NTL):
                    continue
                RB = NT // (MT * NTL)
                step = RB if RB % 2 == 0 else 2 * RB
                # big stages amortise the per-chunk block barrier at narrow widths
                for tgt in ((12288, 24576, 65536) if M * N <= 16 else (12288, 24576)):
                    out.append(dict(MT=MT, NTL=NTL, NT=NT, R=_rows(step, row, tgt), impl=0))
        if min(M, N) >= 2:  # (narrow widths: fixed per-chunk cost beats the padded MMA work)
            MB, NB = cdiv(M, 8), cdiv(N, 8)
            wmax = 8 if z else 16
            wt = []
            for WM in range(1, min(MB, 8) + 1):
                for WN in range(1, min(NB, 8) + 1):
                    if WM * WN > wmax or cdiv(MB, WM) * cdiv(NB, WN) > 16:
                        continue
                    bal = cdiv(MB, WM) * WM * cdiv(NB, WN) * WN / (MB * NB)
                    wt.append((bal * (1 + 0.5 * (WM + WN) / (WM * WN)), WM, WN))
            wt.sort()
            for (_, WM, WN) in wt[:4]:
                WT = cdiv(MB, WM) * cdiv(NB, WN)
                for k in (1, 2, 4, 8):
                    NW = WT * k
                    if NW < 4 and k < 8 and WT * (k * 2) <= 16:
                        continue
                    if NW > 16:
                        break
                    pads = [False] + ([True] if min(M, N) * S * 8 >= 384 else [])
                    # big stages (64 KB, run with 2-3 stages) give each warp more
                    # k-steps per mbarrier round trip
                    for tgt in (16384, 32768, 65536):
                        for pad in pads:
                            out.append(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32,
                                            R=_rows(4 * k, row, tgt), impl=1,
                                            AP=pick_stride(M, z, "t", pad),
                                            BP=pick_stride(N, z, "t", pad)))
                        if tma_ok(M, N, z):  # 2-D TMA boxes, 128B swizzle
                            tb = (cdiv(M * S, 16) + cdiv(N * S, 16)) * 128
                            step = 4 * k if (4 * k) % 8 == 0 else 8 * k
                            Rt = min(256 // step * step, max(step, (tgt // tb) // step * step))
                            out.append(dict(MT=WM, NTL=WN, NT=(NW + 1) * 32, R=Rt, impl=2,
                                            AP=M, BP=N))
            out.extend(edge_candidates(M, N, z))
            out.extend(inline_edge_candidates(M, N, z))
            out.extend(lblock_candidates(M, N, z))
            out.extend(pair_candidates(M, N, z))
    else:
        acc_max = 16 if z else 32
        NTL = 1
        ntls = []
        while NTL <= min(N, 32):
            ntls.append(NTL)
            NTL *= 2
        for NTL in ntls[-3:]:
            TN = cdiv(N, NTL)
            MS = 1
            while NTL * MS <= 32 and MS <= M:
                us = [U for U in (2, 4, 8, 16) if U * TN <= acc_max][-2:]
                for U in us:
                    for NT in (256, 128):
                        GS = NTL * MS
                        rpp = (NT // GS) * U
                        if rpp % 2 or rpp * max(M, N) * S * 8 > 65536:
                            continue
                        R = rpp * max(1, round(16384 / (rpp * M * 8 * S)))
                        out.append(dict(NTL=NTL, MSPLIT=MS, U=U, NT=NT, R=R, impl=0))
                        break
                MS *= 2
    if op == "tsmm":
        out.extend(tsmm_cst_configs(M, N, z))
        out.extend(tsmm_cst_configs(M, N, z, edge=True))
        out.extend(tsmm_cstb_configs(M, N, z))
        out.extend(tsmm_cstb_configs(M, N, z, edge=True))
    if z:
        out.extend(zr_candidates(op, M, N))
        out.extend(g3_candidates(op, M, N, out))
    if op == "tsmm" and N >= 2:
        d = tsmm_mma_default(M, N, z)
        S_ = 2 if z else 1
        NB = cdiv(N, 8)
        for NW in (4, 8, 12, 16):
            for WR in (1, 2, 4):
                if WR * NB * 2 * S_ > 64:
                    continue
                # 12 / 16 consumer warps (3-4 per SMSP; ncu run 23: 2 per SMSP
                # leave the tensor pipe at 88 % on TSMM D 63): only with the
                # accumulators of one row block (ptxas grants 128 / 96 registers)
                if NW > 8 and WR * NB * S_ > 8:
                    continue
                rpp = 8 * WR * NW
                for tgt in (12288, 24576):
                    R = rpp * max(1, round(tgt / (rpp * d["AP"] * S_ * 8)))
                    out.append(dict(WR=WR, AP=d["AP"], NOP=d["NOP"], NT=(NW + 1) * 32, R=R, impl=1))
                    if tma_ok(M, N, z) and rpp <= 256:
                        ab = cdiv(M * S_, 16) * 128
                        Rt = rpp * max(1, min(256 // rpp, round(tgt / (rpp * ab))))
                        out.append(dict(WR=WR, AP=M, NOP=N, NT=(NW + 1) * 32, R=Rt, impl=2))
    # dedupe
    seen, uniq = set(), []
    for c in out:
        k = tuple(sorted(c.items()))
        if k not in seen:
            seen.add(k)
            uniq.append(c)
    return uniq


def strided_capable(op: str, c: dict) -> bool:
    """Kernels whose A/B rows arrive by TMA tensor maps (any 16-byte stride)."""
    return c.get("impl", 0) == 2 if op == "tsmttsm" else c.get("impl", 0) in (2, 3)


def gather_capable(op: str, c: dict) -> bool:
    """Kernels with the element-wise (cp.async) gather producer: any row stride."""
    return bool(c.get("GA")) and (c.get("impl", 0) == 1 if op == "tsmttsm" else c.get("impl", 0) == 4)


def gather_default(op: str, M: int, N: int, z: bool, tuned: dict | None) -> dict:
    """Default configuration of a TSM_FLAG_GATHER plan (every shape has one):
    the tuned configuration when it is gather-capable, else TSMTTSM kernel 1
    with the DMMA default tiles / TSMM kernel 4 (C-stationary, bulk)."""
    c = resolve(op, M, N, z, tuned)
    if (c.get("impl", 0) == 1 if op == "tsmttsm" else c.get("impl", 0) == 4):
        return dict(c, GA=1)  # the tuned configuration, gather-capable instantiation
    if op == "tsmttsm":
        d = dict(tsmttsm_mma_default(M, N, z), GA=1)
        if d["impl"] != 1:  # the TMA branch: same tiles, dense-stride stages
            S = 2 if z else 1
            WT = cdiv(cdiv(M, 8), d["MT"]) * cdiv(cdiv(N, 8), d["NTL"])
            RS = (d["NT"] // 32 - 1) // WT
            step = 4 * RS
            R = max(step, (24576 // ((M + N) * 8 * S)) // step * step)
            d.update(impl=1, R=R, AP=pick_stride(M, z, "t"), BP=pick_stride(N, z, "t"))
        return d
    cands = tsmm_cstb_configs(M, N, z)
    if cands:
        pick = [x for x in cands if x["WR"] == 2] or cands
        return dict(pick[0], stages=3, ctas=1, GA=1)
    # N = 1: one 8-column block (7 padded columns), two row groups of one warp
    S = 2 if z else 1
    R = 32 * max(1, round(16384 / (32 * M * S * 8)))
    return dict(NBW=1, WR=2, NT=3 * 32, R=R, impl=4, stages=3, ctas=1, GA=1)


def strided_default(op: str, M: int, N: int, z: bool, tuned: dict | None):
    """Default configuration of a TSM_FLAG_STRIDED plan: the tuned one when it
    is a TMA kernel, else a TMA heuristic; the gather-capable default for
    shapes without a TMA kernel."""
    c = resolve(op, M, N, z, tuned)
    if strided_capable(op, c):
        return c
    if not tma_ok(M, N, z):
        return gather_default(op, M, N, z, tuned)
    if op == "tsmttsm":
        d = tsmttsm_mma_default(M, N, z)
        return d if strided_capable(op, d) else None
    cands = tsmm_cst_configs(M, N, z)
    if not cands:
        return None
    pick = [x for x in cands if x["WR"] == 2] or cands
    return dict(pick[0], stages=3, ctas=1)


def zr_candidates(op: str, M: int, N: int) -> list:
    """Complex-as-real (ZR=1): the real DMMA kernels on the interleaved 2M x 2N
    view (A, B as real K x 2M, K x 2N).  Flops and bytes equal the complex
    kernel's; 8x8 blocks pad 2M instead of M (Z 17: 40/34 instead of 24/17)."""
    if op == "tsmttsm":
        if min(M, N) < 4:
            return []
        base = [c for c in candidates("tsmttsm", 2 * M, 2 * N, False) if c.get("impl", 0) in (1, 2)]
    else:
        if 2 * M < 16 or 2 * N < 16:
            return []
        base = tsmm_cst_configs(2 * M, 2 * N, False) + tsmm_cst_configs(2 * M, 2 * N, False, edge=True)
    return [dict(c, ZR=1) for c in base]


def g3_candidates(op: str, M: int, N: int, base: list) -> list:
    """3M / Gauss complex products (G3=1): the native complex DMMA candidates
    -- TSMTTSM kernels 1/2 (with or without edge warps), TSMM C-stationary
    kernel 3 (with or without edge columns) -- with 3 real DMMAs per 8x8
    block instead of 4.  Warp tiles keep <= 6 blocks (3 x 2 accumulator
    doubles per block and lane); TSMM C slices <= 48 doubles (MK x NBW x 3)."""
    if op == "tsmttsm":
        return [dict(c, G3=1) for c in base
                if c.get("impl", 0) in (1, 2) and not c.get("ZR", 0) and c["MT"] * c["NTL"] <= 6]
    return [dict(c, G3=1) for c in base
            if c.get("impl", 0) == 3 and not c.get("ZR", 0) and c["WR"] * c["NBW"] <= 6
            and cdiv(M, 4) * c["NBW"] * 3 <= 48]


def to_tsm_config(op: str, c: dict, stages: int, ctas: int) -> dict:
    """gen-style cfg -> tsm_config field dict (include/libtsm.h)."""
    if op == "tsmttsm" and c.get("impl", 0) >= 1:
        p = (c["MT"], c["NTL"], c["AP"], c["BP"])
    elif op == "tsmttsm":
        p = (c["MT"], c["NTL"], 0, 0)
    else:
        p = _tsmm_p(c) + (0,)
    return dict(threads=c["NT"], rows_per_chunk=c["R"], p0=p[0], p1=p[1], p2=p[2], p3=p[3],
                stages=stages, ctas_per_sm=ctas, kernel=c.get("impl", 0) | (flags(c) << 4))


# ---------------------------------------------------------------------------
# DMMA TSMM (tsm_kernels.cuh TsmmMmaCfg): smem strides chosen so m8n8k4
# fragment loads / accumulator stores use the minimum number of wavefronts.
# ---------------------------------------------------------------------------
def _degree(stride: int, z: bool, kind: str) -> float:
    """Smem wavefronts per warp access / minimum, lanes (g = l/4, q = l%4).
    8-byte accesses are served per 16-lane half-warp over 16 8-byte units,
    16-byte ones per 8-lane quarter over 8 16-byte units (measured, ncu r4:
    a pattern whose 32 lanes cover every unit exactly twice -- the former
    model's minimum -- still took 2x the ideal wavefronts when both lanes of
    a unit fell in the same half-warp)."""
    wide_o = kind == "o" and stride % 2 == 0 and not z
    wide = z or wide_o
    lanes = 8 if wide else 16
    worst = 0
    for ph in range(32 // lanes):
        counts = {}
        for lane in range(ph * lanes, ph * lanes + lanes):
            g, q = lane >> 2, lane & 3
            if kind == "a":          # TSMM A fragment: element (row g, col q)
                idx = g * stride + q
            elif kind == "t":        # TSMTTSM A/B fragment: element (row q, col g)
                idx = q * stride + g
            elif z:                  # Z output: element (g, 2q) (e = 0 store)
                idx = g * stride + 2 * q
            elif wide_o:             # D output, 16-byte store of (2q, 2q+1)
                idx = (g * stride + 2 * q) // 2
            else:                    # D output, 8-byte store
                idx = g * stride + 2 * q
            unit = idx % (8 if wide else 16)
            counts[unit] = counts.get(unit, 0) + 1
        worst = max(worst, max(counts.values()))
    return float(worst)


def pick_stride(w: int, z: bool, kind: str, pad: bool = False) -> int:
    """Conflict-minimising smem row stride for a width-w operand.  Padding
    means one bulk copy per row, which the TMA engine cannot sustain for small
    rows (r01 run 8: TSMTTSM D M=16 fell to 10 % of roofline), so the default
    layout is dense (pad=False); padded strides are autotuning candidates for
    wide rows only."""
    if not pad or (w * (2 if z else 1)) % 2:
        return w  # dense: one bulk copy per chunk (odd-width D rows cannot be padded)
    best = None
    for st in range(w, w + 9):
        if st != w and ((st * (2 if z else 1)) % 2):
            continue  # padded rows must stay 16-byte aligned (bulk copies)
        key = (_degree(st, z, kind), st)
        if best is None or key < best:
            best = key
    return best[1]


def tsmm_mma_default(M: int, N: int, z: bool) -> dict:
    S = 2 if z else 1
    MK, NB = cdiv(M, 4), cdiv(N, 8)
    AP, NOP = pick_stride(M, z, "a"), pick_stride(N, z, "o")
    NCP = 8 * NB + 4  # = tsm_kernels.cuh TsmmMmaCfg::NCP
    wr0 = max(1, min(4, 16 // (NB * S)))
    tma = tma_ok(M, N, z)
    for NW in (8, 4):
        for WR in sorted({wr0, max(1, wr0 // 2), 1}, reverse=True):
            rpp = 8 * WR * NW
            if tma:
                if rpp > 256:
                    continue
                ab, ob = cdiv(M * S, 16) * 128, cdiv(N * S, 16) * 128
                R = rpp * max(1, min(256 // rpp, round(16384 / (rpp * ab))))
                smem = 2560 + 8 * MK * 4 * NCP * S + NW * 8 * WR * ob + 3 * R * ab
                if smem <= 200 * 1024:
                    return dict(WR=WR, AP=M, NOP=N, NT=(NW + 1) * 32, R=R, stages=4, ctas=2, impl=2)
                continue
            R = rpp * max(1, round(16384 / (rpp * AP * S * 8)))
            smem = 256 + 8 * (MK * 4 * NCP * S + NW * 8 * WR * NOP * S + 3 * R * AP * S)
            if smem <= 200 * 1024:
                return dict(WR=WR, AP=AP, NOP=NOP, NT=(NW + 1) * 32, R=R, stages=4, ctas=2, impl=1)
    return dict(WR=1, AP=AP, NOP=NOP, NT=160, R=32, stages=2, ctas=1, impl=1)


def tsmm_pick(M: int, N: int, z: bool) -> dict:
    if M * N >= 32 and N >= 4:
        return tsmm_mma_default(M, N, z)
    return tsmm_default(M, N, z)


def tsmm_cst_configs(M: int, N: int, z: bool, edge: bool = False) -> list:
    """C-stationary DMMA TSMM candidates: NBW column blocks per warp such that
    the warp's C slice (MK x NBW fragments) fits in <= 48 registers-doubles.
    edge=True: the last N mod 8 columns by DFMA (EDGE=1) instead of a padded
    8-column DMMA block."""
    if not tma_ok(M, N, z):
        return []
    if edge and (N < 8 or N % 8 == 0):
        return []
    S = 2 if z else 1
    EC = N % 8 if edge else 0
    MK, NB = cdiv(M, 4), cdiv(N - EC, 8)
    out = []
    for NBW in range(1, NB + 1):
        if (NBW * 8 * S) % 16 or MK * NBW * S > 48:
            continue
        NG = cdiv(NB, NBW)
        for RG in (1, 2, 4):
            NW = NG * RG
            if NW > 16 or NW < 2:
                continue
            for WR in (1, 2, 4):
                if WR * NBW * 2 * S > 32 or WR * EC * S > 16:
                    continue
                rpp = 8 * WR * RG
                if rpp > 256:
                    continue
                ab = cdiv(M * S, 16) * 128
                for tgt in (16384, 32768):
                    R = rpp * max(1, min(256 // rpp, round(tgt / (rpp * ab))))
                    c = dict(NBW=NBW, WR=WR, NT=(NW + 1) * 32, R=R, impl=3)
                    if edge:
                        c["EDGE"] = 1
                    out.append(c)
    return out


def tsmm_cstb_configs(M: int, N: int, z: bool, edge: bool = False) -> list:
    """C-stationary DMMA TSMM with bulk copies (impl 4): the widths the TMA
    kernel 3 cannot take (rows not 16-byte multiples or < 128 bytes), and
    any width where one 8-column block per warp (NBW = 1, not possible with
    kernel 3's whole 16-double output boxes) balances better.  edge=True: the
    last N mod 8 columns by DFMA (EDGE=1) instead of a padded DMMA block."""
    if N < 2:
        return []
    if edge and (N < 8 or N % 8 == 0):
        return []
    S = 2 if z else 1
    EC = N % 8 if edge else 0
    MK, NB = cdiv(M, 4), cdiv(N - EC, 8)
    out = []
    for NBW in range(1, NB + 1):
        if MK * NBW * S > 48:
            continue
        NG = cdiv(NB, NBW)
        for RG in (1, 2, 4):
            NW = NG * RG
            if NW > 16 or NW < 2 or RG > 15:
                continue
            for WR in (1, 2, 4):
                if WR * NBW * 2 * S > 32 or WR * EC * S > 16:
                    continue
                rpp = 8 * WR * RG
                for tgt in (16384, 32768):
                    R = rpp * max(1, round(tgt / (rpp * M * S * 8)))
                    c = dict(NBW=NBW, WR=WR, NT=(NW + 1) * 32, R=R, impl=4)
                    if edge:
                        c["EDGE"] = 1
                    out.append(c)
    return out


if __name__ == "__main__":
    sys.exit(main())
