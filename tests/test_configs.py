"""Host-side checks of the kernel configuration space (-m "not gpu").

* every default configuration (all 16384 (op, dtype, M, N)) and every
  autotuning candidate passes libtsm's own validation (tsm_plan_create_config
  validates before touching CUDA: valid -> TSM_ERR_CUDA on this GPU-less box,
  invalid -> TSM_ERR_INVALID_VALUE);
* the smem bank-conflict model used to pick padded strides reproduces the
  textbook cases (dense 8x8 fp64 fragment rows with stride 0 mod 16 words are
  4-way conflicted; stride 8 mod 16 is conflict-free).
"""
import ctypes
import os
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import gen_instances as gi  # noqa: E402

pytestmark = pytest.mark.skipif(torch.cuda.is_available(), reason="validation-only checks need a GPU-less box")


@pytest.fixture(scope="module")
def tsm():
    from paper_1905_03136_b200 import binding
    return binding


def _status(tsm, op, dt, M, N, cfgd):
    h = ctypes.c_void_p()
    c = tsm.TsmConfig(**cfgd)
    return tsm.lib.tsm_plan_create_config(ctypes.byref(h), tsm.OP[op], tsm.DTYPE[dt], M, N, 0,
                                          ctypes.byref(c))


def test_default_configs_valid(tsm):
    bad = []
    tune = gi.load_tune()
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            for M in range(1, 65):
                for N in range(1, 65):
                    c = gi.resolve(op, M, N, dt == "z", tune.get(f"{op}_{dt}_{M}_{N}", {}).get("cfg"))
                    st = _status(tsm, op, dt, M, N, gi.to_tsm_config(op, c, c["stages"], c["ctas"]))
                    if st != 5:
                        bad.append((op, dt, M, N, st, tsm.lib.tsm_last_error_detail()))
    assert not bad, bad[:5]


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (8, 8), (17, 33), (32, 32), (48, 16), (64, 64), (64, 1), (1, 64)])
def test_candidates_valid(tsm, shape):
    M, N = shape
    for op in ("tsmttsm", "tsmm"):
        for dt in ("d", "z"):
            cands = gi.candidates(op, M, N, dt == "z")
            assert cands, (op, dt, shape)
            for c in cands:
                st = _status(tsm, op, dt, M, N, gi.to_tsm_config(op, c, 3, 2))
                assert st == 5, (op, dt, shape, c, tsm.lib.tsm_last_error_detail())


def test_invalid_config_rejected_before_cuda(tsm):
    good = gi.to_tsm_config("tsmttsm", gi.tsmttsm_mma_default(64, 64, False), 3, 1)
    assert good["kernel"] == 2  # DMMA + TMA tensor copies
    assert _status(tsm, "tsmttsm", "d", 64, 64, good) == 5
    for k, v in [("rows_per_chunk", 30), ("rows_per_chunk", 12), ("threads", 100), ("kernel", 3)]:
        bad = dict(good, **{k: v})
        assert _status(tsm, "tsmttsm", "d", 64, 64, bad) == 1, k
    dense = dict(good, kernel=1)  # DMMA with bulk copies: p2/p3 are smem strides
    assert _status(tsm, "tsmttsm", "d", 64, 64, dense) == 5
    assert _status(tsm, "tsmttsm", "d", 64, 64, dict(dense, p2=63)) == 1
    # TMA needs 16-byte rows of >= 128 bytes
    assert _status(tsm, "tsmttsm", "d", 12, 64, dict(good, p0=1, p1=1, threads=32 * 9)) == 1
    # odd-width D rows cannot be padded (not 16-byte multiples)
    assert _status(tsm, "tsmttsm", "d", 63, 64, dict(good, p2=66)) == 1


def test_conflict_model_pins():
    # the bank model: 8-byte accesses per 16-lane half-warp over 16 units, 16-byte
    # ones per 8-lane quarter over 8 units (ncu r4, profiles/r02_ncu_run4.md: the
    # TSMM D 57 C fragment at stride 72 took 2x the ideal wavefronts although its
    # 32 lanes cover every unit exactly twice)
    assert gi._degree(72, False, "t") == 2.0  # the measured case
    assert gi._degree(68, False, "t") == 1.0  # stride 4 mod 16: conflict-free
    assert gi._degree(64, False, "t") == 4.0  # 4 rows on the same 4 units per half-warp
    assert gi.pick_stride(64, False, "t") == 64  # dense by default (one bulk copy per chunk)
    assert gi._degree(gi.pick_stride(64, False, "t", pad=True), False, "t") == 1.0
    # complex (16-byte elements): stride 0 mod 8 units -> the 4 rows of a quarter on 2 units
    assert gi._degree(64, True, "t") == 4.0
    assert gi._degree(66, True, "t") == 1.0
    # TSMM A fragment (8 rows x 4 consecutive): stride 0 mod 16 -> 4 rows per unit per half-warp
    assert gi._degree(64, False, "a") == 4.0
    assert gi._degree(gi.pick_stride(64, False, "a", pad=True), False, "a") == 1.0
    # odd widths stay dense (rows are not 16-byte multiples)
    assert gi.pick_stride(63, False, "a", pad=True) == 63 and gi.pick_stride(33, False, "t", pad=True) == 33


def _win16_row(M, i, g):  # mirror of tsm_kernels.cuh win16_row
    b, h = i & 1, g >> 2
    x = (0 if h == 0 else (M & 3)) if b == 0 else (2 if h == 0 else 4 - (M & 3))
    return 16 * (i >> 1) + 4 * (g & 3) + x


def test_win16_rows_conflict_free_for_odd_strides():
    """TSMM kernels 1 / 4 with a dense odd-width D stage and WR even: the
    16-row window map is a bijection onto the pass rows, and every half-warp
    of an A fragment load (rows of one MMA block, columns q = 0..3) hits 16
    distinct 8-byte units -- the best 8-row permutation leaves 2-way
    conflicts for every odd stride (ncu r4: TSMM D 57 / 63 loads at 2x)."""
    for M in range(9, 65, 2):
        for WR in (2, 4, 8):
            rows = sorted(_win16_row(M, i, g) for i in range(WR) for g in range(8))
            assert rows == list(range(8 * WR)), (M, WR)
            for i in range(WR):
                for ph in range(2):
                    units = {(_win16_row(M, i, g) * M + q) % 16 for g in range(4 * ph, 4 * ph + 4)
                             for q in range(4)}
                    assert len(units) == 16, (M, WR, i, ph)
        # any 8-row permutation: some half-warp stays 2-way conflicted
        import itertools
        best = min(max(len([1 for g in range(4 * ph, 4 * ph + 4) for q in range(4)]) -
                       len({(perm[g] * M + q) % 16 for g in range(4 * ph, 4 * ph + 4) for q in range(4)})
                       for ph in range(2))
                   for perm in itertools.islice(itertools.permutations(range(8)), 0, 40320, 97))
        assert best > 0, M


def _lds128_worst(addr):
    """Max lanes on one 16-byte bank group within an LDS.128 phase (8 lanes)."""
    worst = 0
    for ph in range(4):
        cnt = {}
        for lane in range(8 * ph, 8 * ph + 8):
            gran = (addr(lane >> 2, lane & 3) * 8 // 16) % 8
            cnt[gran] = cnt.get(gran, 0) + 1
        worst = max(worst, max(cnt.values()))
    return worst


def test_pair_layouts_conflict_free():
    # padded dense strides: rows 32 B apart modulo 128 -> one granule per lane
    for w in (16, 20, 32, 40, 48, 56, 64):
        st = gi.pair_stride(w)
        assert st >= w and st % 2 == 0
        assert _lds128_worst(lambda g, q: q * st + 2 * g) == 1, w
    assert _lds128_worst(lambda g, q: q * 64 + 2 * g) == 4  # dense stride 64: 4-way

    # 128B swizzle (TMA boxes): granule (c/2 ^ row).  Contiguous k-step rows
    # conflict 2-way; the kernel's row remap (k0 & ~7) + (k0/4 % 2) + 2q is
    # conflict-free for paired D (LDS.128), plain D (LDS.64) and Z (LDS.128)
    def swz(r, c):
        return r * 16 + ((((c >> 1) ^ r) & 7) << 1) + (c & 1)

    def remap(k0, q):
        return (k0 & ~7) + ((k0 >> 2) & 1) + 2 * q

    def worst64(addr):  # LDS.64: two 16-lane phases, 8-byte units
        w = 0
        for h in range(2):
            cnt = {}
            for lane in range(16 * h, 16 * h + 16):
                u = addr(lane >> 2, lane & 3) % 16
                cnt[u] = cnt.get(u, 0) + 1
            w = max(w, max(cnt.values()))
        return w

    for k0 in range(0, 32, 4):
        for m0 in (0, 8, 16, 24):
            assert _lds128_worst(lambda g, q: swz(k0 + q, (2 * m0 + 2 * g) % 16)) == 2
            assert _lds128_worst(lambda g, q: swz(remap(k0, q), (2 * m0 + 2 * g) % 16)) == 1
            assert worst64(lambda g, q: swz(k0 + q, (m0 + g) % 16)) == 2
            assert worst64(lambda g, q: swz(remap(k0, q), (m0 + g) % 16)) == 1
            assert _lds128_worst(lambda g, q: swz(k0 + q, (2 * (m0 + g)) % 16)) == 2  # Z
            assert _lds128_worst(lambda g, q: swz(remap(k0, q), (2 * (m0 + g)) % 16)) == 1
    # the remap visits every row of an 8-row atom once per two k-steps
    assert sorted(remap(k0, q) for k0 in (0, 4) for q in range(4)) == list(range(8))


def test_cstationary_row_permutation_conflict_free():
    # C-stationary TSMM: MMA row g <-> A/B row rho(g) under the 128B swizzle
    def swz(r, c):
        return r * 16 + ((((c >> 1) ^ r) & 7) << 1) + (c & 1)

    def worst(addr, lanes_per, unit):
        w = 0
        for ph in range(32 // lanes_per):
            cnt = {}
            for lane in range(lanes_per * ph, lanes_per * ph + lanes_per):
                u = unit(addr(lane >> 2, lane & 3))
                cnt[u] = cnt.get(u, 0) + 1
            w = max(w, max(cnt.values()))
        return w

    rho = [0, 5, 2, 7, 1, 4, 3, 6]  # tsm_kernels.cuh tsmm_cst_kernel
    assert sorted(rho) == list(range(8))
    u8, u16 = (lambda d: d % 16), (lambda d: (d // 2) % 8)
    checks = [(lambda p, g, q, ks: swz(p[g], (4 * ks + q) & 15), 16, u8, 16),       # D A loads
              (lambda p, g, q, j: swz(p[g], (8 * j + 2 * q) & 15), 8, u16, 2),      # D stores
              (lambda p, g, q, ks: swz(p[g], (2 * (4 * ks + q)) & 15), 8, u16, 8),  # Z A loads
              (lambda p, g, q, c: swz(p[g], (2 * (8 * (c >> 1) + 2 * q + (c & 1))) & 15), 8, u16, 4)]
    ident = list(range(8))
    got_id, got_rho = [], []
    for f, lp, u, nv in checks:
        got_id.append(max(worst(lambda g, q: f(ident, g, q, v), lp, u) for v in range(nv)))
        got_rho.append(max(worst(lambda g, q: f(rho, g, q, v), lp, u) for v in range(nv)))
    assert got_id == [2, 2, 2, 1] and got_rho == [1, 1, 1, 1]


def test_dense_kstep_row_spacing():
    """Dense (bulk-copy) layouts: k-step rows d apart (tsm_kernels.cuh
    pick_kdist) -- odd strides need d = 4, strides = 2 mod 4 need d = 2,
    strides = 4 mod 8 are conflict-free contiguously, 0 mod 8 never."""
    def lds64(st, d):
        w = 0
        for h in range(2):
            cnt = {}
            for lane in range(16 * h, 16 * h + 16):
                u = (d * (lane & 3) * st + (lane >> 2)) % 16
                cnt[u] = cnt.get(u, 0) + 1
            w = max(w, max(cnt.values()))
        return w

    for st in range(8, 72):
        best = min(lds64(st, d) for d in (1, 2, 4))
        if st % 2:
            assert lds64(st, 4) == 1 and lds64(st, 1) >= 2, st
        elif st % 4 == 2:
            assert lds64(st, 2) == 1, st
        elif st % 8 == 4:
            assert lds64(st, 1) == 1, st
        else:
            assert best >= 2, st


def test_cstb_row_permutation_loads_and_stores():
    """Bulk C-stationary TSMM (kernel 4, dense stride-M stage, dense [RW][N]
    output staging): the permutation chosen by tsm_kernels.cuh
    cstb_pick_rho (3 x load conflicts + store conflicts) is never worse than
    the load-only choice it replaced, and for odd widths (the D shapes that
    need kernel 4) both accesses stay at the 2-way minimum an odd stride
    allows -- the load-only choice left the D 63 stores 4-way (ncu r32)."""
    def rho(sel, g):
        return [g, ((g & 3) << 1) | (g >> 2), ((g & 1) << 2) | (g >> 1),
                ((g & 1) << 2) | (g & 2) | (g >> 2)][sel]

    def worst(unit):
        w = 0
        for ph in range(2):
            cnt = {}
            for lane in range(16 * ph, 16 * ph + 16):
                u = unit(lane >> 2, lane & 3) % 16
                cnt[u] = cnt.get(u, 0) + 1
            w = max(w, max(cnt.values()))
        return w

    def load(sel, M):
        return worst(lambda g, q: rho(sel, g) * M + q)

    def store(sel, N):
        return max(worst(lambda g, q: rho(sel, g) * N + 2 * q + e) for e in (0, 1))

    def pick(M, N):  # mirror of cstb_pick_rho (D)
        return min(range(4), key=lambda s: (3 * load(s, M) + store(s, N), s))

    def pick_old(M):  # the load-only rule
        best = 0
        for s in range(1, 4):
            if load(s, M) < load(best, M):
                best = s
        return best

    for w in range(9, 65):
        new, old = pick(w, w), pick_old(w)
        assert 3 * load(new, w) + store(new, w) <= 3 * load(old, w) + store(old, w), w
        if w % 2:
            assert load(new, w) == 2 and store(new, w) == 2, (w, new)
    assert store(pick_old(63), 63) == 4 and store(pick(63, 63), 63) == 2


def test_flag_encoding_and_new_candidates():
    """tsm_config.kernel flag bits written by the generator (include/libtsm.h):
    3M 512, plain warp order 1024, inline edge 2048; inline-edge candidates
    exist only for widths with an edge and carry no edge warps; 3M
    candidates only for Z."""
    base = dict(MT=2, NTL=2, NT=160, R=64, impl=2, AP=32, BP=32)
    assert gi.to_tsm_config("tsmttsm", dict(base, G3=1), 3, 1)["kernel"] == 2 | 512
    assert gi.to_tsm_config("tsmttsm", dict(base, PLAIN=1), 3, 1)["kernel"] == 2 | 1024
    assert gi.to_tsm_config("tsmttsm", dict(base, EI=1), 3, 1)["kernel"] == 2 | 2048
    assert not [c for c in gi.candidates("tsmttsm", 32, 32, False) if c.get("EI")]
    ei = [c for c in gi.candidates("tsmttsm", 41, 41, False) if c.get("EI")]
    assert ei and all("EDGE" not in c for c in ei)
    assert not [c for c in gi.candidates("tsmttsm", 32, 32, False) if c.get("G3")]
    assert [c for c in gi.candidates("tsmttsm", 32, 32, True) if c.get("G3")]
    assert [c for c in gi.candidates("tsmm", 32, 32, True) if c.get("G3")]


def _lblock_cells(M, N, WT=1):
    """Mirror of tsm_kernels.cuh L-blocks: the cells each L-block's epilogue
    writes (MMA row g, columns 2q + e) and the A / B columns its fragments read."""
    MR, NR = M % 8, N % 8
    MC, NC = M - MR, N - NR
    NL = max(-(-MC // (8 - MR)), -(-NC // (8 - NR)))
    writes = []
    for l in range(NL):
        for g in range(8):
            for j in range(8):
                if g < MR:
                    m = MC + g
                    n = (NC + j if l == 0 else -1) if j < NR else l * (8 - NR) + (j - NR)
                    if n >= NC and j >= NR:
                        n = -1
                elif j < NR:
                    m = l * (8 - MR) + (g - MR)
                    n = NC + j if m < MC else -1
                else:
                    n = -1
                if n >= 0:
                    writes.append((m, n))
    return NL, writes


def test_lblock_mapping_covers_every_edge_cell_once():
    """L-blocks (kernel | 4096): for every M, N >= 8 with 1..6 edge rows and
    columns, the blocks' epilogues write every cell outside the 8-aligned core
    exactly once and no core cell; the block count matches the kernel's NL and
    the generator only offers them where they need fewer MMA blocks than
    padding."""
    for M in range(9, 65):
        for N in range(9, 65):
            MR, NR = M % 8, N % 8
            if not (1 <= MR <= 6 and 1 <= NR <= 6):
                continue
            NL, writes = _lblock_cells(M, N)
            MC, NC = M - MR, N - NR
            edge = {(m, n) for m in range(M) for n in range(N) if m >= MC or n >= NC}
            assert len(writes) == len(set(writes)), (M, N)
            assert set(writes) == edge, (M, N)
            pays = (MC // 8) * (NC // 8) + NL < -(-M // 8) * -(-N // 8)
            offered = bool([c for c in gi.lblock_candidates(M, N, False)])
            assert offered == (pays and bool(gi.inline_edge_candidates(M, N, False))), (M, N)


def test_gather_defaults_exist_for_every_shape():
    """TSM_FLAG_GATHER: every (op, dtype, M, N) has a gather-capable default
    (TSMTTSM kernel 1 / TSMM kernel 4 with the GA flag), and TSM_FLAG_STRIDED
    falls back to it wherever the shape has no TMA kernel."""
    for op in ("tsmttsm", "tsmm"):
        for z in (False, True):
            for (M, N) in [(1, 1), (1, 64), (64, 1), (3, 5), (7, 9), (33, 33), (57, 57), (64, 64), (16, 48)]:
                c = gi.gather_default(op, M, N, z, None)
                assert c.get("GA") == 1 and gi.gather_capable(op, c), (op, z, M, N, c)
                s = gi.strided_default(op, M, N, z, None)
                assert s is not None and (gi.strided_capable(op, s) or gi.gather_capable(op, s)), (op, z, M, N)
