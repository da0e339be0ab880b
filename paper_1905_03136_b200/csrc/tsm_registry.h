// tsm_registry.h -- table of AOT-instantiated kernels (host side).
// Entries are emitted by tools/gen_instances.py into csrc/gen/*.cu.
#pragma once

namespace tsm {

enum KernelKind { KIND_TSMTTSM = 0, KIND_TSMM = 1 };

struct KernelEntry {
  int op;   // KernelKind
  int dt;   // 0 = D, 1 = Z
  int M, N;
  const void* func;  // __global__ function (launched with cudaLaunchKernel)
  int NT;            // threads per block
  int R;             // rows per chunk
  // tile description (TSMTTSM: MT, NTL; TSMM: NTL, MSPLIT, U)
  int p0, p1, p2, p3;  // DMMA TSMTTSM: WM, WN, AP, BP; DMMA TSMM: WR, AP, NOP, -
  int stages;        // default pipeline depth
  int ctas_per_sm;   // target resident CTAs per SM (clipped by occupancy)
  int impl;          // 0 = register-tile DFMA kernel, 1 = DMMA (mma.sync m8n8k4 f64) kernel,
                     // 2 = DMMA + TMA tensor copies, 3 = C-stationary DMMA TSMM
  int edge;          // DMMA TSMTTSM flags: bit 0 = DFMA edge warps for the cells outside the
                     // 8-aligned core, bit 1 = paired 16-byte fragment loads, bits 2-3 =
                     // edge warps - 1, bit 4 = complex-as-real, bit 5 = 3M (Gauss) complex
                     // products, bit 6 = plain warp order (launch argument), bit 7 = inline
                     // edge, bit 8 = L-blocks, bit 9 = gather-capable (tsm_config.kernel bits 4..13)
};

// number of DFMA edge warps encoded in KernelEntry::edge
inline int edge_warps(int flags) { return (flags & 1) ? 1 + ((flags >> 2) & 3) : 0; }

// bit 4: complex (Z) computed by the real kernel on the interleaved view -- A, B
// as real K x 2M, K x 2N; TSMTTSM combines the 2M x 2N real product, TSMM uses
// the real 2M x 2N image of C (tsm_kernels.cuh ZR)
inline bool zr_flag(int flags) { return (flags & 16) != 0; }

// bit 5: Z TSMTTSM by the 3M (Gauss) method -- 3 real DMMAs per 8x8 block
// (T1 = Ar^T Br, T2 = Ai^T Bi, T3 = (Ar+Ai)^T (Br+Bi)) instead of 4
inline bool g3_flag(int flags) { return (flags & 32) != 0; }

// bit 7: inline edge -- the DMMA TSMTTSM consumer warps compute the cells outside
// the 8-aligned core themselves (DFMA interleaved with their DMMAs), no edge warps
inline bool ei_flag(int flags) { return (flags & 128) != 0; }

// bit 8: L-blocks (D DMMA TSMTTSM) -- the cells outside the 8-aligned core by
// MMA blocks pairing edge rows with core columns and core rows with edge
// columns (tsm_kernels.cuh LB), instead of padded blocks
inline bool lb_flag(int flags) { return (flags & 256) != 0; }

// bit 9: the gather-capable instantiation (strided views of any row stride,
// NEXT N4) of TSMTTSM kernel 1 / TSMM kernel 4
inline bool ga_flag(int flags) { return (flags & 512) != 0; }

// the real problem a complex-as-real entry runs (identity otherwise)
inline KernelEntry real_view(const KernelEntry& k) {
  KernelEntry v = k;
  if (zr_flag(k.edge)) {
    v.M = 2 * k.M;
    v.N = 2 * k.N;
    v.dt = 0;
    v.edge = k.edge & ~16;
  }
  return v;
}

struct KernelTable {
  const KernelEntry* entries;
  int count;
};

}  // namespace tsm
