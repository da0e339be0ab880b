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
                     // edge warps - 1 (tsm_config.kernel bits 4..7)
};

// number of DFMA edge warps encoded in KernelEntry::edge
inline int edge_warps(int flags) { return (flags & 1) ? 1 + ((flags >> 2) & 3) : 0; }

struct KernelTable {
  const KernelEntry* entries;
  int count;
};

}  // namespace tsm
