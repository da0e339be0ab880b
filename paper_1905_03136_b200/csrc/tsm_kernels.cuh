// tsm_kernels.cuh -- libtsm device code for sm_100a (B200).
//
// Width-specialised kernel templates, instantiated per (M, N, type) and tile
// configuration by csrc/gen/ (generated from tune/b200.json).
//
//   tsmttsm_kernel  C = A^T B
//   tsmm_kernel     B = A C
//
// Design (DESIGN.md §4 has the roofline for each):
//  * Persistent grid, grid-stride over CONTIGUOUS row chunks (the paper's grid
//    stride loop, at chunk granularity).  A chunk of R rows
//    of a row-major K x M matrix is one contiguous R*M*s byte range, so it is
//    moved with ONE cp.async.bulk (TMA bulk copy, SASS UBLKCP) into a
//    multi-stage shared-memory ring completed on mbarriers.  This is the
//    B200 replacement of the paper's leap frogging: the
//    next chunks are in flight while the current one is consumed, with no
//    registers spent on staging.  R is even, so chunk sizes are multiples of
//    16 B even for odd widths (the paper's misalignment hurdle,
//    PAPER.md:1100-1108); a single odd last row is handled from global.
//  * TSMTTSM: each thread owns an interleaved ("transposed")
//    register tile of TM x TN cells of C (Listing 5), with
//    MT x NTL tiles per row (powers of two).  Threads of a warp work on the
//    same row(s) so shared-memory reads are broadcasts / contiguous.
//    Thread-local sums -> warp butterfly -> fixed-order block sum in smem ->
//    per-block partial in the workspace -> the last NFIN blocks to finish
//    (ticket counter) sum the partials in fixed block order (T3/T4).  No
//    floating-point atomics: results are deterministic.
//  * TSMM: C is staged in smem once per persistent block;
//    each thread computes TN interleaved columns of U rows
//    (K-unroll with C reuse), optionally splitting the M
//    reduction over MSPLIT lanes (butterfly-combined).  Output rows are
//    staged in smem and written with cp.async.bulk stores: every B byte is
//    written once, in full sectors, with no write-allocate (S4).
//
// This file has NO dependency on the oracle (oracle/) or on any host header
// besides the CUDA toolkit built-ins, so the same source can also be compiled
// at run time by NVRTC for shapes outside the AOT set.
#pragma once

#ifndef TSM_NVRTC
#include <cstdint>
#endif

namespace tsm {

typedef unsigned long long u64;
typedef unsigned int u32;

// --------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk async copies, proxy fences.
// --------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return static_cast<u32>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TSM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TSM_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Global -> shared bulk copy completing `bytes` transaction bytes on `bar`.
// Streaming data: evict-first L2 policy (each byte is read exactly once).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar,
                                         u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ u64 policy_evict_first() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Shared -> global bulk store (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// Shared -> global bulk reduce-add (f64, round-to-nearest; bulk-group completion):
// dst[i] += src[i], done by the memory system (TSMM update with beta = 1).
__device__ __forceinline__ void bulk_red_add(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// Strided row views without TMA (NEXT N4, "gather" mode): one element per lane
// per instruction, asynchronous (Ampere-style cp.async, 8 bytes D / 16 bytes Z);
// completion is tracked by the stage's mbarrier through
// cp.async.mbarrier.arrive.noinc (one arrival per producer lane).
template <int BYTES>
__device__ __forceinline__ void cp_async_el(void* dst, const void* src) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(u64* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// rows x W elements (S doubles each) of a row-strided global matrix (row stride
// ld elements, first row r0) -> shared rows of stride sp elements; lanes of one
// warp split the elements.
template <int W, int S>
__device__ __forceinline__ void gather_rows(double* dst, int sp, const double* src, long long r0, long long ld,
                                            int rows, int lane) {
  for (int i = lane; i < rows * W; i += 32) {
    const int r = i / W, c = i - r * W;
    cp_async_el<8 * S>(dst + (r * sp + c) * S, src + ((r0 + r) * ld + c) * S);
  }
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ u32 ld_acquire_gpu(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// NEXT N3: the TSMTTSM grid
// reduction fused with the cross-GPU sum over peer memory (CUDA IPC mappings
// of every rank's slot buffer, NVLink P2P stores).  Slot buffer of a rank:
//   [0, 256) bytes   header: u64 cnt[2] (arrivals per parity) at 0, u32 err at 16,
//                    u64 seq[2 parities][kMaxPeers ranks] at 32 (call number + 1 of
//                    the data in each slot, written by the slot's source rank)
//   [256, ...)       double slot[2 parities][kMaxPeers ranks][kPeerCells]
// Each rank's finishers store their cells of the local C into slot[par][rank]
// of EVERY rank; the last finisher then adds 1 to every rank's cnt[par]
// (system-scope atomics after a system fence); every finisher waits for
// cnt[par] >= target and sums the nranks slots in rank order into C -- C is
// replicated and bitwise identical to the deterministic allgather + rank-order
// sum.  Parities alternate per call: a rank can only reuse a parity after every
// rank has finished the call before (it needed their arrivals), so a slot is
// never overwritten while it is read.  A bounded wait (timeout_ns, default 2 s)
// sets err and leaves C = NaN instead of hanging the GPU.  Every reader also
// checks each slot's sequence number against this call's, so data from another
// call (a rank that timed out and ran ahead) is reported, never summed; and once
// err is set every later call on that rank fails fast (C = NaN, no stores to
// peers, no arrivals) until tsm_peer_reset.  The parity / target / sequence are
// launch arguments, so a captured CUDA graph cannot replay a fused call.
constexpr int kMaxPeers = 8;
constexpr int kPeerCells = 64 * 64 * 2;
constexpr int kPeerHeaderBytes = 256;
struct PeerArgs {
  double* base[kMaxPeers];  // slot buffers of every rank (this rank's own at [rank])
  int nranks;               // 0: no peer reduction (C is the local result)
  int rank;
  int parity;
  u64 target;               // cnt[parity] value that means "all ranks arrived"
  u64 seq;                  // this call's number + 1 (stored beside the slot data)
  u64 timeout_ns;           // bounded wait for the other ranks
};
constexpr int kPeerErrOffset = 16;  // u32 err flag (bytes into the header)
constexpr int kPeerSeqOffset = 32;  // u64 seq[2][kMaxPeers]
__device__ __forceinline__ u64* peer_seq(const PeerArgs& q, int owner, int src) {
  return reinterpret_cast<u64*>(reinterpret_cast<char*>(q.base[owner]) + kPeerSeqOffset) +
         q.parity * kMaxPeers + src;
}
__device__ __forceinline__ u32* peer_err(const PeerArgs& q) {
  return reinterpret_cast<u32*>(reinterpret_cast<char*>(q.base[q.rank]) + kPeerErrOffset);
}
__device__ __forceinline__ u32 ld_acquire_sys32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double* peer_slot(const PeerArgs& q, int owner, int src) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(q.base[owner]) + kPeerHeaderBytes) +
         (static_cast<long long>(q.parity) * kMaxPeers + src) * kPeerCells;
}

// Complex multiply-add on (re, im) accumulators, plain (non-conjugating):
//   re += ar*br - ai*bi ; im += ar*bi + ai*br   (4 DFMA, 8 flops)
__device__ __forceinline__ void zfma(double& re, double& im, double ar, double ai, double br,
                                     double bi) {
  re = fma(ar, br, re);
  re = fma(-ai, bi, re);
  im = fma(ar, bi, im);
  im = fma(ai, br, im);
}

// Position in the smem ring: stage index s, mbarrier phase parity ph of that
// stage's current use, and how many times the ring wrapped (incremental, so
// the hot loops carry no integer division by the run-time stage count).
// Spread the warps of one tile (or column group) over the 4 SM sub-partitions.
// Warp w runs on SMSP w % 4; with the plain order tile = w % T, T a multiple of
// 4 puts every warp of a tile on one SMSP, so a partial tile leaves that SMSP's
// tensor pipe half idle (ncu r23: D 56, tiles of 14/14/14/7 DMMAs, 82 % pipe).
// Ordering the (slot, tile) pairs by L(w) = (w % 4) * (nw / 4) + w / 4 gives each
// SMSP consecutive pairs, i.e. all tiles.  A bijection on [0, nw) for nw % 4 == 0.
// order = 1 (plan flag kernel | 1024) keeps the plain order: which one balances
// better depends on the tile shape, so the autotuner measures both.
__device__ __forceinline__ int spread_warp(int w, int nw, int order) {
  return (order == 0 && nw % 4 == 0 && w < nw) ? (w % 4) * (nw / 4) + w / 4 : w;
}

// compile-time int as a value (dispatching generic lambdas on a constant)
template <int V>
struct IC {
  static constexpr int value = V;
};

struct Ring {
  int s = 0;
  u32 ph = 0;
  int round = 0;
  __device__ __forceinline__ void next(int stages) {
    if (++s == stages) {
      s = 0;
      ph ^= 1u;
      round++;
    }
  }
};

// Workspace layout shared by host and device code.
struct WsLayout {
  static constexpr int kCounterBytes = 256;  // u32 ticket, u32 done, padding
};

// 16-row windows (D, odd dense A stride M, WR even): MMA block i of a warp's
// pass and lane row g -> pass row.  Blocks 2t, 2t+1 share rows [16t, 16t+16);
// half-warp h = g >> 2 of block b takes the 4 rows w = 4p + x(b, h), p = g & 3,
// with x(0,0) = 0, x(0,1) = M mod 4, x(1,0) = 2, x(1,1) = 4 - M mod 4.  The
// rows of one half-warp are then a coset M w = c (mod 4), so its 16 LDS.64 of
// the A fragment (columns q = 0..3) hit 16 distinct 8-byte units -- an 8-row
// block cannot do better than 2-way for an odd stride (ncu r4: TSMM D 57 / 63
// A loads at 2x the ideal wavefronts).
__device__ __forceinline__ constexpr int win16_row(int M, int i, int g) {
  const int b = i & 1, h = g >> 2;
  const int x = b == 0 ? (h == 0 ? 0 : (M & 3)) : (h == 0 ? 2 : 4 - (M & 3));
  return 16 * (i >> 1) + 4 * (g & 3) + x;
}

// --------------------------------------------------------------------------
// TMA tensor copies (cp.async.bulk.tensor.2d, SASS UTMALDG / UTMASTG).
// A row-major K x W (doubles) operand is described by a 2-D tensor map
// (host: cuTensorMapEncodeTiled) with 16-double (128-byte) boxes of R rows and
// the 128-byte swizzle: inside each 1024-byte atom the 16-byte chunk c of row
// r lands at chunk c ^ (r & 7), so the column-wise fragment reads of the
// DMMA kernels hit the minimum number of smem wavefronts.  Rows beyond K are
// zero-filled by the TMA unit (no tail code).
// --------------------------------------------------------------------------
struct alignas(64) TmaDesc {
  unsigned long long raw[16];  // CUtensorMap (opaque, 128 bytes)
};
__device__ __forceinline__ void tma_load_2d(void* dst, const TmaDesc* desc, int x, int y, u64* bar,
                                            u64 policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const TmaDesc* desc, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   desc),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
// Tensor reduce-add of a box (element type from the tensor map: f64).
__device__ __forceinline__ void tma_red_add_2d(const TmaDesc* desc, int x, int y, const void* src) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   desc),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
// x with its sign bit XORed with mask (0 or 1<<63): conjugation on the integer
// pipe, exact, NaN-preserving.
__device__ __forceinline__ double flip_sign(double x, u64 mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ static_cast<long long>(mask));
}
// Byte offset o' >= o such that base + o' is 1024-byte aligned in the shared
// window (computed from the shared address, applied as pointer arithmetic).
__device__ __forceinline__ int align1024(const void* base, int o) {
  const u32 a = smem_u32(base) + static_cast<u32>(o);
  return o + static_cast<int>((1024u - (a & 1023u)) & 1023u);
}
// offset (doubles) of element (r, c), c < 16, inside a 128B-swizzled box region
__device__ __forceinline__ int swz128(int r, int c) {
  return r * 16 + ((((c >> 1) ^ r) & 7) << 1) + (c & 1);
}

// ==========================================================================
// TSMTTSM
// ==========================================================================
struct TsmttsmArgs {
  TmaDesc tmA, tmB;    // tensor maps (TMA kernels only)
  const double* A;     // K x M (x2 doubles for Z), row-major
  const double* B;     // K x N
  double* C;           // M x N
  double* partials;    // gridDim.x x (M*N*S) doubles
  u32* counters;       // [0] ticket, [1] done
  long long K;         // rows
  long long nchunks;   // ceil(K_even / R)  (TMA kernels: ceil(K / R))
  int stages;          // smem ring depth
  int nfin;            // finisher blocks of the grid reduction
  int order;           // consumer-warp order (spread_warp)
  u64 conj;            // Z: sign mask XORed into Im(A) -- 1<<63 gives C = A^H B (NEXT N2)
  PeerArgs peer;       // NEXT N3: fused cross-GPU reduction (peer.nranks == 0: off)
  long long lda, ldb;  // row strides (elements) of A and B (= M, N when dense)
  int gather;          // DMMA bulk kernel: strided rows copied element-wise (NEXT N4)
};

// M, N: widths.  Z: complex.  MT, NTL: tiles per row along m / n (powers of
// two).  NT: threads per block.  R: rows per chunk (even).
template <int M_, int N_, bool Z_, int MT_, int NTL_, int NT_, int R_>
struct TsmttsmCfg {
  static constexpr int M = M_, N = N_, MT = MT_, NTL = NTL_, NT = NT_, R = R_;
  static constexpr bool Z = Z_;
  static constexpr int S = Z ? 2 : 1;  // doubles per element
  static constexpr int TM = (M + MT - 1) / MT;
  static constexpr int TN = (N + NTL - 1) / NTL;
  static constexpr int TPR = MT * NTL;  // threads per row
  static constexpr int RB = NT / TPR;   // row slots per block
  static constexpr int CELLS = M * N * S;
  static constexpr int STAGE_DOUBLES = R * (M + N) * S;
  static_assert(NT % 32 == 0 && NT % TPR == 0, "TPR must divide NT");
  static_assert((TPR & (TPR - 1)) == 0, "TPR must be a power of two");
  static_assert(R % 2 == 0, "R must be even (16-byte bulk copies)");
  static_assert(TM * MT >= M && TN * NTL >= N, "tiles must cover C");
  static_assert(MT <= M || M == 0, "no empty tiles along m");
  static_assert(NTL <= N || N == 0, "no empty tiles along n");
};

template <class Cfg>
__device__ __forceinline__ void tsmttsm_row(const double* __restrict__ ar,
                                            const double* __restrict__ br, int tm, int tn,
                                            double (&c)[Cfg::TM][Cfg::TN][Cfg::S], u64 conj) {
  constexpr int TM = Cfg::TM, TN = Cfg::TN, MT = Cfg::MT, NTL = Cfg::NTL;
  constexpr int M = Cfg::M, N = Cfg::N;
  if constexpr (!Cfg::Z) {
    double a[TM], b[TN];
#pragma unroll
    for (int i = 0; i < TM; i++) {
      const int m = tm + i * MT;
      if ((i + 1) * MT <= M)
        a[i] = ar[m];
      else
        a[i] = (m < M) ? ar[m] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int n = tn + j * NTL;
      if ((j + 1) * NTL <= N)
        b[j] = br[n];
      else
        b[j] = (n < N) ? br[n] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) c[i][j][0] = fma(a[i], b[j], c[i][j][0]);
  } else {
    const double2* ar2 = reinterpret_cast<const double2*>(ar);
    const double2* br2 = reinterpret_cast<const double2*>(br);
    double2 a[TM], b[TN];
#pragma unroll
    for (int i = 0; i < TM; i++) {
      const int m = tm + i * MT;
      if ((i + 1) * MT <= M)
        a[i] = ar2[m];
      else
        a[i] = (m < M) ? ar2[m] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int n = tn + j * NTL;
      if ((j + 1) * NTL <= N)
        b[j] = br2[n];
      else
        b[j] = (n < N) ? br2[n] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < TM; i++) a[i].y = flip_sign(a[i].y, conj);
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++)
        zfma(c[i][j][0], c[i][j][1], a[i].x, a[i].y, b[j].x, b[j].y);
  }
}

// T3 -> T4: write this block's M x N partial (in smem sP) to the workspace,
// take a ticket; the last NFIN blocks to arrive sum all partials in fixed
// block order (each cell by one thread, its g-range split into fixed
// contiguous segments combined in segment order).  No floating-point atomics.
template <int NT, int CELLS>
__device__ __forceinline__ void grid_reduce(const TsmttsmArgs& p, const double* sP, double* scratch) {
  __shared__ u32 s_ticket;
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  double* myP = p.partials + static_cast<long long>(blockIdx.x) * CELLS;
  for (int idx = tid; idx < CELLS; idx += NT) __stcg(&myP[idx], sP[idx]);
  // nfin == 0: the reduction-overhead baseline (TSM_FLAG_NO_GRID_REDUCE,
  // PAPER.md:1000-1016 "a kernel without a global reduction"): partials only
  if (p.nfin == 0) return;

  // ---- T4: deterministic grid reduction by the last NFIN blocks ----
  __threadfence();
  __syncthreads();
  if (tid == 0) s_ticket = atomicAdd(&p.counters[0], 1u);
  __syncthreads();
  const int nfin = p.nfin;
  const int t = static_cast<int>(s_ticket);
  if (t < G - nfin) return;
  const int f = t - (G - nfin);
  const PeerArgs& pq = p.peer;
  // A single finisher (nfin == 1) holds ticket G-1: every block has published
  // its partial already (fence before its ticket), so it needs no wait -- an
  // acquire fence orders its partial reads after the ticket.
  const bool solo = nfin == 1 && pq.nranks == 0;
  if (tid == 0) {
    if (solo)
      __threadfence();
    else
      while (ld_acquire_gpu(&p.counters[0]) < static_cast<u32>(G)) __nanosleep(64);
  }
  __syncthreads();
  // finisher f owns cells [c0, c1); TPC threads per cell split the block
  // range into contiguous segments, combined afterwards in segment order.
  // N3 fail-fast: an earlier fused call on this rank timed out or saw a foreign
  // sequence number -> no stores to peers, no arrivals, C = NaN (tsm_peer_reset)
  __shared__ int s_failed;
  if (pq.nranks > 0) {
    if (tid == 0) s_failed = ld_acquire_sys32(peer_err(pq)) != 0u;
    __syncthreads();
  }
  const bool failed = pq.nranks > 0 && s_failed;
  // local C cell -> C (single GPU), or -> slot[parity][rank] of every rank (N3)
  auto put = [&](int idx, double v) {
    if (pq.nranks == 0) {
      p.C[idx] = v;
    } else if (!failed) {
      for (int r = 0; r < pq.nranks; r++) __stcg(peer_slot(pq, r, pq.rank) + idx, v);
    }
  };
  const int cpf = (CELLS + nfin - 1) / nfin;
  const int c0 = f * cpf;
  const int c1 = (c0 + cpf < CELLS) ? c0 + cpf : CELLS;
  const int ncell = c1 - c0;
  if (ncell > 0) {
    int tpc = NT / ncell;
    if (tpc < 1) tpc = 1;
    if (tpc > 32) tpc = 32;
    double* sSeg = scratch;  // [tpc][ncell] when tpc > 1
    const int seg = tid / ncell;
    const int cl = tid % ncell;
    if (tpc == 1) {
      for (int idx = c0 + tid; idx < c1; idx += NT) {
        double s0 = 0.0;
#pragma unroll 8
        for (int g = 0; g < G; g++) s0 += __ldcg(&p.partials[static_cast<long long>(g) * CELLS + idx]);
        put(idx, s0);
      }
    } else {
      if (seg < tpc) {
        const int g0 = static_cast<int>((static_cast<long long>(G) * seg) / tpc);
        const int g1 = static_cast<int>((static_cast<long long>(G) * (seg + 1)) / tpc);
        double s0 = 0.0;
#pragma unroll 8
        for (int g = g0; g < g1; g++)
          s0 += __ldcg(&p.partials[static_cast<long long>(g) * CELLS + c0 + cl]);
        sSeg[seg * ncell + cl] = s0;
      }
      __syncthreads();
      if (tid < ncell) {
        double s0 = sSeg[tid];
        for (int q = 1; q < tpc; q++) s0 += sSeg[q * ncell + tid];
        put(c0 + tid, s0);
      }
    }
  }
  if (solo) {
    // reset for the next call: no other block touches the counters again in
    // this launch, and the launch boundary orders the store before the next one
    if (tid == 0) p.counters[0] = 0;
    return;
  }
  // (single GPU: C needs no fence -- the launch boundary publishes it; the
  // counter reset only has to follow every finisher's wait, which the
  // counters[1] atomics order)
  __syncthreads();
  if (tid == 0) {
    // N3: one system-scope fence per block after the CTA barrier (cumulative over
    // the block's peer stores) instead of one per thread
    if (pq.nranks > 0) __threadfence_system();
    const u32 d = atomicAdd(&p.counters[1], 1u);
    if (d == static_cast<u32>(nfin - 1)) {  // last finisher: reset for the next call
      p.counters[0] = 0;
      p.counters[1] = 0;
      if (pq.nranks > 0 && !failed) {  // every finisher of this rank has stored (and fenced): signal
        __threadfence_system();
        for (int r = 0; r < pq.nranks; r++) *reinterpret_cast<volatile u64*>(peer_seq(pq, r, pq.rank)) = pq.seq;
        __threadfence_system();
        for (int r = 0; r < pq.nranks; r++)
          atomicAdd_system(reinterpret_cast<unsigned long long*>(pq.base[r]) + pq.parity, 1ull);
      }
    }
  }
  if (pq.nranks == 0) return;
  // ---- N3: wait for every rank's cells, then the rank-order sum of this finisher's cells ----
  __shared__ int s_ok;
  if (tid == 0) {
    const u64* cnt = reinterpret_cast<const u64*>(pq.base[pq.rank]) + pq.parity;
    const u64 t0 = globaltimer_ns();
    int ok = failed ? 0 : 1;
    while (ok && ld_acquire_sys(cnt) < pq.target) {
      __nanosleep(128);
      if (globaltimer_ns() - t0 > pq.timeout_ns) {  // a rank never arrived: report, do not hang
        atomicExch(peer_err(pq), 1u);
        ok = 0;
      }
    }
    // every slot must hold THIS call's data (a rank that ran ahead after a
    // timeout would otherwise be summed silently)
    for (int r = 0; ok && r < pq.nranks; r++)
      if (ld_acquire_sys(peer_seq(pq, pq.rank, r)) != pq.seq) {
        atomicExch(peer_err(pq), 1u);
        ok = 0;
      }
    s_ok = ok;
  }
  __syncthreads();
  for (int idx = c0 + tid; idx < c1; idx += NT) {
    double v = __longlong_as_double(0x7ff8000000000000ll);  // NaN if the wait timed out
    if (s_ok) {
      v = __ldcv(peer_slot(pq, pq.rank, 0) + idx);
      for (int r = 1; r < pq.nranks; r++) v += __ldcv(peer_slot(pq, pq.rank, r) + idx);
    }
    p.C[idx] = v;
  }
  // seqlock-style re-check: a slot rewritten by a rank that ran ahead while it
  // was being read is reported (C = NaN), never returned as this call's sum
  __syncthreads();
  if (tid == 0 && s_ok) {
    for (int r = 0; r < pq.nranks; r++)
      if (ld_acquire_sys(peer_seq(pq, pq.rank, r)) != pq.seq) {
        atomicExch(peer_err(pq), 1u);
        s_ok = 0;
      }
  }
  __syncthreads();
  if (!s_ok)
    for (int idx = c0 + tid; idx < c1; idx += NT) p.C[idx] = __longlong_as_double(0x7ff8000000000000ll);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmttsm_kernel(const TsmttsmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NT = Cfg::NT;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, MT = Cfg::MT, NTL = Cfg::NTL;
  constexpr int TPR = Cfg::TPR, RB = Cfg::RB, CELLS = Cfg::CELLS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  double* ring = reinterpret_cast<double*>(smem_raw + 128);
  const int tid = threadIdx.x;
  const int rs = tid / TPR;  // row slot
  const int tile = tid % TPR;
  const int tm = tile % MT;  // threads mapped in M direction first
  const int tn = tile / MT;
  const long long K = p.K;
  const long long K_even = K & ~1LL;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncthreads();

  u64 pol = 0;
  auto issue = [&](long long c, int s) {
    const long long r0 = c * R;
    const long long rows = (K_even - r0 < R) ? (K_even - r0) : R;
    const u32 ba = static_cast<u32>(rows * M * S * 8);
    const u32 bb = static_cast<u32>(rows * N * S * 8);
    double* dA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
    double* dB = dA + R * M * S;
    mbar_arrive_expect_tx(&full[s], ba + bb);
    bulk_g2s(dA, p.A + r0 * M * S, ba, &full[s], pol);
    bulk_g2s(dB, p.B + r0 * N * S, bb, &full[s], pol);
  };
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < stages; s++) {
      const long long c = blockIdx.x + static_cast<long long>(s) * G;
      if (c < p.nchunks) issue(c, s);
    }
  }

  double acc[TM][TN][S];
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++)
#pragma unroll
      for (int q = 0; q < S; q++) acc[i][j][q] = 0.0;

  Ring ring_it;
  for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
    const int s = ring_it.s;
    mbar_wait(&full[s], ring_it.ph);
    const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
    const double* sB = sA + R * M * S;
    const long long r0 = c * R;
    const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
    if (rows == R) {
#pragma unroll 2
      for (int r = rs; r < R; r += RB)
        tsmttsm_row<Cfg>(sA + r * M * S, sB + r * N * S, tm, tn, acc, p.conj);
    } else {
      for (int r = rs; r < rows; r += RB)
        tsmttsm_row<Cfg>(sA + r * M * S, sB + r * N * S, tm, tn, acc, p.conj);
    }
    __syncthreads();  // stage s fully consumed by every thread
    if (tid == 0) {
      const long long c2 = c + static_cast<long long>(stages) * G;
      if (c2 < p.nchunks) issue(c2, s);
    }
  }
  // Odd last row (K odd): block 0, slot 0 reads it straight from global.
  if ((K & 1) && blockIdx.x == 0 && rs == 0)
    tsmttsm_row<Cfg>(p.A + (K - 1) * M * S, p.B + (K - 1) * N * S, tm, tn, acc, p.conj);

  // ---- T3: block-level reduction (fixed order) ----
  // (a) butterfly over the row-slot lanes of a warp (same tile, TPR < 32).
  if constexpr (TPR < 32) {
#pragma unroll
    for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++)
#pragma unroll
          for (int q = 0; q < S; q++)
            acc[i][j][q] += __shfl_xor_sync(0xffffffffu, acc[i][j][q], off);
  }
  // (b) holders add into the smem block partial slot by slot, in slot order.
  constexpr int NSLOT = (TPR < 32) ? NT / 32 : RB;
  const int slot = (TPR < 32) ? tid / 32 : rs;
  const bool holder = (TPR < 32) ? ((tid & 31) < TPR) : true;
  double* sP = ring;  // ring is idle now (every issued chunk was consumed)
#pragma unroll 1
  for (int sl = 0; sl < NSLOT; sl++) {
    if (holder && slot == sl) {
#pragma unroll
      for (int i = 0; i < TM; i++) {
        const int m = tm + i * MT;
#pragma unroll
        for (int j = 0; j < TN; j++) {
          const int n = tn + j * NTL;
          if (m < M && n < N) {
#pragma unroll
            for (int q = 0; q < S; q++) {
              const int idx = (m * N + n) * S + q;
              sP[idx] = (sl == 0) ? acc[i][j][q] : sP[idx] + acc[i][j][q];
            }
          }
        }
      }
    }
    __syncthreads();
  }
  grid_reduce<NT, CELLS>(p, sP, ring);
}

// ==========================================================================
// TSMTTSM on the FP64 tensor pipe (DMMA.8x8x4, mma.sync m8n8k4 f64)
// ==========================================================================
// For FMA-heavy widths the register-tile kernel above is issue/latency bound
// (ncu r01: FP64 pipe 48 % at M=N=64 with 8 warps/SM).  Here each consumer
// warp owns a (8*WM) x (8*WN) region of C as WM x WN 8x8 accumulator blocks and
// consumes 4 rows (one k-step) per mma.sync: per 4 rows a warp issues WM + WN
// fragment loads and WM*WN DMMAs (256 FMAs each) instead of 4*TM*TN DFMAs per
// lane.  Operands (PTX m8n8k4 .row.col fragment layout; g = lane/4, q = lane%4):
//   MMA-A = A^T block (8 m x 4 k):  lane holds A[k0+q][m0+g]
//   MMA-B = B block   (4 k x 8 n):  lane holds B[k0+q][n0+g]
//   acc   = C block   (8 m x 8 n):  lane holds C[m0+g][n0+2q], C[m0+g][n0+2q+1]
// Z: re += Ar Br + (-Ai) Bi ; im += Ar Bi + Ai Br  (4 real DMMAs per block).
// Warp specialisation: warp NW is the TMA producer (one elected lane issues the
// bulk copies after the consumers release a stage on its `empty` mbarrier),
// warps 0..NW-1 consume; there is no block-wide barrier in the main loop.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// a + b evaluated where it stands (volatile asm: the compiler neither hoists it
// out of a loop nor keeps it live across iterations)
__device__ __forceinline__ double dadd_here(double a, double b) {
  double r;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// WM x WN: 8x8 blocks per warp tile; NW: consumer warps; R: rows per chunk;
// AP, BP: smem row strides (elements) of the A and B stages.  AP = M / BP = N
// is the dense layout (one bulk copy per chunk); a padded stride (A row
// stride = 8 mod 16 words for D, 4 mod 8 16-byte units for Z) makes the
// fragment loads (4 rows x 8 consecutive elements) hit the minimum number of
// smem wavefronts; the producer then issues one bulk copy per row.
// Shared-memory wavefronts of one fragment load over a dense operand of row
// stride `st` elements when the 4 rows of a k-step are d apart (rows d*q,
// lanes g = 0..7 read consecutive elements; m-offsets shift every lane alike).
// D: LDS.64, two 16-lane phases of 8-byte units; paired D: LDS.128 (g reads
// elements 2g, 2g+1), four 8-lane phases of 16-byte units; Z: LDS.128 of one
// complex element.  Returns the worst lanes-per-unit count (1 = conflict-free).
constexpr int frag_conflict(int st, int d, bool z, bool pair) {
  int worst = 0;
  const int lanes = (z || pair) ? 8 : 16, units = (z || pair) ? 8 : 16;
  for (int ph = 0; ph < 32 / lanes; ph++) {
    int cnt[16] = {};
    for (int l = ph * lanes; l < ph * lanes + lanes; l++) {
      const int g = l >> 2, q = l & 3;
      const int e = d * q * st + (pair ? 2 * g : g);  // element index (complex for Z)
      const int u = z ? e % units : pair ? (e / 2) % units : e % units;
      if (++cnt[u] > worst) worst = cnt[u];
    }
  }
  return worst;
}

// Row spacing d of the k-step rows for a dense layout: the d in {1, 2, 4} (with
// R a multiple of the 4d-row atom) with the fewest conflicts on A and B.
// Rows are assigned per 4d-row atom: k-step t reads rows
// (t/d)*4d + t%d + d*q, so odd strides (d = 4) and strides = 2 mod 4 (d = 2)
// become conflict-free without padding; strides = 0 mod 8 cannot.
constexpr int pick_kdist(int ap, int bp, bool z, bool pair, int r) {
  int best = 1, bc = 1 << 20;
  for (int d = 1; d <= 4; d *= 2) {
    if (r % (4 * d)) continue;
    const int c = frag_conflict(ap, d, z, pair) + frag_conflict(bp, d, z, pair);
    if (c < bc) {
      bc = c;
      best = d;
    }
  }
  return best;
}

// TMA = true: A and B arrive by 2-D tensor copies into 128B-swizzled boxes
// (AP, BP ignored; requires M*S and N*S even and >= 16 doubles).
// EDGE = true: DMMA covers only the 8-aligned core MC x NC of C
// (MC = 8*floor(M/8)); one extra consumer warp computes the E = M*N - MC*NC
// edge cells with DFMA (worth it when M or N is just above a multiple of 8,
// where 8x8 blocks would waste up to (ceil8(M)/M)^2 of the DMMA work).
// LB = true (D, kernel | 4096): "L-blocks" instead of padding for the cells
// outside the 8-aligned core MC x NC, all on the tensor pipe.  With ER = M - MC
// edge rows and EC = N - NC edge columns (both 1..6), L-block l is the 8 x 8
// MMA block with rows {MC .. M-1} plus the core rows [l (8-ER), (l+1)(8-ER)) and
// columns {NC .. N-1} plus the core columns [l (8-EC), (l+1)(8-EC)).  Its
// edge-row x core-column and core-row x edge-column cells are the edge strips
// (each cell in exactly one block; the corner from block 0); its core x core
// interior repeats core cells and is dropped.  NL = max(ceil(MC / (8-ER)),
// ceil(NC / (8-EC))) blocks replace the ceil(M/8) ceil(N/8) - MB NB padded
// ones: D 57 57 blocks instead of 64, D 49 43 instead of 49, D 41 31 / 36.
// An MMA output block is an 8 x 8 outer-product structure, so a strip one cell
// wide is at best 1/8 useful per block; pairing a row strip with a column
// strip in one block doubles that.
// PAIR = true (D only): blocks are used in pairs covering 16 consecutive m (n);
// block 2p holds the even, block 2p+1 the odd rows (columns) of the pair, so
// one 16-byte LDS.128 per lane feeds both fragments (half the load
// instructions of one LDS.64 per fragment).
template <int M_, int N_, bool Z_, int WM_, int WN_, int NW_, int R_, int AP_ = M_, int BP_ = N_,
          bool TMA_ = false, int EDGE_ = 0, bool PAIR_ = false, bool ZR_ = false, bool G3_ = false,
          bool EI_ = false, bool LB_ = false, bool GA_ = false>
struct TsmttsmMmaCfg {
  static constexpr int M = M_, N = N_, WM = WM_, WN = WN_, NW = NW_, R = R_;
  // EI ("inline edge", kernel | 2048): the edge cells are computed by the
  // consumer warps themselves, interleaved with their DMMAs (no edge warps)
  static constexpr bool EI = EI_;
  static constexpr bool LB = LB_;
  // GA (kernel | 8192): the gather-capable instantiation (strided views, NEXT N4).
  // A separate instantiation: the gather producer code in every kernel made
  // NVRTC's ptxas allocate fewer registers and spill in the edge-warp / inline-
  // edge kernels (D 49 edge warps 96 -> 72 registers + 24 B stack, +15 % time).
  static constexpr bool GA = GA_;
  static_assert(!GA_ || !TMA_, "gather mode: the bulk-copy kernel");
  static constexpr bool Z = Z_, TMA = TMA_, EDGE = EDGE_ > 0 || EI_ || LB_, PAIR = PAIR_, ZR = ZR_, G3 = G3_;
  static constexpr bool DEDGE = EDGE_ > 0 || EI_;  // DFMA edge strips (edge warps or inline)
  static_assert(!(EI_ && EDGE_ > 0), "inline edge excludes edge warps");
  // (complex-as-real runs the real kernel on 2M x 2N: L-blocks apply to that product)
  static_assert(!LB_ || (!EI_ && EDGE_ == 0), "L-blocks exclude the DFMA edges");
  static_assert(!G3 || Z_, "3M (Gauss) products: complex kernel");
  static_assert(!ZR || (!Z_ && M_ % 2 == 0 && N_ % 2 == 0), "complex-as-real: real kernel on 2M x 2N");
  static_assert(!PAIR || (!Z_ && WM_ % 2 == 0 && WN_ % 2 == 0), "pairs: real, even tiles");
  static constexpr int S = Z ? 2 : 1;
  static constexpr int NA = G3 ? 3 : S;  // accumulator blocks per 8x8 block of C (3M: T1, T2, T3)
  static constexpr int NBA = (M * S + 15) / 16, NBB = (N * S + 15) / 16;  // 16-double boxes
  static constexpr int AP = TMA ? NBA * 16 / S : AP_, BP = TMA ? NBB * 16 / S : BP_;
  static_assert(!TMA || ((M * S) % 2 == 0 && (N * S) % 2 == 0 && M * S >= 16 && N * S >= 16),
                "TMA tensor path: 16-byte rows of >= 128 bytes");
  static_assert(!TMA || R % 8 == 0, "TMA swizzle atoms are 8 rows");
  static constexpr int MC = EDGE ? (M / 8) * 8 : M, NC = EDGE ? (N / 8) * 8 : N;  // DMMA core
  // 8x8 blocks of the core (pair mode: whole 16-wide pairs)
  // 8x8 blocks of the core.  Pair mode pairs blocks (2p, 2p+1) over the
  // 16-wide band [16p, 16p+16); an odd last block (MB odd) is loaded single.
  static constexpr int MB = (MC + 7) / 8;
  static constexpr int NB = (NC + 7) / 8;
  static constexpr int E = M * N - MC * NC;                    // edge cells (DFMA warps)
  // edge strips as outer products: rows m in [MC, M) x all n (lanes over n),
  // columns n in [NC, N) x m < MC (lanes over m)
  static constexpr int MR = M - MC, NR = N - NC;
  static constexpr int UN = (N + 31) / 32, UM = (MC + 31) / 32;
  static constexpr int EREGS = (MR * UN + UM * NR) * S;        // accumulator doubles per lane
  static constexpr int NE = EDGE_;                             // edge warps (split the rows)
  static_assert(!LB_ || (MR >= 1 && MR <= 6 && NR >= 1 && NR <= 6), "L-blocks: 1..6 edge rows and columns");
  static constexpr int NL = !LB_ ? 0
                            : ((MC + 7 - MR) / (8 - MR) > (NC + 7 - NR) / (8 - NR) ? (MC + 7 - MR) / (8 - MR)
                                                                                    : (NC + 7 - NR) / (8 - NR));
  static_assert(NE >= 0 && NE <= 4, "0..4 edge warps");
  static_assert(!EDGE || (MB >= 1 && NB >= 1 && E > 0), "edge mode needs a core and an edge");
  static constexpr int WTM = (MB + WM - 1) / WM, WTN = (NB + WN - 1) / WN;
  static constexpr int WT = WTM * WTN;                          // warp tiles covering C
  static constexpr int RS = NW / WT;                            // row slots (k-step groups)
  static constexpr int NT = (NW + NE + 1) * 32;                 // + edge + producer warp
  static constexpr int CELLS = M * N * S;
  static constexpr int OUT_CELLS = ZR ? CELLS / 2 : CELLS;  // doubles of the block partial
  static constexpr int STAGE_DOUBLES = R * (AP + BP) * S;
  // k-step row spacing (see pick_kdist); the 128B swizzle needs rows 2 apart
  static constexpr int KD = TMA ? 2 : pick_kdist(AP, BP, Z, PAIR, R);
  static_assert(R % (4 * KD) == 0, "rows per chunk: whole k-step atoms");
  static_assert(NW % WT == 0 && RS >= 1, "consumer warps must be a multiple of the warp tiles");
  static_assert(R % 4 == 0, "R must be a multiple of the k-step (4 rows)");
  static_assert(WM <= MB && WN <= NB, "warp tile larger than C");
  static_assert(AP == M || ((AP * S) % 2 == 0 && (M * S) % 2 == 0), "padded A rows: 16-byte rows");
  static_assert(BP == N || ((BP * S) % 2 == 0 && (N * S) % 2 == 0), "padded B rows: 16-byte rows");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmttsm_mma_kernel(const __grid_constant__ TsmttsmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NW = Cfg::NW;
  constexpr int WM = Cfg::WM, WN = Cfg::WN, WTM = Cfg::WTM, MB = Cfg::MB, NB = Cfg::NB;
  constexpr int WT = Cfg::WT, RS = Cfg::RS, CELLS = Cfg::CELLS, AP = Cfg::AP, BP = Cfg::BP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  u64* empty = full + 16;
  // ring: 1024-byte aligned for the 128B-swizzle atoms of the TMA boxes.
  // Pointer arithmetic on smem_raw (never an integer round trip) keeps the
  // shared address space visible to the compiler: fragment loads stay LDS.
  double* ring = reinterpret_cast<double*>(smem_raw + (Cfg::TMA ? align1024(smem_raw, 256) : 256));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const long long K = p.K;
  const long long K_even = K & ~1LL;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], (Cfg::GA && p.gather) ? 32 : 1);  // gather: one noinc arrival per producer lane
      mbar_init(&empty[s], NW + Cfg::NE);  // consumer + edge warps release a stage
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncthreads();

  // accumulators: [WM][WN] blocks x 2 doubles (x re/im; 3M: x T1, T2, T3)
  constexpr int NA = Cfg::NA;
  double acc[WM][WN][NA][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++)
#pragma unroll
      for (int z = 0; z < NA; z++) acc[i][j][z][0] = acc[i][j][z][1] = 0.0;

  const int wl = spread_warp(warp, NW, p.order);  // (slot, tile) of this consumer warp
  const int slot = wl / WT;
  const int wt = wl % WT;
  const int wm = wt % WTM, wn = wt / WTM;

  // offset (doubles) of element (row r, column x) of an operand of width W
  // elements: dense row stride `st`, or the swizzled TMA boxes
  auto off = [&](int r, int x, int st) -> int {
    if constexpr (Cfg::TMA) {
      const int c = x * S;  // first double of the element
      return (c >> 4) * (R * 16) + swz128(r, c & 15);
    } else {
      return (r * st + x) * S;
    }
  };

  // one k-step: 4 rows of the stage (row strides ap, bp elements), or of global
  // memory for the odd tail row (strides M, N; non-TMA only).  K-step k0 (t = k0/4)
  // reads rows (t/KD)*4KD + t%KD + KD*q: rows KD apart, chosen so that every
  // fragment load hits distinct banks (swizzled TMA boxes: KD = 2 puts the 4
  // rows in different swizzle phases; dense rows: see pick_kdist).  The sum over
  // k is unchanged: A and B fragments of a lane always read the same row, and
  // the k-steps of a 4KD-row atom visit each of its rows once.
  // cm, cn (IC<.>): accumulator blocks of this warp's tile that lie inside C --
  // compile-time, so partial tiles issue no predicated-off DMMAs (which still
  // occupy the tensor pipe: ncu r19, D 40 ran 30 block-slots for 25 blocks).
  auto kstep = [&](auto cm, auto cn, const double* __restrict__ sA, const double* __restrict__ sB, int k0,
                   int rows, int ap, int bp) {
    constexpr int CM = decltype(cm)::value, CN = decltype(cn)::value;
    constexpr int KD = Cfg::KD;
    const int kr = (k0 & ~(4 * KD - 1)) + ((k0 >> 2) & (KD - 1)) + KD * q;
    const bool rv = kr < rows;
    if constexpr (!Cfg::Z) {
      double a[WM], b[WN];
      if constexpr (Cfg::PAIR) {
        // one 16-byte load per lane: (m, m+1) -> fragments of blocks 2p, 2p+1
#pragma unroll
        for (int ip = 0; ip < CM / 2; ip++) {
          const int m = (wm * WM + 2 * ip) * 8 + 2 * g;
          double2 v = make_double2(0.0, 0.0);
          if (rv && m + 1 < M)
            v = *reinterpret_cast<const double2*>(sA + off(kr, m, ap));
          else if (rv && m < M)
            v.x = sA[off(kr, m, ap)];
          a[2 * ip] = v.x;
          a[2 * ip + 1] = v.y;
        }
#pragma unroll
        for (int jp = 0; jp < CN / 2; jp++) {
          const int n = (wn * WN + 2 * jp) * 8 + 2 * g;
          double2 v = make_double2(0.0, 0.0);
          if (rv && n + 1 < N)
            v = *reinterpret_cast<const double2*>(sB + off(kr, n, bp));
          else if (rv && n < N)
            v.x = sB[off(kr, n, bp)];
          b[2 * jp] = v.x;
          b[2 * jp + 1] = v.y;
        }
        // odd tile: its last block (the globally last, MB odd) is contiguous, loaded single
        if constexpr (CM % 2) {
          const int m = (wm * WM + CM - 1) * 8 + g;
          a[CM - 1] = (rv && m < M) ? sA[off(kr, m, ap)] : 0.0;
        }
        if constexpr (CN % 2) {
          const int n = (wn * WN + CN - 1) * 8 + g;
          b[CN - 1] = (rv && n < N) ? sB[off(kr, n, bp)] : 0.0;
        }
      } else {
#pragma unroll
        for (int i = 0; i < CM; i++) {
          const int m = (wm * WM + i) * 8 + g;
          a[i] = (rv && m < M) ? sA[off(kr, m, ap)] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CN; j++) {
          const int n = (wn * WN + j) * 8 + g;
          b[j] = (rv && n < N) ? sB[off(kr, n, bp)] : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < CM; i++)
#pragma unroll
        for (int j = 0; j < CN; j++) dmma(acc[i][j][0][0], acc[i][j][0][1], a[i], b[j]);
    } else {
      double2 a[WM], b[WN];
#pragma unroll
      for (int i = 0; i < CM; i++) {
        const int m = (wm * WM + i) * 8 + g;
        a[i] = (rv && m < M) ? *reinterpret_cast<const double2*>(sA + off(kr, m, ap))
                             : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < CN; j++) {
        const int n = (wn * WN + j) * 8 + g;
        b[j] = (rv && n < N) ? *reinterpret_cast<const double2*>(sB + off(kr, n, bp))
                             : make_double2(0.0, 0.0);
      }
      if constexpr (Cfg::G3) {
        // 3M (Gauss) products: T1 += ar br, T2 += ai bi, T3 += (ar + ai)(br + bi);
        // C = (T1 - T2) + i (T3 - T1 - T2) is formed once per block partial.
        // 3 DMMAs per block instead of 4; the operand sums cost one DADD per
        // fragment (exact for the integer-valued parity inputs).
        double sa[WM], sb[WN];
#pragma unroll
        for (int i = 0; i < CM; i++) {
          a[i].y = flip_sign(a[i].y, p.conj);  // A^H B (N2)
          sa[i] = a[i].x + a[i].y;
        }
#pragma unroll
        for (int j = 0; j < CN; j++) sb[j] = b[j].x + b[j].y;
#pragma unroll
        for (int i = 0; i < CM; i++)
#pragma unroll
          for (int j = 0; j < CN; j++) {
            dmma(acc[i][j][0][0], acc[i][j][0][1], a[i].x, b[j].x);  // T1 += ar br
            dmma(acc[i][j][1][0], acc[i][j][1][1], a[i].y, b[j].y);  // T2 += ai bi
            dmma(acc[i][j][2][0], acc[i][j][2][1], sa[i], sb[j]);    // T3 += (ar+ai)(br+bi)
          }
      } else {
#pragma unroll
      for (int i = 0; i < CM; i++) {
        a[i].y = flip_sign(a[i].y, p.conj);  // A^H B (N2)
        const double nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < CN; j++) {
            dmma(acc[i][j][0][0], acc[i][j][0][1], a[i].x, b[j].x);  // re += ar br
            dmma(acc[i][j][0][0], acc[i][j][0][1], nai, b[j].y);     // re -= ai bi
            dmma(acc[i][j][1][0], acc[i][j][1][1], a[i].x, b[j].y);  // im += ar bi
            dmma(acc[i][j][1][0], acc[i][j][1][1], a[i].y, b[j].x);  // im += ai br
          }
      }
      }
    }
  };

  // edge cells (EDGE mode) as two outer-product strips: the row strip
  // m in [MC, M) x n in [0, N) with lanes over n (B values loaded once per row,
  // A[k][m] broadcast), and the column strip m in [0, MC) x n in [NC, N) with
  // lanes over m (A loaded once, B[k][n] broadcast).  Per row and lane:
  // ceil(N/32) + ceil(MC/32) loads + MR + NR broadcasts for the
  // MR*ceil(N/32) + ceil(MC/32)*NR DFMA (or complex) updates.
  constexpr int MR = Cfg::MR, NR = Cfg::NR, UN = Cfg::UN, UM = Cfg::UM;
  constexpr int MRA = MR > 0 ? MR : 1, NRA = NR > 0 ? NR : 1;
  double er[Cfg::DEDGE ? MRA : 1][Cfg::DEDGE ? UN : 1][S];  // row strip (MC + mi, lane + 32u)
  double ec[Cfg::DEDGE ? UM : 1][Cfg::DEDGE ? NRA : 1][S];  // column strip (lane + 32u, NC + ni)
  if constexpr (Cfg::DEDGE) {
#pragma unroll
    for (int i = 0; i < MRA; i++)
#pragma unroll
      for (int u = 0; u < UN; u++)
#pragma unroll
        for (int z = 0; z < S; z++) er[i][u][z] = 0.0;
#pragma unroll
    for (int u = 0; u < UM; u++)
#pragma unroll
      for (int i = 0; i < NRA; i++)
#pragma unroll
        for (int z = 0; z < S; z++) ec[u][i][z] = 0.0;
  }
  // DFMA over rows [r_begin, rows) step NE of a stage (or of global memory: the odd tail row)
  auto edge_rows = [&](const double* __restrict__ sA, const double* __restrict__ sB, int r_begin, int rows,
                       int ap, int bp) {
#pragma unroll 2
    for (int r = r_begin; r < rows; r += Cfg::NE) {
      if constexpr (MR > 0) {
        double bv[UN][S];
#pragma unroll
        for (int u = 0; u < UN; u++) {
          const int n = lane + 32 * u;
#pragma unroll
          for (int z = 0; z < S; z++) bv[u][z] = (n < N) ? sB[off(r, n, bp) + z] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < MR; i++) {
          const int m = Cfg::MC + i;
          if constexpr (!Cfg::Z) {
            const double a = sA[off(r, m, ap)];
#pragma unroll
            for (int u = 0; u < UN; u++) er[i][u][0] = fma(a, bv[u][0], er[i][u][0]);
          } else {
            const double2 a = *reinterpret_cast<const double2*>(sA + off(r, m, ap));
            const double ai = flip_sign(a.y, p.conj);
#pragma unroll
            for (int u = 0; u < UN; u++) zfma(er[i][u][0], er[i][u][1], a.x, ai, bv[u][0], bv[u][1]);
          }
        }
      }
      if constexpr (NR > 0) {
        double av[UM][S];
#pragma unroll
        for (int u = 0; u < UM; u++) {
          const int m = lane + 32 * u;
#pragma unroll
          for (int z = 0; z < S; z++) av[u][z] = (m < Cfg::MC) ? sA[off(r, m, ap) + z] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < NR; i++) {
          const int n = Cfg::NC + i;
          if constexpr (!Cfg::Z) {
            const double b = sB[off(r, n, bp)];
#pragma unroll
            for (int u = 0; u < UM; u++) ec[u][i][0] = fma(av[u][0], b, ec[u][i][0]);
          } else {
            const double2 b = *reinterpret_cast<const double2*>(sB + off(r, n, bp));
#pragma unroll
            for (int u = 0; u < UM; u++)
              zfma(ec[u][i][0], ec[u][i][1], av[u][0], flip_sign(av[u][1], p.conj), b.x, b.y);
          }
        }
      }
    }
  };

  // EI: the consumer warps of a row slot share the edge work of the 4 rows of
  // each k-step.  Groups: row-strip lane group u (cells (MC+i, lane+32u), i <
  // MR, one B load + MR broadcasts of A) for u < UN, then column-strip lane
  // group u (cells (lane+32u, NC+i), one A load + NR broadcasts of B); group g
  // belongs to the warp tile g % WT of the slot.
  constexpr int NGRP = UN + UM;
  auto edge_inline = [&](const double* __restrict__ sA, const double* __restrict__ sB, int k0, int rows,
                         int ap, int bp) {
    constexpr int KD = Cfg::KD;
    const int base = (k0 & ~(4 * KD - 1)) + ((k0 >> 2) & (KD - 1));
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int r = base + KD * j;
      if (r >= rows) break;  // (warp-uniform)
#pragma unroll
      for (int g = 0; g < NGRP; g++) {
        if (g % Cfg::WT != wt) continue;  // (warp-uniform)
        if (g < UN) {
          if constexpr (MR > 0) {
            const int u = g, n = lane + 32 * u;
            double bv[S];
#pragma unroll
            for (int z = 0; z < S; z++) bv[z] = (n < N) ? sB[off(r, n, bp) + z] : 0.0;
#pragma unroll
            for (int i = 0; i < MR; i++) {
              if constexpr (!Cfg::Z) {
                er[i][u][0] = fma(sA[off(r, Cfg::MC + i, ap)], bv[0], er[i][u][0]);
              } else {
                const double2 a = *reinterpret_cast<const double2*>(sA + off(r, Cfg::MC + i, ap));
                zfma(er[i][u][0], er[i][u][1], a.x, flip_sign(a.y, p.conj), bv[0], bv[S - 1]);
              }
            }
          }
        } else {
          if constexpr (NR > 0) {
            const int u = g - UN, m = lane + 32 * u;
            double av[S];
#pragma unroll
            for (int z = 0; z < S; z++) av[z] = (m < Cfg::MC) ? sA[off(r, m, ap) + z] : 0.0;
            if constexpr (Cfg::Z) av[S - 1] = flip_sign(av[S - 1], p.conj);
#pragma unroll
            for (int i = 0; i < NR; i++) {
              if constexpr (!Cfg::Z) {
                ec[u][i][0] = fma(av[0], sB[off(r, Cfg::NC + i, bp)], ec[u][i][0]);
              } else {
                const double2 b = *reinterpret_cast<const double2*>(sB + off(r, Cfg::NC + i, bp));
                zfma(ec[u][i][0], ec[u][i][1], av[0], av[S - 1], b.x, b.y);
              }
            }
          }
        }
      }
    }
  };

  // LB: the L-blocks l = wt, wt + WT, ... of this warp's tile (one DMMA each per
  // k-step, A and B fragments gathered from the block's row / column lists)
  constexpr int NLW = Cfg::LB ? (Cfg::NL + Cfg::WT - 1) / Cfg::WT : 1;
  double lacc[NLW][NA][2];  // (Z: re, im; 3M: T1, T2, T3 -- as the core blocks)
#pragma unroll
  for (int t = 0; t < NLW; t++)
#pragma unroll
    for (int z = 0; z < NA; z++) lacc[t][z][0] = lacc[t][z][1] = 0.0;
  auto lstep = [&](const double* __restrict__ sA, const double* __restrict__ sB, int k0, int rows, int ap,
                   int bp) {
    constexpr int KD = Cfg::KD;
    const int kr = (k0 & ~(4 * KD - 1)) + ((k0 >> 2) & (KD - 1)) + KD * q;
    const bool rv = kr < rows;
#pragma unroll
    for (int t = 0; t < NLW; t++) {
      const int l = wt + t * Cfg::WT;
      if (l >= Cfg::NL) break;  // (warp-uniform)
      const int mr = g < MR ? Cfg::MC + g : l * (8 - MR) + (g - MR);  // MMA row g -> m
      const int nc = g < NR ? Cfg::NC + g : l * (8 - NR) + (g - NR);  // MMA column g -> n
      const bool av = rv && (g < MR || mr < Cfg::MC), bv = rv && (g < NR || nc < Cfg::NC);
      if constexpr (!Cfg::Z) {
        const double a = av ? sA[off(kr, mr, ap)] : 0.0;
        const double b = bv ? sB[off(kr, nc, bp)] : 0.0;
        dmma(lacc[t][0][0], lacc[t][0][1], a, b);
      } else {
        double2 a = av ? *reinterpret_cast<const double2*>(sA + off(kr, mr, ap)) : make_double2(0.0, 0.0);
        const double2 b = bv ? *reinterpret_cast<const double2*>(sB + off(kr, nc, bp)) : make_double2(0.0, 0.0);
        a.y = flip_sign(a.y, p.conj);  // A^H B (N2)
        if constexpr (Cfg::G3) {
          dmma(lacc[t][0][0], lacc[t][0][1], a.x, b.x);              // T1 += ar br
          dmma(lacc[t][1][0], lacc[t][1][1], a.y, b.y);              // T2 += ai bi
          dmma(lacc[t][2][0], lacc[t][2][1], a.x + a.y, b.x + b.y);  // T3 += (ar+ai)(br+bi)
        } else {
          dmma(lacc[t][0][0], lacc[t][0][1], a.x, b.x);   // re += ar br
          dmma(lacc[t][0][0], lacc[t][0][1], -a.y, b.y);  // re -= ai bi
          dmma(lacc[t][1][0], lacc[t][1][1], a.x, b.y);   // im += ar bi
          dmma(lacc[t][1][0], lacc[t][1][1], a.y, b.x);   // im += ai br
        }
      }
    }
  };

  if (warp == NW + Cfg::NE) {
    // ---------------- producer warp: bulk / tensor copies into the ring ----------------
    const u64 pol = policy_evict_first();
    Ring ring_it;
    for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
      const int s = ring_it.s;
      if (ring_it.round > 0 && lane == 0) mbar_wait(&empty[s], ring_it.ph ^ 1u);
      __syncwarp();
      const long long r0 = c * R;
      double* dA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
      double* dB = dA + R * AP * S;
      if constexpr (Cfg::TMA) {
        // whole boxes (rows past K are zero-filled and still counted)
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], static_cast<u32>((Cfg::NBA + Cfg::NBB) * R * 128));
          for (int b = 0; b < Cfg::NBA; b++)
            tma_load_2d(dA + b * R * 16, &p.tmA, b * 16, static_cast<int>(r0), &full[s], pol);
          for (int b = 0; b < Cfg::NBB; b++)
            tma_load_2d(dB + b * R * 16, &p.tmB, b * 16, static_cast<int>(r0), &full[s], pol);
        }
      } else if (Cfg::GA && p.gather) {  // strided rows (N4): element copies, any row stride
        if constexpr (Cfg::GA) {
          const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
          gather_rows<M, S>(dA, AP, p.A, r0, p.lda, rows, lane);
          gather_rows<N, S>(dB, BP, p.B, r0, p.ldb, rows, lane);
          cp_async_mbar_arrive_noinc(&full[s]);
        }
      } else {
        const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<u32>(rows * (M + N) * S * 8));
        __syncwarp();
        if constexpr (AP == M) {
          if (lane == 0) bulk_g2s(dA, p.A + r0 * M * S, static_cast<u32>(rows * M * S * 8), &full[s], pol);
        } else {
          for (int r = lane; r < rows; r += 32)
            bulk_g2s(dA + r * AP * S, p.A + (r0 + r) * M * S, static_cast<u32>(M * S * 8), &full[s], pol);
        }
        if constexpr (BP == N) {
          if (lane == 0) bulk_g2s(dB, p.B + r0 * N * S, static_cast<u32>(rows * N * S * 8), &full[s], pol);
        } else {
          for (int r = lane; r < rows; r += 32)
            bulk_g2s(dB + r * BP * S, p.B + (r0 + r) * N * S, static_cast<u32>(N * S * 8), &full[s], pol);
        }
      }
    }
  } else if (Cfg::DEDGE && warp >= NW) {  // (warp < NW + NE: the producer is NW + NE)
    // ---------------- edge warps: DFMA on the cells outside the DMMA core ----------------
    // (edge warp ew takes rows ew, ew + NE, ... of every chunk)
    const int ew = warp - NW;
    Ring ring_it;
    for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
      const int s = ring_it.s;
      mbar_wait(&full[s], ring_it.ph);
      const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
      const double* sB = sA + R * AP * S;
      const long long r0 = c * R;
      edge_rows(sA, sB, ew, Cfg::TMA ? R : static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R), AP, BP);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if constexpr (!Cfg::TMA) {
      if ((K & 1) && blockIdx.x == 0 && ew == 0)
        edge_rows(p.A + (K - 1) * p.lda * S, p.B + (K - 1) * p.ldb * S, 0, 1, M, N);
    }
  } else {
    // ---------------- consumer warps ----------------
    auto consume = [&](auto cm, auto cn) {
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        mbar_wait(&full[s], ring_it.ph);
        const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
        const double* sB = sA + R * AP * S;
        const long long r0 = c * R;
        const int rows = Cfg::TMA ? R : static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
        if (rows == R) {
#pragma unroll 2
          for (int k0 = slot * 4; k0 < R; k0 += RS * 4) {
            kstep(cm, cn, sA, sB, k0, R, AP, BP);
            if constexpr (Cfg::EI) edge_inline(sA, sB, k0, R, AP, BP);
            if constexpr (Cfg::LB) lstep(sA, sB, k0, R, AP, BP);
          }
        } else {  // partial chunk: every k-step of the atoms that hold rows < rows
          const int kend = (rows + 4 * Cfg::KD - 1) & ~(4 * Cfg::KD - 1);
          for (int k0 = slot * 4; k0 < kend; k0 += RS * 4) {
            kstep(cm, cn, sA, sB, k0, rows, AP, BP);
            if constexpr (Cfg::EI) edge_inline(sA, sB, k0, rows, AP, BP);
            if constexpr (Cfg::LB) lstep(sA, sB, k0, rows, AP, BP);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // odd last row: a k-step whose rows 1..3 are zero, from global memory
      if constexpr (!Cfg::TMA) {
        if ((K & 1) && blockIdx.x == 0 && slot == 0) {
          kstep(cm, cn, p.A + (K - 1) * p.lda * S, p.B + (K - 1) * p.ldb * S, 0, 1, M, N);
          if constexpr (Cfg::EI) edge_inline(p.A + (K - 1) * p.lda * S, p.B + (K - 1) * p.ldb * S, 0, 1, M, N);
          if constexpr (Cfg::LB) lstep(p.A + (K - 1) * p.lda * S, p.B + (K - 1) * p.ldb * S, 0, 1, M, N);
        }
      }
    };
    // warp-uniform dispatch on whether this warp's tile is the last (partial) one
    constexpr int RM = MB - (WTM - 1) * WM, RN = NB - (Cfg::WTN - 1) * WN;  // blocks in C
    const bool lm = (wm == WTM - 1), ln = (wn == Cfg::WTN - 1);
    if (lm && ln)
      consume(IC<RM>{}, IC<RN>{});
    else if (lm)
      consume(IC<RM>{}, IC<WN>{});
    else if (ln)
      consume(IC<WM>{}, IC<RN>{});
    else
      consume(IC<WM>{}, IC<WN>{});
  }
  __syncthreads();  // ring idle: every issued chunk was consumed

  // ---- T3: block partial, slot by slot in slot order ----
  double* sP = ring;
#pragma unroll 1
  for (int sl = 0; sl < (RS > Cfg::NE ? RS : Cfg::NE); sl++) {
    if (warp < NW && slot == sl) {
#pragma unroll
      for (int i = 0; i < WM; i++) {
        // pair mode: blocks 2p / 2p+1 hold the even / odd m of band 16p; the odd last block is contiguous
        const bool msingle = !Cfg::PAIR || ((MB & 1) && wm * WM + i == MB - 1);
        const int m = msingle ? (wm * WM + i) * 8 + g : (wm * WM + (i & ~1)) * 8 + 2 * g + (i & 1);
#pragma unroll
        for (int j = 0; j < WN; j++) {
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const bool nsingle = !Cfg::PAIR || ((NB & 1) && wn * WN + j == NB - 1);
            const int n = nsingle ? (wn * WN + j) * 8 + 2 * q + e
                                  : (wn * WN + (j & ~1)) * 8 + 2 * (2 * q + e) + (j & 1);
            if (m < M && n < N && (wm * WM + i) < MB && (wn * WN + j) < NB) {
              double v[S];
              if constexpr (Cfg::G3) {  // re = T1 - T2, im = T3 - T1 - T2
                v[0] = acc[i][j][0][e] - acc[i][j][1][e];
                v[1] = acc[i][j][2][e] - acc[i][j][0][e] - acc[i][j][1][e];
              } else {
#pragma unroll
                for (int z = 0; z < S; z++) v[z] = acc[i][j][z][e];
              }
#pragma unroll
              for (int z = 0; z < S; z++) {
                const int idx = (m * N + n) * S + z;
                sP[idx] = (sl == 0) ? v[z] : sP[idx] + v[z];
              }
            }
          }
        }
      }
    }
    if constexpr (Cfg::EI) {  // inline edge: the owning warp tile of each group, slot by slot
      if (warp < NW && slot == sl) {
        auto put = [&](int m, int n, const double* v) {
#pragma unroll
          for (int z = 0; z < S; z++) {
            const int idx = (m * N + n) * S + z;
            sP[idx] = (sl == 0) ? v[z] : sP[idx] + v[z];
          }
        };
#pragma unroll
        for (int g = 0; g < NGRP; g++) {
          if (g % Cfg::WT != wt) continue;
          if (g < UN) {
            if constexpr (MR > 0) {
#pragma unroll
              for (int i = 0; i < MR; i++)
                if (lane + 32 * g < N) put(Cfg::MC + i, lane + 32 * g, er[i][g]);
            }
          } else {
            if constexpr (NR > 0) {
#pragma unroll
              for (int i = 0; i < NR; i++)
                if (lane + 32 * (g - UN) < Cfg::MC) put(lane + 32 * (g - UN), Cfg::NC + i, ec[g - UN][i]);
            }
          }
        }
      }
    }
    if constexpr (Cfg::LB) {  // L-blocks: the edge cells of each block, slot by slot
      if (warp < NW && slot == sl) {
#pragma unroll
        for (int t = 0; t < NLW; t++) {
          const int l = wt + t * Cfg::WT;
          if (l >= Cfg::NL) break;
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int j = 2 * q + e;  // MMA column; g is the MMA row
            int m = -1, n = -1;
            if (g < MR) {  // edge row x (edge columns: block 0 only | core columns)
              m = Cfg::MC + g;
              n = j < NR ? (l == 0 ? Cfg::NC + j : -1) : l * (8 - NR) + (j - NR);
              if (n >= Cfg::NC && j >= NR) n = -1;
            } else if (j < NR) {  // core row x edge column
              m = l * (8 - MR) + (g - MR);
              n = m < Cfg::MC ? Cfg::NC + j : -1;
            }
            if (n >= 0) {
              double v[S];
              if constexpr (Cfg::G3) {  // re = T1 - T2, im = T3 - T1 - T2
                v[0] = lacc[t][0][e] - lacc[t][1][e];
                v[S - 1] = lacc[t][2][e] - lacc[t][0][e] - lacc[t][1][e];
              } else {
#pragma unroll
                for (int z = 0; z < S; z++) v[z] = lacc[t][z][e];
              }
#pragma unroll
              for (int z = 0; z < S; z++) {
                const int idx = (m * N + n) * S + z;
                sP[idx] = (sl == 0) ? v[z] : sP[idx] + v[z];
              }
            }
          }
        }
      }
    }
    if constexpr (Cfg::DEDGE && !Cfg::EI) {  // edge cells are disjoint from the core; edge warps in order
      if (warp == NW + sl && sl < Cfg::NE) {
        auto put = [&](int m, int n, const double* v) {
#pragma unroll
          for (int z = 0; z < S; z++) {
            const int idx = (m * N + n) * S + z;
            sP[idx] = (sl == 0) ? v[z] : sP[idx] + v[z];
          }
        };
        if constexpr (MR > 0) {
#pragma unroll
          for (int i = 0; i < MR; i++)
#pragma unroll
            for (int u = 0; u < UN; u++)
              if (lane + 32 * u < N) put(Cfg::MC + i, lane + 32 * u, er[i][u]);
        }
        if constexpr (NR > 0) {
#pragma unroll
          for (int u = 0; u < UM; u++)
#pragma unroll
            for (int i = 0; i < NR; i++)
              if (lane + 32 * u < Cfg::MC) put(lane + 32 * u, Cfg::NC + i, ec[u][i]);
        }
      }
    }
    __syncthreads();
  }
  if constexpr (Cfg::ZR) {
    // complex C from the real product P = Ar^T Br of the interleaved (re, im)
    // columns: C[m][n] = (P[2m][2n] - P[2m+1][2n+1]) + i (P[2m][2n+1] + P[2m+1][2n]);
    // A^H B (conj, N2) flips the sign of the Im(A) rows: + P[2m+1][2n+1], - P[2m+1][2n]
    constexpr int NZ = N / 2, MNZ = (M / 2) * NZ;
    double* sQ = ring + CELLS;
    for (int idx = tid; idx < MNZ; idx += Cfg::NT) {
      const int m = 2 * (idx / NZ), n = 2 * (idx % NZ);
      sQ[2 * idx] = sP[m * N + n] - flip_sign(sP[(m + 1) * N + n + 1], p.conj);
      sQ[2 * idx + 1] = sP[m * N + n + 1] + flip_sign(sP[(m + 1) * N + n], p.conj);
    }
    __syncthreads();
    grid_reduce<Cfg::NT, Cfg::OUT_CELLS>(p, sQ, sQ + Cfg::OUT_CELLS);
  } else {
    grid_reduce<Cfg::NT, CELLS>(p, sP, ring + CELLS);
  }
}

// ==========================================================================
// TSMM
// ==========================================================================
struct TsmmArgs {
  TmaDesc tmA, tmB;   // tensor maps (TMA kernels only): A loads, B stores
  const double* A;    // K x M
  const double* C;    // M x N
  double* B;          // K x N
  long long K;
  long long nchunks;  // ceil(K_even / R)  (TMA kernels: ceil(K / R))
  int stages;
  int reduce;         // 0: B = A C' (store); 1: B += A C' (bulk / TMA reduce-add; NEXT N1)
  double alpha_re, alpha_im;  // C' = alpha * C (alpha = 1: C used as given, bit-exact)
  int order;          // consumer-warp order (spread_warp)
  u64 conj;           // Z: sign mask XORed into Im(C) -- 1<<63 uses conj(C) (NEXT N2)
  long long lda, ldb; // row strides (elements) of A and B (= M, N when dense)
  int gather;         // kernel 4: strided rows of A copied element-wise, B stored element-wise (N4)
};

// TSMM: the C the kernels multiply by, C' = alpha * (conj ? conj(c) : c).
// alpha = 1 + 0i leaves C bit-exact (and NaN/Inf untouched).
__device__ __forceinline__ void c_prime(const TsmmArgs& p, double& re, double& im) {
  im = flip_sign(im, p.conj);
  if (p.alpha_im == 0.0) {
    re *= p.alpha_re;
    im *= p.alpha_re;
  } else {
    const double r = p.alpha_re * re - p.alpha_im * im;
    im = p.alpha_re * im + p.alpha_im * re;
    re = r;
  }
}
// B rows out of smem staging: store, or add into B (update mode)
__device__ __forceinline__ void b_out_bulk(const TsmmArgs& p, void* dst, const void* src, u32 bytes) {
  if (p.reduce)
    bulk_red_add(dst, src, bytes);
  else
    bulk_s2g(dst, src, bytes);
}
__device__ __forceinline__ void b_out_tma(const TsmmArgs& p, int x, int y, const void* src) {
  if (p.reduce)
    tma_red_add_2d(&p.tmB, x, y, src);
  else
    tma_store_2d(&p.tmB, x, y, src);
}

// NTL: threads per row along n (interleaved columns), MSPLIT: lanes sharing
// one output that split the m-sum (butterfly-combined), U: rows per thread per
// pass (C reuse), NT: threads per block, R: rows per chunk.
template <int M_, int N_, bool Z_, int NTL_, int MSPLIT_, int U_, int NT_, int R_>
struct TsmmCfg {
  static constexpr int M = M_, N = N_, NTL = NTL_, MSPLIT = MSPLIT_, U = U_, NT = NT_, R = R_;
  static constexpr bool Z = Z_;
  static constexpr int S = Z ? 2 : 1;
  static constexpr int TN = (N + NTL - 1) / NTL;      // outputs per thread per row
  static constexpr int MQ = (M + MSPLIT - 1) / MSPLIT;  // m terms per thread
  static constexpr int GS = NTL * MSPLIT;               // threads per row group
  static constexpr int RB = NT / GS;                    // row slots per block
  static constexpr int ROWS_PER_PASS = RB * U;
  static constexpr int A_STAGE_DOUBLES = R * M * S;
  static constexpr int OUT_DOUBLES = ROWS_PER_PASS * N * S;  // one pass, double-buffered
  static constexpr int C_DOUBLES = M * N * S;
  static_assert(NT % 32 == 0 && NT % GS == 0, "GS must divide NT");
  static_assert((GS & (GS - 1)) == 0 && GS <= 32, "GS power of two <= 32");
  static_assert((MSPLIT & (MSPLIT - 1)) == 0 && MSPLIT <= 32, "MSPLIT power of two <= 32");
  static_assert(R % ROWS_PER_PASS == 0 && ROWS_PER_PASS % 2 == 0,
                "R multiple of rows per pass; passes of even rows (16-byte bulk stores)");
  static_assert(NTL <= N && MSPLIT <= M, "no empty lanes");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmm_kernel(const TsmmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NT = Cfg::NT;
  constexpr int NTL = Cfg::NTL, MSPLIT = Cfg::MSPLIT, U = Cfg::U, TN = Cfg::TN, MQ = Cfg::MQ;
  constexpr int GS = Cfg::GS, RB = Cfg::RB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  double* sC = reinterpret_cast<double*>(smem_raw + 128);
  constexpr int C_PAD = ((Cfg::C_DOUBLES + 15) / 16) * 16;  // keep 128 B alignment
  double* sOut = sC + C_PAD;                                 // 2 x OUT_DOUBLES
  double* ring = sOut + 2 * Cfg::OUT_DOUBLES;                // stages x A_STAGE_DOUBLES

  const int tid = threadIdx.x;
  const int g = tid % GS;
  const int ms = g % MSPLIT;
  const int tn = g / MSPLIT;
  const int rs = tid / GS;
  const long long K = p.K;
  const long long K_even = K & ~1LL;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  // S1: stage C' = alpha * C (conj for N2) once per persistent block.
  for (int i = tid; i < M * N; i += NT) {
    if constexpr (Cfg::Z) {
      double re = __ldg(&p.C[2 * i]), im = __ldg(&p.C[2 * i + 1]);
      c_prime(p, re, im);
      sC[2 * i] = re;
      sC[2 * i + 1] = im;
    } else {
      sC[i] = p.alpha_re * __ldg(&p.C[i]);
    }
  }
  __syncthreads();

  u64 pol = 0;
  auto issue = [&](long long c, int s) {
    const long long r0 = c * R;
    const long long rows = (K_even - r0 < R) ? (K_even - r0) : R;
    const u32 ba = static_cast<u32>(rows * M * S * 8);
    double* dA = ring + static_cast<long long>(s) * Cfg::A_STAGE_DOUBLES;
    mbar_arrive_expect_tx(&full[s], ba);
    bulk_g2s(dA, p.A + r0 * M * S, ba, &full[s], pol);
  };
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < stages; s++) {
      const long long c = blockIdx.x + static_cast<long long>(s) * G;
      if (c < p.nchunks) issue(c, s);
    }
  }

  // Compute U rows x TN columns for rows r_u = base + rs + u*RB.
  auto compute_pass = [&](const double* __restrict__ sA, int base, int rows, double* out) {
    double acc[U][TN][S];
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int j = 0; j < TN; j++)
#pragma unroll
        for (int q = 0; q < S; q++) acc[u][j][q] = 0.0;
#pragma unroll 4
    for (int qm = 0; qm < MQ; qm++) {
      const int m = ms + qm * MSPLIT;
      const bool mv = ((qm + 1) * MSPLIT <= M) || (m < M);
      if constexpr (!Cfg::Z) {
        double cv[TN], av[U];
#pragma unroll
        for (int j = 0; j < TN; j++) {
          const int n = tn + j * NTL;
          cv[j] = (mv && n < N) ? sC[m * N + n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int r = base + rs + u * RB;
          av[u] = (mv && r < rows) ? sA[r * M + m] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
          for (int j = 0; j < TN; j++) acc[u][j][0] = fma(av[u], cv[j], acc[u][j][0]);
      } else {
        const double2* sC2 = reinterpret_cast<const double2*>(sC);
        const double2* sA2 = reinterpret_cast<const double2*>(sA);
        double2 cv[TN], av[U];
#pragma unroll
        for (int j = 0; j < TN; j++) {
          const int n = tn + j * NTL;
          cv[j] = (mv && n < N) ? sC2[m * N + n] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int r = base + rs + u * RB;
          av[u] = (mv && r < rows) ? sA2[r * M + m] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
          for (int j = 0; j < TN; j++)
            zfma(acc[u][j][0], acc[u][j][1], av[u].x, av[u].y, cv[j].x, cv[j].y);
      }
    }
    if constexpr (MSPLIT > 1) {
#pragma unroll
      for (int off = 1; off < MSPLIT; off <<= 1)
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
          for (int j = 0; j < TN; j++)
#pragma unroll
            for (int q = 0; q < S; q++)
              acc[u][j][q] += __shfl_xor_sync(0xffffffffu, acc[u][j][q], off);
    }
    // rows are pass-local in `out` (the staging buffer holds one pass)
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int r = base + rs + u * RB;
#pragma unroll
      for (int j = 0; j < TN; j++) {
        const int n = tn + j * NTL;
        if (r < rows && n < N && (j % MSPLIT) == ms) {
#pragma unroll
          for (int q = 0; q < S; q++) out[((r - base) * N + n) * S + q] = acc[u][j][q];
        }
      }
    }
  };

  Ring ring_it;
  int pass = 0;  // global pass counter -> output buffer parity
  for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
    const int s = ring_it.s;
    mbar_wait(&full[s], ring_it.ph);
    const double* sA = ring + static_cast<long long>(s) * Cfg::A_STAGE_DOUBLES;
    const long long r0 = c * R;
    const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
#pragma unroll 1
    for (int base = 0; base < rows; base += Cfg::ROWS_PER_PASS, pass++) {
      double* out = sOut + (pass & 1) * Cfg::OUT_DOUBLES;
      if (tid == 0) bulk_wait_read<1>();  // the store of pass-2 has read this buffer
      __syncthreads();
      compute_pass(sA, base, rows, out);
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
      __syncthreads();           // pass complete (and, on the last pass, stage s consumed)
      if (tid == 0) {
        const int prow = (rows - base < Cfg::ROWS_PER_PASS) ? rows - base : Cfg::ROWS_PER_PASS;
        b_out_bulk(p, p.B + (r0 + base) * N * S, out, static_cast<u32>(prow * N * S * 8));
        bulk_commit();
      }
    }
    if (tid == 0) {
      const long long c2 = c + static_cast<long long>(stages) * G;
      if (c2 < p.nchunks) issue(c2, s);
    }
  }
  // Odd last row (K odd): block 0 computes it from global A and smem C.
  if ((K & 1) && blockIdx.x == 0) {
    const double* a = p.A + (K - 1) * M * S;
    for (int n = tid; n < N; n += NT) {
      if constexpr (!Cfg::Z) {
        double s0 = 0.0;
        for (int m = 0; m < M; m++) s0 = fma(a[m], sC[m * N + n], s0);
        double* o = p.B + (K - 1) * N + n;
        *o = p.reduce ? *o + s0 : s0;
      } else {
        double re = 0.0, im = 0.0;
        for (int m = 0; m < M; m++)
          zfma(re, im, a[2 * m], a[2 * m + 1], sC[2 * (m * N + n)], sC[2 * (m * N + n) + 1]);
        double* o = p.B + 2 * ((K - 1) * N + n);
        o[0] = p.reduce ? o[0] + re : re;
        o[1] = p.reduce ? o[1] + im : im;
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

// ==========================================================================
// TSMM on the FP64 tensor pipe (DMMA.8x8x4)
// ==========================================================================
// B rows are computed as (8 rows x 8 n) blocks: B_blk += A_blk (8 rows x 4 m)
// * C_blk (4 m x 8 n), mma.sync m8n8k4 .row.col:
//   MMA-A  lane holds A[r0+g][m0+q]      (from the A stage, row stride AP)
//   MMA-B  lane holds C[m0+q][n0+g]      (from smem C, row stride NCP, zero padded)
//   acc    lane holds B[r0+g][n0+2q+e]   (e = 0, 1)
// Each consumer warp owns WR row blocks x all NB column blocks of a pass and
// writes its own rows: registers -> per-warp smem staging -> cp.async.bulk
// stores (one contiguous store, or one per row when the staging rows are
// padded).  Row strides are chosen (tools/gen_instances.py) so fragment loads
// and accumulator stores hit the minimum number of smem wavefronts; padded A
// rows are filled by one cp.async.bulk per row from the producer warp.
// TMA = true: A arrives by 2-D tensor copies into 128B-swizzled 16-double
// boxes (conflict-free fragments, rows past K zero-filled) and every warp
// writes its output rows into swizzled staging boxes that one TMA tensor store
// per box moves to B (rows past K are clipped by the TMA unit).  AP / NOP are
// ignored; requires M*S and N*S even and >= 16 doubles.
template <int M_, int N_, bool Z_, int WR_, int NW_, int R_, int AP_, int NOP_, bool TMA_ = false>
struct TsmmMmaCfg {
  static constexpr int M = M_, N = N_, WR = WR_, NW = NW_, R = R_;
  static constexpr bool Z = Z_, TMA = TMA_;
  static constexpr int S = Z ? 2 : 1;
  static constexpr int MK = (M + 3) / 4;  // k-steps over m
  static constexpr int NB = (N + 7) / 8;  // 8-column blocks
  static constexpr int NBA = (M * S + 15) / 16, NBO = (N * S + 15) / 16;  // TMA boxes per row
  static constexpr int AP = TMA ? NBA * 16 / S : AP_;
  static constexpr int NOP = TMA ? NBO * 16 / S : NOP_;
  // C row stride (elements), = 4 mod 8 units: the MMA-B fragment (rows q,
  // columns g) of each 16-lane half-warp (D LDS.64) / 8-lane quarter (Z
  // LDS.128) then hits distinct banks (ncu r4: 8 mod 16 left the D loads 2-way)
  static constexpr int NCP = 8 * NB + 4;
  static constexpr int RW = 8 * WR;        // rows per warp per pass
  static constexpr int RPP = RW * NW;      // rows per pass
  static constexpr int NT = (NW + 1) * 32;
  static constexpr bool CREG = MK * NB * S <= 32;  // C fragments held in registers
  static constexpr int C_DOUBLES = MK * 4 * NCP * S;
  static constexpr int OUT_DOUBLES = RW * NOP * S;  // per warp
  static constexpr int STAGE_DOUBLES = R * AP * S;
  static_assert(R % RPP == 0 && R % 2 == 0, "R must be a multiple of the rows per pass");
  static_assert(AP >= M && NOP >= N, "strides must cover the rows");
  static_assert(AP == M || ((AP * S) % 2 == 0 && (M * S) % 2 == 0),
                "padded A rows: 16-byte aligned rows of 16-byte multiple size");
  static_assert(NOP == N || ((NOP * S) % 2 == 0 && (N * S) % 2 == 0),
                "padded output rows: 16-byte aligned rows of 16-byte multiple size");
  static_assert(!TMA || ((M * S) % 2 == 0 && (N * S) % 2 == 0 && M * S >= 16 && N * S >= 16),
                "TMA tensor path: 16-byte rows of >= 128 bytes");
  static_assert(!TMA || (R % 8 == 0 && R <= 256 && RW <= 256), "TMA box rows");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmm_mma_kernel(const __grid_constant__ TsmmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NW = Cfg::NW, WR = Cfg::WR;
  constexpr int AP = Cfg::AP, NOP = Cfg::NOP, MK = Cfg::MK, NB = Cfg::NB, NCP = Cfg::NCP;
  constexpr int RW = Cfg::RW, RPP = Cfg::RPP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  u64* empty = full + 16;
  double* sC = reinterpret_cast<double*>(smem_raw + 256);
  // staging and ring start on 1024-byte boundaries (128B swizzle atoms)
  const int after_c = 256 + ((Cfg::C_DOUBLES + 15) / 16) * 16 * 8;  // byte offsets
  double* sOut = reinterpret_cast<double*>(smem_raw + (Cfg::TMA ? align1024(smem_raw, after_c) : after_c));
  unsigned char* after_o = reinterpret_cast<unsigned char*>(sOut + ((NW * Cfg::OUT_DOUBLES + 15) / 16) * 16);
  double* ring = reinterpret_cast<double*>(
      after_o + (Cfg::TMA ? align1024(after_o, 0) : 0));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  // swizzled (TMA) boxes: MMA row g <-> A/B row rho(g), conflict-free (see tsmm_cst_kernel);
  // dense odd D strides with WR even: 16-row windows (win16_row)
  const int rho = Cfg::TMA ? ((((g & 1) << 2) | (g & 2) | (g >> 2)) ^ (g & 1)) : g;
  constexpr bool WIN16 = !Cfg::TMA && !Cfg::Z && Cfg::WR % 2 == 0 && Cfg::AP % 2 == 1;
  auto prow = [&](int i) -> int {  // pass row of MMA row g of block i
    if constexpr (WIN16)
      return win16_row(Cfg::AP, i, g);
    else
      return 8 * i + rho;
  };
  const long long K = p.K;
  const long long K_even = K & ~1LL;
  const long long Kc = Cfg::TMA ? K : K_even;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  // S1: C' = alpha * C (conj for N2) -> smem once, zero padded to MK*4 rows x NCP columns
  for (int i = tid; i < MK * 4 * NCP; i += Cfg::NT) {
    const int m = i / NCP, n = i % NCP;
    double re = 0.0, im = 0.0;
    if (m < M && n < N) {
      re = __ldg(&p.C[(m * N + n) * S]);
      if constexpr (Cfg::Z) im = __ldg(&p.C[(m * N + n) * S + 1]);
      c_prime(p, re, im);
    }
    sC[i * S] = re;
    if constexpr (Cfg::Z) sC[i * S + 1] = im;
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer warp ----------------
    const u64 pol = policy_evict_first();
    Ring ring_it;
    for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
      const int s = ring_it.s;
      if (ring_it.round > 0 && lane == 0) mbar_wait(&empty[s], ring_it.ph ^ 1u);
      __syncwarp();
      const long long r0 = c * R;
      double* dA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
      if constexpr (Cfg::TMA) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], static_cast<u32>(Cfg::NBA * R * 128));
          for (int b = 0; b < Cfg::NBA; b++)
            tma_load_2d(dA + b * R * 16, &p.tmA, b * 16, static_cast<int>(r0), &full[s], pol);
        }
      } else {
        const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<u32>(rows * M * S * 8));
        __syncwarp();
        if constexpr (AP == M) {
          if (lane == 0) bulk_g2s(dA, p.A + r0 * M * S, static_cast<u32>(rows * M * S * 8), &full[s], pol);
        } else {
          for (int r = lane; r < rows; r += 32)
            bulk_g2s(dA + r * AP * S, p.A + (r0 + r) * M * S, static_cast<u32>(M * S * 8), &full[s], pol);
        }
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    double* stg = sOut + warp * Cfg::OUT_DOUBLES;
    // C fragments (MMA-B): lane holds C[4ks+q][8j+g]
    double creg[Cfg::CREG ? MK : 1][Cfg::CREG ? NB : 1][S];
    if constexpr (Cfg::CREG) {
#pragma unroll
      for (int ks = 0; ks < MK; ks++)
#pragma unroll
        for (int j = 0; j < NB; j++)
#pragma unroll
          for (int z = 0; z < S; z++) creg[ks][j][z] = sC[((4 * ks + q) * NCP + 8 * j + g) * S + z];
    }
    // offset (doubles) of element (row r, column x): dense / padded rows, or swizzled boxes
    auto aoff = [&](int r, int x) -> int {
      if constexpr (Cfg::TMA)
        return ((x * S) >> 4) * (R * 16) + swz128(r, (x * S) & 15);
      else
        return (r * AP + x) * S;
    };
    auto ooff = [&](int r, int x) -> int {  // output staging (rows of this warp)
      if constexpr (Cfg::TMA)
        return ((x * S) >> 4) * (RW * 16) + swz128(r, (x * S) & 15);
      else
        return (r * NOP + x) * S;
    };
    Ring ring_it;
    for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
      const int s = ring_it.s;
      mbar_wait(&full[s], ring_it.ph);
      const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
      const long long r0 = c * R;
      const int rows = static_cast<int>((Kc - r0 < R) ? (Kc - r0) : R);
#pragma unroll 1
      for (int pr = 0; pr < rows; pr += RPP) {
        const int wr0 = pr + warp * RW;
        if (wr0 >= rows) break;
        double acc[WR][NB][S][2];
#pragma unroll
        for (int i = 0; i < WR; i++)
#pragma unroll
          for (int j = 0; j < NB; j++)
#pragma unroll
            for (int z = 0; z < S; z++) acc[i][j][z][0] = acc[i][j][z][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < MK; ks++) {
          const int m = 4 * ks + q;
          const bool mv = (4 * ks + 4 <= M) || (m < M);
          double a[WR][S];
#pragma unroll
          for (int i = 0; i < WR; i++) {
            const int r = wr0 + prow(i);
#pragma unroll
            for (int z = 0; z < S; z++) a[i][z] = mv ? sA[aoff(r, m) + z] : 0.0;
          }
          double cf[NB][S];
#pragma unroll
          for (int j = 0; j < NB; j++)
#pragma unroll
            for (int z = 0; z < S; z++) {
              if constexpr (Cfg::CREG)
                cf[j][z] = creg[ks][j][z];
              else
                cf[j][z] = sC[((4 * ks + q) * NCP + 8 * j + g) * S + z];
            }
#pragma unroll
          for (int i = 0; i < WR; i++) {
            if constexpr (!Cfg::Z) {
#pragma unroll
              for (int j = 0; j < NB; j++) dmma(acc[i][j][0][0], acc[i][j][0][1], a[i][0], cf[j][0]);
            } else {
              const double nai = -a[i][1];
#pragma unroll
              for (int j = 0; j < NB; j++) {
                dmma(acc[i][j][0][0], acc[i][j][0][1], a[i][0], cf[j][0]);  // re += ar cr
                dmma(acc[i][j][0][0], acc[i][j][0][1], nai, cf[j][1]);      // re -= ai ci
                dmma(acc[i][j][1][0], acc[i][j][1][1], a[i][0], cf[j][1]);  // im += ar ci
                dmma(acc[i][j][1][0], acc[i][j][1][1], a[i][1], cf[j][0]);  // im += ai cr
              }
            }
          }
        }
        // S4: registers -> staging (after this warp's previous stores read it)
        bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int i = 0; i < WR; i++)
#pragma unroll
          for (int j = 0; j < NB; j++) {
            const int n = 8 * j + 2 * q;
            const int rr = prow(i);
            if constexpr (!Cfg::Z && (Cfg::TMA || NOP % 2 == 0)) {
              // 16-byte store (conflict-free: NOP = 2 mod 4, or swizzled boxes)
              double* dst = stg + ooff(rr, n);
              if (n + 1 < N || (Cfg::TMA && n < NOP))
                *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0][0], acc[i][j][0][1]);
              else if (n < N)
                dst[0] = acc[i][j][0][0];
            } else {
#pragma unroll
              for (int e = 0; e < 2; e++) {
                if (n + e < N) {
                  if constexpr (Cfg::Z) {
                    *reinterpret_cast<double2*>(stg + ooff(rr, n + e)) =
                        make_double2(acc[i][j][0][e], acc[i][j][1][e]);
                  } else {
                    stg[ooff(rr, n + e)] = acc[i][j][0][e];
                  }
                }
              }
            }
          }
        fence_proxy_async_smem();
        __syncwarp();
        const int nr = (rows - wr0 < RW) ? rows - wr0 : RW;
        if constexpr (Cfg::TMA) {
          if (lane == 0) {
            for (int b = 0; b < Cfg::NBO; b++)
              b_out_tma(p, b * 16, static_cast<int>(r0 + wr0), stg + b * RW * 16);
            bulk_commit();
          }
        } else if constexpr (NOP == N) {
          if (lane == 0) {
            b_out_bulk(p, p.B + (r0 + wr0) * N * S, stg, static_cast<u32>(nr * N * S * 8));
            bulk_commit();
          }
        } else {
          for (int r = lane; r < nr; r += 32)
            b_out_bulk(p, p.B + (r0 + wr0 + r) * N * S, stg + r * NOP * S, static_cast<u32>(N * S * 8));
          bulk_commit();
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // Odd last row (K odd, bulk-copy kernels): warp 0 of block 0, plain fma.
    if (!Cfg::TMA && (K & 1) && blockIdx.x == 0 && warp == 0) {
      const double* a = p.A + (K - 1) * M * S;
      for (int n = lane; n < N; n += 32) {
        if constexpr (!Cfg::Z) {
          double s0 = 0.0;
          for (int m = 0; m < M; m++) s0 = fma(a[m], sC[m * NCP + n], s0);
          double* o = p.B + (K - 1) * N + n;
          *o = p.reduce ? *o + s0 : s0;
        } else {
          double re = 0.0, im = 0.0;
          for (int m = 0; m < M; m++)
            zfma(re, im, a[2 * m], a[2 * m + 1], sC[2 * (m * NCP + n)], sC[2 * (m * NCP + n) + 1]);
          double* o = p.B + 2 * ((K - 1) * N + n);
          o[0] = p.reduce ? o[0] + re : re;
          o[1] = p.reduce ? o[1] + im : im;
        }
      }
    }
    bulk_wait_all();
  }
}

// --------------------------------------------------------------------------
// TSMM, "C-stationary" DMMA kernel (impl 3).  The N columns of B are split
// into NG column groups of NBW 8-column blocks; a consumer warp serves one
// column group and keeps ITS slice of C as MMA-B fragments in registers for
// the whole kernel (MK x NBW fragments: the paper's "C in registers",
// PAPER.md:701-703, made affordable by distributing C over warps).  Per
// k-step a warp loads only A fragments (128B-swizzled TMA boxes:
// conflict-free) for WR row blocks and issues WR*NBW DMMAs.  Each warp writes
// its (8*WR rows x 8*NBW columns) tile to a private swizzled staging box and
// stores it with one TMA tensor store per 16-double box -- no cross-warp
// barrier; rows past K and columns past N are clipped by the TMA unit.
// Requires the TMA conditions (M*S, N*S even and >= 16) and 8*NBW*S a
// multiple of 16 doubles (whole output boxes per warp).
// --------------------------------------------------------------------------
// EC > 0 ("edge columns", kernel | 16): the last EC = N mod 8 columns are
// computed with DFMA by the warps of the last column group (each lane adds its
// m = 4ks+q terms, a 4-lane butterfly finishes the sum) instead of padding a
// whole 8-column DMMA block; C' of those columns is staged in smem.
template <int M_, int N_, bool Z_, int NBW_, int WR_, int NW_, int R_, bool ZR_ = false, int EC_ = 0,
          bool G3_ = false>
struct TsmmCstCfg {
  static constexpr int M = M_, N = N_, NBW = NBW_, WR = WR_, NW = NW_, R = R_, EC = EC_;
  static constexpr bool Z = Z_, ZR = ZR_, G3 = G3_;
  static_assert(!G3 || Z_, "3M (Gauss) products: complex kernel");
  static_assert(!ZR || (!Z_ && M_ % 2 == 0 && N_ % 2 == 0), "complex-as-real: real kernel on 2M x 2N");
  static_assert(EC == 0 || (EC == N % 8 && N >= 8), "edge columns: EC = N mod 8, N >= 8");
  static constexpr int S = Z ? 2 : 1;
  static constexpr int NA = G3 ? 3 : S;             // C fragments / accumulators per block (3M: 3)
  static constexpr int MK = (M + 3) / 4;            // k-steps over m
  static constexpr int NB = (N - EC + 7) / 8;       // 8-column DMMA blocks of B
  static constexpr int NG = (NB + NBW - 1) / NBW;   // column groups
  static constexpr int RG = NW / NG;                // warps per column group
  static constexpr int RW = 8 * WR;                 // rows per warp per pass
  static constexpr int RPP = RW * RG;               // rows per pass
  static constexpr int NBA = (M * S + 15) / 16;     // A boxes per row
  static constexpr int OB = NBW * 8 * S / 16;       // output boxes per warp
  static constexpr int NBL = NB - (NG - 1) * NBW;   // DMMA blocks of the last column group
  static constexpr int OBL = ((8 * NBL + EC) * S + 15) / 16;  // its boxes (incl. edge columns)
  static constexpr int NT = (NW + 1) * 32;
  // 3M C slices: Re c, Im c and Re c + Im c are MK x NBW x 3 doubles per lane.
  // When they and the accumulators do not fit the registers ptxas grants a
  // thread under __launch_bounds__(NT) (65536 over NT rounded up to 128
  // threads, in steps of 8: 96 at NT = 544), the sum is recomputed per k-step
  // (one DADD per block, FP64 pipe) instead of kept: ptxas otherwise spills the
  // slice to local memory inside the k-loop (Z 64, NW 16: 192 -> 32 B of
  // spill stores, Z 57 WR 2: 276 -> 168 B; long_sb 12 % of the stall
  // samples of Z 64, ncu run 13).
  static constexpr int CF_REGS = MK * NBW * 3 * 2, ACC_REGS = WR * NBW * 3 * 4;
  static constexpr int REG_BUDGET = (65536 / (((NT + 127) / 128) * 128)) & ~7;
  static constexpr bool G3R = G3 && CF_REGS + ACC_REGS + 40 > REG_BUDGET;
  static constexpr int NCF = G3 ? (G3R ? 2 : 3) : S;  // C fragments held per block
  static constexpr int STAGE_DOUBLES = R * NBA * 16;
  static constexpr int OUT_DOUBLES = (OB > OBL ? OB : OBL) * RW * 16;  // per warp
  static constexpr int CE_DOUBLES = ((MK * 4 * EC * S + 127) / 128) * 128;  // edge C' in smem
  static_assert(NW % NG == 0 && RG >= 1, "consumer warps must be a multiple of the column groups");
  static_assert((NBW * 8 * S) % 16 == 0, "a warp's columns must fill whole 16-double boxes");
  static_assert((M * S) % 2 == 0 && (N * S) % 2 == 0 && M * S >= 16 && N * S >= 16,
                "TMA tensor path: 16-byte rows of >= 128 bytes");
  static_assert(R % RPP == 0 && R % 8 == 0 && R <= 256 && RW <= 256, "TMA box rows");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmm_cst_kernel(const __grid_constant__ TsmmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NW = Cfg::NW, WR = Cfg::WR;
  constexpr int MK = Cfg::MK, NB = Cfg::NB, NBW = Cfg::NBW, NG = Cfg::NG, RW = Cfg::RW;
  constexpr int RPP = Cfg::RPP, OB = Cfg::OB, EC = Cfg::EC, NA = Cfg::NA;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  u64* empty = full + 16;
  double* sCe = reinterpret_cast<double*>(smem_raw + 256);  // [MK*4][EC] edge columns of C'
  double* sOut = reinterpret_cast<double*>(smem_raw + align1024(smem_raw, 256 + Cfg::CE_DOUBLES * 8));
  double* ring = sOut + NW * Cfg::OUT_DOUBLES;  // multiple of 1024 bytes

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const long long K = p.K;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  if constexpr (EC > 0) {  // edge columns of C' (rows >= M zero)
    for (int i = tid; i < MK * 4 * EC; i += Cfg::NT) {
      const int m = i / EC, n = (N - EC) + i % EC;
      double re = 0.0, im = 0.0;
      if (m < M) {
        if constexpr (Cfg::ZR) {
          const double* c2 = p.C + ((m >> 1) * (N >> 1) + (n >> 1)) * 2;
          double cr = __ldg(c2), ci = __ldg(c2 + 1);
          c_prime(p, cr, ci);
          re = ((m & 1) == (n & 1)) ? cr : ((m & 1) ? -ci : ci);
        } else {
          re = __ldg(&p.C[(m * N + n) * S]);
          if constexpr (Cfg::Z) im = __ldg(&p.C[(m * N + n) * S + 1]);
          c_prime(p, re, im);
        }
      }
      sCe[i * S] = re;
      if constexpr (Cfg::Z) sCe[i * S + 1] = im;
    }
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer warp: TMA boxes of A ----------------
    if (lane == 0) {
      const u64 pol = policy_evict_first();
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        if (ring_it.round > 0) mbar_wait(&empty[s], ring_it.ph ^ 1u);
        double* dA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
        mbar_arrive_expect_tx(&full[s], static_cast<u32>(Cfg::NBA * R * 128));
        for (int b = 0; b < Cfg::NBA; b++)
          tma_load_2d(dA + b * R * 16, &p.tmA, b * 16, static_cast<int>(c * R), &full[s], pol);
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    const int wl = spread_warp(warp, NW, p.order);
    const int cg = wl % NG, rg = wl / NG;
    const int nb0 = cg * NBW;  // first 8-column block of this warp
    // MMA row g of a block is A/B row rho(g) = bitrev3(g) ^ (g & 1) =
    // [0,5,2,7,1,4,3,6]: under the 128B swizzle the A fragment loads (D: 16
    // lanes per 8-byte phase, Z: 8 lanes per 16-byte phase) and the 16-byte
    // staging stores then touch distinct banks (identity rows: 2-way conflicts).
    const int rho = ((((g & 1) << 2) | (g & 2) | (g >> 2)) ^ (g & 1));
    double* stg = sOut + warp * Cfg::OUT_DOUBLES;
    // this warp's C slice as MMA-B fragments: lane holds C[4ks+q][8(nb0+j)+g]
    // (3M: Re c, Im c, Re c + Im c)
    double cf[MK][NBW][Cfg::NCF];
#pragma unroll
    for (int ks = 0; ks < MK; ks++)
#pragma unroll
      for (int j = 0; j < NBW; j++) {
        const int m = 4 * ks + q, n = 8 * (nb0 + j) + g;
        if constexpr (Cfg::ZR) {
          // complex C as the real 2M x 2N matrix C' with B_real = A_real C':
          // C'[2m][2n] = C'[2m+1][2n+1] = Re c, C'[2m][2n+1] = Im c, C'[2m+1][2n] = -Im c
          double v = 0.0;
          if (m < M && n < N) {
            const double* c2 = p.C + ((m >> 1) * (N >> 1) + (n >> 1)) * 2;
            double re = __ldg(c2), im = __ldg(c2 + 1);
            c_prime(p, re, im);
            v = ((m & 1) == (n & 1)) ? re : ((m & 1) ? -im : im);
          }
          cf[ks][j][0] = v;
        } else {
#pragma unroll
          for (int z = 0; z < S; z++) cf[ks][j][z] = (m < M && n < N) ? __ldg(&p.C[(m * N + n) * S + z]) : 0.0;
          if constexpr (Cfg::Z) {
            c_prime(p, cf[ks][j][0], cf[ks][j][1]);
            if constexpr (Cfg::G3 && !Cfg::G3R) cf[ks][j][2] = cf[ks][j][0] + cf[ks][j][1];
          } else {
            cf[ks][j][0] *= p.alpha_re;
          }
        }
      }
    auto aoff = [&](int r, int x) -> int {  // element (row r, column x) of the A stage
      return ((x * S) >> 4) * (R * 16) + swz128(r, (x * S) & 15);
    };
    // blocks of this warp's column group inside C (the last group may be
    // partial): compile-time, so no DMMA is issued for columns past N
    auto consume = [&](auto nbv, auto ecv) {
      constexpr int NBV = decltype(nbv)::value;  // DMMA blocks of this group inside C
      constexpr int ECV = decltype(ecv)::value;  // DFMA edge columns (last group only)
      constexpr int ECA = ECV > 0 ? ECV : 1;
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        mbar_wait(&full[s], ring_it.ph);
        const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
        const long long r0 = c * R;
        const int rows = static_cast<int>((K - r0 < R) ? (K - r0) : R);
  #pragma unroll 1
        for (int pr = 0; pr < rows; pr += RPP) {
          const int wr0 = pr + rg * RW;
          if (wr0 >= rows) break;
          double acc[WR][NBW][NA][2];
  #pragma unroll
          for (int i = 0; i < WR; i++)
  #pragma unroll
            for (int j = 0; j < NBW; j++)
  #pragma unroll
              for (int z = 0; z < NA; z++) acc[i][j][z][0] = acc[i][j][z][1] = 0.0;
          double eacc[WR][ECA][S];
  #pragma unroll
          for (int i = 0; i < WR; i++)
  #pragma unroll
            for (int e = 0; e < ECA; e++)
  #pragma unroll
              for (int z = 0; z < S; z++) eacc[i][e][z] = 0.0;
  #pragma unroll
          for (int ks = 0; ks < MK; ks++) {
            const int m = 4 * ks + q;
            const bool mv = (4 * ks + 4 <= M) || (m < M);
            // G3R: Re c + Im c of this k-step, once for all WR > 1 row blocks
            // (volatile: recomputed every k-step, never kept live; with WR = 1
            // it stays next to its DMMA, which ptxas allocates better: Z 64
            // NT 544 32 B of spill stores instead of 72)
            constexpr bool HOIST = Cfg::G3R && WR > 1;
            double csum[HOIST ? NBV : 1];
            if constexpr (HOIST) {
  #pragma unroll
              for (int j = 0; j < NBV; j++) csum[j] = dadd_here(cf[ks][j][0], cf[ks][j][1]);
            }
  #pragma unroll
            for (int i = 0; i < WR; i++) {
              const int r = wr0 + 8 * i + rho;
              if constexpr (!Cfg::Z) {
                const double a = mv ? sA[aoff(r, m)] : 0.0;
  #pragma unroll
                for (int j = 0; j < NBV; j++) dmma(acc[i][j][0][0], acc[i][j][0][1], a, cf[ks][j][0]);
                if constexpr (ECV > 0) {
  #pragma unroll
                  for (int e = 0; e < ECV; e++) eacc[i][e][0] = fma(a, sCe[m * EC + e], eacc[i][e][0]);
                }
              } else {
                const double2 a = mv ? *reinterpret_cast<const double2*>(sA + aoff(r, m)) : make_double2(0.0, 0.0);
                if constexpr (Cfg::G3) {
                  // 3M: T1 += ar cr, T2 += ai ci, T3 += (ar + ai)(cr + ci)
                  const double sa = a.x + a.y;
  #pragma unroll
                  for (int j = 0; j < NBV; j++) {
                    dmma(acc[i][j][0][0], acc[i][j][0][1], a.x, cf[ks][j][0]);
                    dmma(acc[i][j][1][0], acc[i][j][1][1], a.y, cf[ks][j][1]);
                    if constexpr (HOIST)
                      dmma(acc[i][j][2][0], acc[i][j][2][1], sa, csum[j]);
                    else if constexpr (Cfg::G3R)
                      dmma(acc[i][j][2][0], acc[i][j][2][1], sa, dadd_here(cf[ks][j][0], cf[ks][j][1]));
                    else
                      dmma(acc[i][j][2][0], acc[i][j][2][1], sa, cf[ks][j][2]);
                  }
                } else {
                const double nai = -a.y;
  #pragma unroll
                for (int j = 0; j < NBV; j++) {
                  dmma(acc[i][j][0][0], acc[i][j][0][1], a.x, cf[ks][j][0]);  // re += ar cr
                  dmma(acc[i][j][0][0], acc[i][j][0][1], nai, cf[ks][j][1]);  // re -= ai ci
                  dmma(acc[i][j][1][0], acc[i][j][1][1], a.x, cf[ks][j][1]);  // im += ar ci
                  dmma(acc[i][j][1][0], acc[i][j][1][1], a.y, cf[ks][j][0]);  // im += ai cr
                }
                }
                if constexpr (ECV > 0) {
  #pragma unroll
                  for (int e = 0; e < ECV; e++) {
                    const double2 ce = *reinterpret_cast<const double2*>(sCe + (m * EC + e) * 2);
                    zfma(eacc[i][e][0], eacc[i][e][1], a.x, a.y, ce.x, ce.y);
                  }
                }
              }
            }
          }
          // registers -> private swizzled staging -> TMA tensor stores
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
  #pragma unroll
          for (int i = 0; i < WR; i++)
  #pragma unroll
            for (int j = 0; j < NBV; j++) {  // blocks past N: clipped by the TMA store
              const int rr = 8 * i + rho;
              if constexpr (!Cfg::Z) {
                const int c0 = 8 * j + 2 * q;  // column within the warp's tile (doubles)
                *reinterpret_cast<double2*>(stg + (c0 >> 4) * (RW * 16) + swz128(rr, c0 & 15)) =
                    make_double2(acc[i][j][0][0], acc[i][j][0][1]);
              } else {
  #pragma unroll
                for (int e = 0; e < 2; e++) {
                  const int c0 = 2 * (8 * j + 2 * q + e);
                  double re = acc[i][j][0][e], im = acc[i][j][1][e];
                  if constexpr (Cfg::G3) {  // re = T1 - T2, im = T3 - T1 - T2
                    re = acc[i][j][0][e] - acc[i][j][1][e];
                    im = acc[i][j][2][e] - acc[i][j][0][e] - acc[i][j][1][e];
                  }
                  *reinterpret_cast<double2*>(stg + (c0 >> 4) * (RW * 16) + swz128(rr, c0 & 15)) =
                      make_double2(re, im);
                }
              }
            }
          if constexpr (ECV > 0) {
            // edge columns: sum the 4 q-lanes' partial m-sums (fixed butterfly order)
  #pragma unroll
            for (int i = 0; i < WR; i++)
  #pragma unroll
              for (int e = 0; e < ECV; e++) {
                double v[S];
  #pragma unroll
                for (int z = 0; z < S; z++) {
                  v[z] = eacc[i][e][z];
                  v[z] += __shfl_xor_sync(0xffffffffu, v[z], 1);
                  v[z] += __shfl_xor_sync(0xffffffffu, v[z], 2);
                }
                if (q == 0) {
                  const int rr = 8 * i + rho, c0 = (8 * NBV + e) * S;
                  double* dst = stg + (c0 >> 4) * (RW * 16) + swz128(rr, c0 & 15);
                  if constexpr (S == 2)
                    *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[S - 1]);
                  else
                    dst[0] = v[0];
                }
              }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && nb0 < NB) {
            constexpr int NBOX = ECV > 0 ? Cfg::OBL : OB;
            for (int b = 0; b < NBOX; b++)
              b_out_tma(p, nb0 * 8 * S + b * 16, static_cast<int>(r0 + wr0), stg + b * RW * 16);
            bulk_commit();
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    };
    constexpr int NBL = NB - (NG - 1) * NBW;
    if (cg == NG - 1)
      consume(IC<NBL>{}, IC<EC>{});
    else
      consume(IC<NBW>{}, IC<0>{});
    if (lane == 0) bulk_wait_all();
  }
}

// --------------------------------------------------------------------------
// TSMM, C-stationary DMMA kernel with bulk copies (impl 4): the C-in-registers
// design of impl 3 for widths the TMA tensor path cannot take (odd D widths:
// rows are not 16-byte multiples; D widths < 16).  A arrives as one dense
// bulk copy per chunk (row stride M).  The NG warps of a row group write their
// column slices into a shared double-buffered staging block [RW rows][N], meet
// at a named barrier (id 1 + row group), and one lane stores the RW contiguous
// rows of B with a single bulk copy (or bulk reduce-add in update mode).
// Before that barrier the issuing lane waits until its previous store has read
// the other buffer, so a buffer is rewritten only after its store completed.
// --------------------------------------------------------------------------
// Row permutations rho(g) for the impl-4 A fragment (rows rho(g), columns q of
// a dense stride-M stage) and the worst lanes-per-bank-unit they give.
//   0: identity  1: [0,2,4,6,1,3,5,7]  2: [0,4,1,5,2,6,3,7]  3: bitrev [0,4,2,6,1,5,3,7]
__host__ __device__ constexpr int cstb_rho(int sel, int g) {
  return sel == 1 ? (((g & 3) << 1) | (g >> 2))
       : sel == 2 ? (((g & 1) << 2) | (g >> 1))
       : sel == 3 ? (((g & 1) << 2) | (g & 2) | (g >> 2))
                  : g;
}
constexpr int cstb_conflict(int sel, int M, bool z) {
  // D: two 16-lane phases of 8-byte units; Z: four 8-lane phases of 16-byte units
  const int lanes = z ? 8 : 16, units = z ? 8 : 16;
  int worst = 0;
  for (int ph = 0; ph < 32 / lanes; ph++) {
    int cnt[16] = {};
    for (int l = ph * lanes; l < ph * lanes + lanes; l++) {
      const int u = (cstb_rho(sel, l >> 2) * M + (l & 3)) % units;
      if (++cnt[u] > worst) worst = cnt[u];
    }
  }
  return worst;
}
// D output staging stores: lane (g, q) writes element (rho(g), 2q + e) of the
// dense [RW][N] block, one 8-byte store per e -> worst lanes per 8-byte unit
// over the two 16-lane phases.
constexpr int cstb_store_conflict(int sel, int N) {
  int worst = 0;
  for (int e = 0; e < 2; e++)
    for (int ph = 0; ph < 2; ph++) {
      int cnt[16] = {};
      for (int l = ph * 16; l < ph * 16 + 16; l++) {
        const int u = (cstb_rho(sel, l >> 2) * N + 2 * (l & 3) + e) % 16;
        if (++cnt[u] > worst) worst = cnt[u];
      }
    }
  return worst;
}
// Row permutation minimising the A fragment loads' conflicts (MK*WR loads per
// pass, weight 3) plus the D staging stores' (2*NBW*WR per pass, weight 1):
// ncu r32 showed the stores of D 63 4-way conflicted under the load-only choice.
constexpr int cstb_pick_rho(int M, int N, bool z) {
  int best = 0, bc = 1 << 20;
  for (int sel = 0; sel < 4; sel++) {
    const int c = 3 * cstb_conflict(sel, M, z) + (z ? 0 : cstb_store_conflict(sel, N));
    if (c < bc) {
      bc = c;
      best = sel;
    }
  }
  return best;
}

// EC > 0 (kernel | 16): the last EC = N mod 8 columns of B by DFMA in the
// warps of the last column group (as kernel 3's edge columns) instead of a
// padded 8-column DMMA block: D 57 costs 57 x 60 lane-FMAs per row instead of
// 64 x 60 on the shared FP64 pipe.
template <int M_, int N_, bool Z_, int NBW_, int WR_, int NW_, int R_, int EC_ = 0, bool GA_ = false>
struct TsmmCstbCfg {
  static constexpr int M = M_, N = N_, NBW = NBW_, WR = WR_, NW = NW_, R = R_, EC = EC_;
  static constexpr bool GA = GA_;  // gather-capable instantiation (kernel | 8192, see TsmttsmMmaCfg)
  static constexpr bool Z = Z_;
  static_assert(EC == 0 || (EC == N % 8 && N >= 8), "edge columns: EC = N mod 8, N >= 8");
  static constexpr int S = Z ? 2 : 1;
  static constexpr int MK = (M + 3) / 4;            // k-steps over m
  static constexpr int NB = (N - EC + 7) / 8;       // 8-column DMMA blocks of B
  static constexpr int NG = (NB + NBW - 1) / NBW;   // column groups
  static constexpr int RG = NW / NG;                // row groups (warps per column group)
  static constexpr int RW = 8 * WR;                 // rows per row group per pass
  static constexpr int RPP = RW * RG;               // rows per pass
  static constexpr int NT = (NW + 1) * 32;
  static constexpr int STAGE_DOUBLES = ((R * M * S + 15) / 16) * 16;
  static constexpr int OUT_DOUBLES = ((RW * N * S + 15) / 16) * 16;  // one staging buffer
  static constexpr int CE_DOUBLES = ((MK * 4 * EC * S + 15) / 16) * 16;  // edge columns of C' in smem
  static constexpr int RHO = cstb_pick_rho(M, N, Z);  // conflict-minimising row permutation
  static_assert(NW % NG == 0 && RG >= 1 && RG <= 15, "consumer warps: a multiple of the column groups, <= 15 row groups");
  static_assert(R % RPP == 0 && R % 2 == 0, "rows per chunk: whole passes");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT) tsmm_cstb_kernel(const __grid_constant__ TsmmArgs p) {
  constexpr int M = Cfg::M, N = Cfg::N, S = Cfg::S, R = Cfg::R, NW = Cfg::NW, WR = Cfg::WR;
  constexpr int MK = Cfg::MK, NB = Cfg::NB, NBW = Cfg::NBW, NG = Cfg::NG, RW = Cfg::RW;
  constexpr int RPP = Cfg::RPP, EC = Cfg::EC;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  u64* empty = full + 16;
  double* sCe = reinterpret_cast<double*>(smem_raw + 256);  // [MK*4][EC] edge columns of C'
  double* stage_out = sCe + Cfg::CE_DOUBLES;
  double* ring = stage_out + Cfg::RG * 2 * Cfg::OUT_DOUBLES;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const long long K = p.K;
  const long long K_even = K & ~1LL;
  const int G = gridDim.x;
  const int stages = p.stages;

  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], (Cfg::GA && p.gather) ? 32 : 1);  // gather: one noinc arrival per producer lane
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  if constexpr (EC > 0) {  // edge columns of C' (rows >= M zero)
    for (int i = tid; i < MK * 4 * EC; i += Cfg::NT) {
      const int m = i / EC, n = (N - EC) + i % EC;
      double re = 0.0, im = 0.0;
      if (m < M) {
        re = __ldg(&p.C[(m * N + n) * S]);
        if constexpr (Cfg::Z) im = __ldg(&p.C[(m * N + n) * S + 1]);
        c_prime(p, re, im);
      }
      sCe[i * S] = re;
      if constexpr (Cfg::Z) sCe[i * S + 1] = im;
    }
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer warp: one bulk copy per chunk of A ----------------
    if (Cfg::GA && p.gather) {  // strided rows of A (N4): element copies by the 32 lanes, any row stride
      if constexpr (Cfg::GA) {
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        if (ring_it.round > 0) mbar_wait(&empty[s], ring_it.ph ^ 1u);
        const long long r0 = c * R;
        const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
        gather_rows<M, S>(ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES, M, p.A, r0, p.lda, rows, lane);
        cp_async_mbar_arrive_noinc(&full[s]);
      }
      }
    } else if (lane == 0) {
      const u64 pol = policy_evict_first();
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        if (ring_it.round > 0) mbar_wait(&empty[s], ring_it.ph ^ 1u);
        const long long r0 = c * R;
        const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
        const u32 bytes = static_cast<u32>(rows * M * S * 8);
        double* dA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(dA, p.A + r0 * M * S, bytes, &full[s], pol);
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    const int wl = spread_warp(warp, NW, p.order);
    const int cg = wl % NG, rg = wl / NG;
    const int nb0 = cg * NBW;
    const bool issuer = (cg == 0 && lane == 0);
    const int rho = cstb_rho(Cfg::RHO, g);  // MMA row g <-> stage row rho(g) (bank conflicts)
    // D, odd M, WR even: 16-row windows instead (conflict-free A fragment loads)
    constexpr bool WIN16 = !Cfg::Z && WR % 2 == 0 && M % 2 == 1;
    auto prow = [&](int i) -> int {
      if constexpr (WIN16)
        return win16_row(M, i, g);
      else
        return 8 * i + rho;
    };
    // this warp's C' slice as MMA-B fragments: lane holds C'[4ks+q][8(nb0+j)+g]
    double cf[MK][NBW][S];
#pragma unroll
    for (int ks = 0; ks < MK; ks++)
#pragma unroll
      for (int j = 0; j < NBW; j++) {
        const int m = 4 * ks + q, n = 8 * (nb0 + j) + g;
        double re = 0.0, im = 0.0;
        if (m < M && n < N) {
          re = __ldg(&p.C[(m * N + n) * S]);
          if constexpr (Cfg::Z) im = __ldg(&p.C[(m * N + n) * S + 1]);
          c_prime(p, re, im);
        }
        cf[ks][j][0] = re;
        if constexpr (Cfg::Z) cf[ks][j][S - 1] = im;
      }
    auto consume = [&](auto nbv, auto ecv) {
      constexpr int NBV = decltype(nbv)::value;  // blocks of this column group inside C
      constexpr int ECV = decltype(ecv)::value;  // DFMA edge columns (last group only)
      constexpr int ECA = ECV > 0 ? ECV : 1;
      int pass = 0;
      Ring ring_it;
      for (long long c = blockIdx.x; c < p.nchunks; c += G, ring_it.next(stages)) {
        const int s = ring_it.s;
        mbar_wait(&full[s], ring_it.ph);
        const double* sA = ring + static_cast<long long>(s) * Cfg::STAGE_DOUBLES;
        const long long r0 = c * R;
        const int rows = static_cast<int>((K_even - r0 < R) ? (K_even - r0) : R);
#pragma unroll 1
        for (int pr = 0; pr < rows; pr += RPP) {
          const int wr0 = pr + rg * RW;
          if (wr0 >= rows) break;  // uniform across the row group
          double acc[WR][NBW][S][2];
#pragma unroll
          for (int i = 0; i < WR; i++)
#pragma unroll
            for (int j = 0; j < NBW; j++)
#pragma unroll
              for (int z = 0; z < S; z++) acc[i][j][z][0] = acc[i][j][z][1] = 0.0;
          double eacc[WR][ECA][S];
#pragma unroll
          for (int i = 0; i < WR; i++)
#pragma unroll
            for (int e = 0; e < ECA; e++)
#pragma unroll
              for (int z = 0; z < S; z++) eacc[i][e][z] = 0.0;
#pragma unroll
          for (int ks = 0; ks < MK; ks++) {
            const int m = 4 * ks + q;
            const bool mv = (4 * ks + 4 <= M) || (m < M);
#pragma unroll
            for (int i = 0; i < WR; i++) {
              const int r = wr0 + prow(i);  // rows past `rows`: stale, never stored
              if constexpr (!Cfg::Z) {
                const double a = mv ? sA[r * M + m] : 0.0;
#pragma unroll
                for (int j = 0; j < NBV; j++) dmma(acc[i][j][0][0], acc[i][j][0][1], a, cf[ks][j][0]);
                if constexpr (ECV > 0) {  // this lane's m-term of the edge columns (m >= M: C' row 0)
#pragma unroll
                  for (int e = 0; e < ECV; e++) eacc[i][e][0] = fma(a, sCe[m * EC + e], eacc[i][e][0]);
                }
              } else {
                const double2 a = mv ? *reinterpret_cast<const double2*>(sA + (r * M + m) * 2)
                                     : make_double2(0.0, 0.0);
                const double nai = -a.y;
#pragma unroll
                for (int j = 0; j < NBV; j++) {
                  dmma(acc[i][j][0][0], acc[i][j][0][1], a.x, cf[ks][j][0]);  // re += ar cr
                  dmma(acc[i][j][0][0], acc[i][j][0][1], nai, cf[ks][j][1]);  // re -= ai ci
                  dmma(acc[i][j][1][0], acc[i][j][1][1], a.x, cf[ks][j][1]);  // im += ar ci
                  dmma(acc[i][j][1][0], acc[i][j][1][1], a.y, cf[ks][j][0]);  // im += ai cr
                }
                if constexpr (ECV > 0) {
#pragma unroll
                  for (int e = 0; e < ECV; e++) {
                    const double2 ce = *reinterpret_cast<const double2*>(sCe + (m * EC + e) * 2);
                    zfma(eacc[i][e][0], eacc[i][e][1], a.x, a.y, ce.x, ce.y);
                  }
                }
              }
            }
          }
          // registers -> this row group's staging buffer (pass & 1), dense [RW][N]
          double* stg = stage_out + (rg * 2 + (pass & 1)) * Cfg::OUT_DOUBLES;
#pragma unroll
          for (int i = 0; i < WR; i++)
#pragma unroll
            for (int j = 0; j < NBV; j++)
#pragma unroll
              for (int e = 0; e < 2; e++) {
                const int rr = prow(i), n = 8 * (nb0 + j) + 2 * q + e;
                if (n < N) {
#pragma unroll
                  for (int z = 0; z < S; z++) stg[(rr * N + n) * S + z] = acc[i][j][z][e];
                }
              }
          if constexpr (ECV > 0) {
            // edge columns: sum the 4 q-lanes' partial m-sums (fixed butterfly order)
#pragma unroll
            for (int i = 0; i < WR; i++)
#pragma unroll
              for (int e = 0; e < ECV; e++) {
                double v[S];
#pragma unroll
                for (int z = 0; z < S; z++) {
                  v[z] = eacc[i][e][z];
                  v[z] += __shfl_xor_sync(0xffffffffu, v[z], 1);
                  v[z] += __shfl_xor_sync(0xffffffffu, v[z], 2);
                }
                if (q == 0) {
                  const int rr = prow(i), n = N - EC + e;
#pragma unroll
                  for (int z = 0; z < S; z++) stg[(rr * N + n) * S + z] = v[z];
                }
              }
          }
          fence_proxy_async_smem();
          if (issuer) bulk_wait_read<0>();  // the previous pass's store has read the other buffer
          // Named barrier of the row group.  Its warps reach it from different
          // instantiations of this lambda (the last column group's has other
          // block / edge counts), i.e. from different instructions, which the
          // .aligned form (bar.sync) forbids -- compute-sanitizer synccheck
          // flagged it -- so the non-aligned barrier.sync, after reconverging
          // the warp from the issuer-only wait.
          __syncwarp();
          asm volatile("barrier.sync %0, %1;" ::"r"(1 + rg), "r"(NG * 32) : "memory");
          if (Cfg::GA && p.gather) {
            // strided B (N4): the NG warps of the row group store the staged rows
            // element-wise (each element by one thread; update mode: B += value).
            // A buffer is rewritten two passes later, after the next pass's
            // barrier, which every thread reaches only after this loop.
            const int nr = (rows - wr0 < RW) ? rows - wr0 : RW;
            for (int i = cg * 32 + lane; i < nr * N; i += NG * 32) {
              const int r = i / N, n = i - r * N;
              double* o = p.B + ((r0 + wr0 + r) * p.ldb + n) * S;
#pragma unroll
              for (int z = 0; z < S; z++) o[z] = p.reduce ? o[z] + stg[i * S + z] : stg[i * S + z];
            }
          } else if (issuer) {
            const int nr = (rows - wr0 < RW) ? rows - wr0 : RW;
            b_out_bulk(p, p.B + (r0 + wr0) * N * S, stg, static_cast<u32>(nr * N * S * 8));
            bulk_commit();
          }
          pass++;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    };
    constexpr int NBL = NB - (NG - 1) * NBW;
    if (cg == NG - 1)
      consume(IC<NBL>{}, IC<EC>{});
    else
      consume(IC<NBW>{}, IC<0>{});
    if (issuer) bulk_wait_all();
    // Odd last row (K odd): warp 0 of block 0 from global A and C' (plain fma).
    if ((K & 1) && blockIdx.x == 0 && warp == 0) {
      const double* a = p.A + (K - 1) * p.lda * S;
      for (int n = lane; n < N; n += 32) {
        double re = 0.0, im = 0.0;
        for (int m = 0; m < M; m++) {
          double cr = __ldg(&p.C[(m * N + n) * S]), ci = 0.0;
          if constexpr (Cfg::Z) ci = __ldg(&p.C[(m * N + n) * S + 1]);
          c_prime(p, cr, ci);
          if constexpr (Cfg::Z) {
            zfma(re, im, a[2 * m], a[2 * m + 1], cr, ci);
          } else {
            re = fma(a[m], cr, re);
          }
        }
        double* o = p.B + ((K - 1) * p.ldb + n) * S;
        o[0] = p.reduce ? o[0] + re : re;
        if constexpr (Cfg::Z) o[1] = p.reduce ? o[1] + im : im;
      }
    }
  }
}

}  // namespace tsm
