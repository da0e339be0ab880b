/*
 * libtsm.h -- C ABI of libtsm, a B200-native (sm_100a) library for the two
 * tall & skinny matrix products of Ernst, Hager, Thies, Wellein,
 * "Performance Engineering for Real and Complex Tall & Skinny Matrix
 * Multiplication Kernels on GPUs" (arXiv 1905.03136; /root/reference/PAPER.md).
 *
 *   TSMTTSM   C = A^T B   PAPER.md:64-68 ("A^T B = C"), PAPER.md:342-349 (Listing 1):
 *             C[m][n] = sum_{k<K} A[k][m] * B[k][n]
 *   TSMM      B = A C     PAPER.md:64-68 ("A C = B"), PAPER.md:372-375:
 *             B[k][n] = sum_{m<M} A[k][m] * C[m][n]
 *
 * Sizes: 1 <= M, N <= 64 ("skinny"), K >= 1 ("tall" means
 * K > 10^6 but every K >= 1 is supported).
 *
 * Layout (all matrices): row-major and contiguous, leading dimension = width.
 *   A[k][m] at A + k*M + m (K x M), B[k][n] at B + k*N + n (K x N),
 *   C[m][n] at C + m*N + n (M x N)   -- PAPER.md:91 "row-major tall & skinny";
 *   C row-major is DESIGN.md reading R2.
 * Scalar types: D = IEEE double; Z = complex double as interleaved (re, im)
 * pairs (tsm_zcomplex; the layout of cuDoubleComplex and torch.complex128),
 * PAPER.md:70-72, 194-196.  The Z transpose is the PLAIN transpose -- no
 * conjugation of A in TSMTTSM and none of C in TSMM (reading R1).
 *
 * Memory ownership: every matrix / workspace pointer is caller-owned DEVICE
 * memory (e.g. a torch CUDA tensor) on the plan's device; the library never
 * allocates device memory.  Base pointers of A, B, C and the workspace must be
 * 16-byte aligned (TSM_ERR_MISALIGNED otherwise); outputs must not overlap
 * inputs (TSM_ERR_INVALID_VALUE).  Outputs are fully overwritten (beta = 0).
 *
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  Every call only enqueues work on that stream and returns without
 * synchronising the host; asynchronous device faults surface at the caller's
 * next synchronisation.  Calls on different streams are safe if each has its
 * own workspace.
 *
 * Determinism: for a fixed (plan, K, inputs, GPU model) results are bitwise
 * reproducible: the TSMTTSM reduction is a fixed-order two-level sum (no
 * floating-point atomics; the paper's atomics, are replaced
 * by a fixed-order grid reduction).  Different plans or K may
 * differ within the parity tolerance (|dC| <= 1e-12 |A|^T|B|,
 * |dB| <= 1e-13 |A||C|).
 *
 * Errors: every entry point returns tsm_status and never aborts, throws or
 * prints.  Arguments are validated before any launch; a failed launch maps to
 * TSM_ERR_CUDA.  tsm_last_error_detail() returns a thread-local description of
 * the last failure.
 */
#ifndef LIBTSM_H
#define LIBTSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSM_VERSION_MAJOR 0
#define TSM_VERSION_MINOR 1

typedef enum {
  TSM_SUCCESS = 0,
  TSM_ERR_INVALID_VALUE = 1, /* bad size, null pointer, overlap, op/dtype mismatch */
  TSM_ERR_UNSUPPORTED = 2,   /* shape/feature not available in this build */
  TSM_ERR_MISALIGNED = 3,    /* a base pointer is not 16-byte aligned */
  TSM_ERR_WORKSPACE = 4,     /* workspace missing or smaller than required */
  TSM_ERR_CUDA = 5,          /* CUDA runtime / launch error */
  TSM_ERR_NCCL = 6,          /* NCCL error or NCCL unavailable */
  TSM_ERR_INTERNAL = 7
} tsm_status;

typedef enum { TSM_OP_TSMTTSM = 0, TSM_OP_TSMM = 1 } tsm_op;
typedef enum { TSM_D = 0, TSM_Z = 1 } tsm_dtype;

typedef struct tsm_zcomplex {
  double re, im;
} tsm_zcomplex;

typedef struct tsm_plan_s *tsm_plan;
typedef struct tsm_comm_s *tsm_comm;
typedef void *tsm_stream; /* cudaStream_t */

/* ------------------------------------------------------------------------ */
/* Plans (pick the (M,N,type) instantiation    */
/* and its B200-tuned launch parameters).                                    */
/* ------------------------------------------------------------------------ */

/* Create a plan for one (op, dtype, M, N) on CUDA device `device`.
 * Selects the width-specialised kernel instantiated for exactly (M, N, dtype)
 * and its tuned launch parameters (tile, threads, pipeline depth, grid).
 * Benchmark shapes are compiled ahead of time; any other (M, N) is compiled
 * on first use by NVRTC (sm_100a) from the same C++ template and cached.
 * Errors: TSM_ERR_INVALID_VALUE (M or N outside [1,64], bad enum, out==NULL),
 *         TSM_ERR_UNSUPPORTED (shared memory / occupancy cannot be met),
 *         TSM_ERR_INTERNAL (run-time compilation failed),
 *         TSM_ERR_CUDA (device query failed).  The plan owns host state only;
 *         it is immutable and may be used from several threads. */
tsm_status tsm_plan_create(tsm_plan *out, tsm_op op, tsm_dtype dtype, int M, int N,
                           int device);

/* Kernel configuration of a plan (the autotuning space):
 *   TSMTTSM: p0 = MT, p1 = NTL: register tiles per row along m / n (powers of
 *            two <= M, N; tile = ceil(M/MT) x ceil(N/NTL) cells per thread,
 *            interleaved "transposed" mapping); p2 unused.
 *   TSMM:    p0 = NTL lanes along n (interleaved columns),
 *            p1 = MSPLIT lanes splitting the m-sum, p2 = U rows per thread
 *            (C reuse); NTL*MSPLIT <= 32, powers of two.
 *   threads: block size (multiple of 32); rows_per_chunk: rows per pipeline
 *   stage (even); stages: smem ring depth; ctas_per_sm: resident CTAs per SM
 *   (clipped by occupancy). */
typedef struct tsm_config {
  int threads;
  int rows_per_chunk;
  int p0, p1, p2;
  int stages;
  int ctas_per_sm;
  int kernel; /* 0 = register-tile DFMA kernel; 1 = DMMA kernel (FP64 tensor pipe,
                 mma.sync m8n8k4 f64; threads = 32 * (consumer warps + 1 producer warp)):
                 TSMTTSM: p0 = WM, p1 = WN 8x8 accumulator blocks per warp, p2 = AP,
                          p3 = BP smem row strides (elements) of A and B (= M, N: dense);
                          rows_per_chunk a multiple of 4.
                 TSMM:    p0 = WR 8-row blocks per warp, p1 = AP smem row stride of A,
                          p2 = NOP smem row stride of the output staging.
                 2 = DMMA with 2-D TMA tensor copies (M*S, N*S even and >= 16).
                 3 = TSMM only: C-stationary DMMA (p0 = NBW 8-column blocks per warp,
                     p1 = WR 8-row blocks per warp; TMA conditions as 2).
                 4 = TSMM only: C-stationary DMMA with bulk copies and shared
                     per-row-group output staging (any width; p0 = NBW, p1 = WR).
                 Flags (OR-ed in, DMMA TSMTTSM kernels 1/2 unless noted):
                   16  DFMA edge warps for the cells outside the 8-aligned core;
                       bits 6-7 = edge warps - 1 (1..4 warps splitting the rows).
                       TSMM kernels 3 and 4: the last N mod 8 columns of B by DFMA
                       in the warps of the last column group instead of a padded
                       8-column DMMA block (N >= 8, N not a multiple of 8);
                   32  paired 16-byte fragment loads (D, even p0/p1);
                   256 complex-as-real (Z; TSMTTSM 1/2, TSMM 3): the real kernel runs
                       on the interleaved (re, im) view -- A, B as real K x 2M, K x 2N --
                       and p0..p3, threads, rows refer to that 2M x 2N real problem;
                   512 3M / Gauss complex products (Z; TSMTTSM 1/2, not with 256):
                       T1 = Ar^T Br, T2 = Ai^T Bi, T3 = (Ar+Ai)^T (Br+Bi) on the
                       tensor pipe, C = (T1 - T2) + i (T3 - T1 - T2) -- 3 real
                       DMMAs per 8x8 block instead of 4 (same bytes, 3/4 of the
                       FP64 work; error within the |A|^T|B| tolerance, exact
                       on integer-valued inputs);
                   1024 plain consumer-warp order (DMMA kernels): by default the
                       warps of one C tile / column group are spread over the 4 SM
                       sub-partitions; this flag keeps warp w on tile w % tiles.
                       A launch argument, not a separate kernel;
                   2048 inline edge (DMMA TSMTTSM 1/2, not with 16): DMMA on the
                       8-aligned core, and the consumer warps themselves compute
                       the cells outside it with DFMA between their DMMAs (each
                       warp tile of a row slot owns some edge lane groups).
                 Invalid combinations return TSM_ERR_INVALID_VALUE. */
  int p3;
} tsm_config;

/* Create a plan with an explicit configuration (used by the on-B200
 * autotuner, tools/autotune.py).  If the configuration is not one of the
 * ahead-of-time instantiations, the kernel is compiled at run time by NVRTC
 * from the same template source.  Errors as tsm_plan_create, plus
 * TSM_ERR_INVALID_VALUE for an inconsistent configuration and
 * TSM_ERR_INTERNAL if run-time compilation fails. */
tsm_status tsm_plan_create_config(tsm_plan *out, tsm_op op, tsm_dtype dtype, int M, int N,
                                  int device, const tsm_config *cfg);

/* The configuration a plan resolved to (stages/ctas after clipping). */
tsm_status tsm_plan_get_config(tsm_plan p, tsm_config *cfg);

/* Plan flags.
 *   TSM_FLAG_CONJ  Z plans only.  TSMTTSM: C = A^H B (conjugate transpose of A,
 *                  what complex classical Gram-Schmidt against a basis A needs,
 *                  PAPER.md:108-112).  TSMM: B = A conj(C).  Same kernels: the
 *                  sign of Im(A) / Im(C) is flipped on load (exact). */
#define TSM_FLAG_CONJ 1u
/*   TSM_FLAG_STRIDED  (NEXT row N4) choose a kernel that takes strided row
 *                  views (tsmttsm_ld_* / tsmm_ld_*): a TMA kernel, whose tensor
 *                  maps carry the row stride, for shapes with 16-byte rows of
 *                  >= 128 bytes (D widths even and >= 16, Z widths >= 8) --
 *                  calls then need 16-byte row strides and bases; other shapes
 *                  get the gather-capable kernel of TSM_FLAG_GATHER. */
#define TSM_FLAG_STRIDED 2u
/*   TSM_FLAG_NO_GRID_REDUCE  MEASUREMENT ONLY (TSMTTSM): the reduction-     */
/*                  overhead baseline of PAPER.md:1000-1016 ("a kernel      */
/*                  without a global reduction"): every block computes and  */
/*                  writes its partial to the workspace, the grid reduction */
/*                  (T4) is skipped and C is NOT written.  Not for results. */
#define TSM_FLAG_NO_GRID_REDUCE 4u
/*   TSM_FLAG_GATHER  (NEXT row N4) a gather-capable kernel (TSMTTSM kernel 1,*/
/*                  TSMM kernel 4) for strided views of ANY row stride and,  */
/*                  for D, 8-byte aligned A / B bases (column subsets at odd  */
/*                  offsets): the producer warp copies row elements with     */
/*                  cp.async (8 / 16 bytes) completing on the stage mbarrier,*/
/*                  TSMM stores B rows element-wise.  Every shape has one.   */
/*                  TSM_FLAG_STRIDED picks a TMA kernel when the shape has   */
/*                  one (16-byte row strides and bases) and this otherwise.  */
#define TSM_FLAG_GATHER 8u

/* tsm_plan_create / tsm_plan_create_config with flags: cfg == NULL selects the
 * tuned default configuration.  TSM_ERR_INVALID_VALUE for unknown flags or
 * TSM_FLAG_CONJ on a D plan. */
tsm_status tsm_plan_create_ex(tsm_plan *out, tsm_op op, tsm_dtype dtype, int M, int N, int device,
                              const tsm_config *cfg, unsigned flags);
tsm_status tsm_plan_get_flags(tsm_plan p, unsigned *flags);

/* Build tooling: compile the kernel a plan would use (default configuration,
 * cfg, or the TSM_FLAG_STRIDED default) with NVRTC into the kernel cache
 * (<directory of libtsm.so>/kcache, or TSM_JIT_CACHE_DIR) without touching a
 * device.  Plans load cached kernels instead of compiling them.  Errors as
 * tsm_plan_create_config; TSM_ERR_INTERNAL if NVRTC fails. */
tsm_status tsm_jit_precompile(tsm_op op, tsm_dtype dtype, int M, int N, const tsm_config *cfg,
                              unsigned flags);

/* Bytes of device workspace a TSMTTSM call with K rows needs (partials of the
 * fixed-order grid reduction plus 2 counter words); 0 for TSMM plans.
 * The first 256 bytes hold counters that MUST be zero before the first use of
 * a workspace (cudaMemset / torch.zeros, or tsm_workspace_init); every
 * successful call leaves them zero again. */
tsm_status tsm_plan_workspace_bytes(tsm_plan p, int64_t K, size_t *bytes);

/* Zero the counter words of a workspace (enqueued on `stream`). */
tsm_status tsm_workspace_init(void *ws, size_t ws_bytes, tsm_stream stream);

/* Human/JSON-readable description of the chosen instantiation and launch
 * parameters for K rows, written into buf (NUL-terminated, truncated to len). */
tsm_status tsm_plan_describe(tsm_plan p, int64_t K, char *buf, size_t len);

tsm_status tsm_plan_destroy(tsm_plan p);

const char *tsm_status_string(tsm_status s);
const char *tsm_last_error_detail(void);

/* ------------------------------------------------------------------------ */
/* TSMTTSM  C = A^T B                         */
/*   A: K x M device, B: K x N device, C: M x N device (overwritten).        */
/*   ws: workspace of >= tsm_plan_workspace_bytes(p, K) bytes.               */
/*   Grid-reduction progress rule (T4): each block writes its partial, takes */
/*   a ticket, and the last `nfin` blocks to arrive wait (spin) until every  */
/*   block of the launch has arrived, then sum the partials in fixed block   */
/*   order.  The grid is at most SMs x CTAs/SM, so on an otherwise idle GPU  */
/*   every block is resident and the wait ends.  The call relies on the      */
/*   remaining blocks becoming resident eventually: a kernel running         */
/*   concurrently on another stream (or another MPS client) that holds SMs   */
/*   indefinitely -- e.g. a persistent kernel, or an NCCL kernel waiting for */
/*   a peer that itself waits on this call -- can stall it.  Concurrent      */
/*   kernels that finish on their own (any libtsm call, NCCL collectives     */
/*   whose peers progress independently) only delay it.  With nfin = 1     */
/*   (tsm_plan_describe) the single finisher is the block holding the last  */
/*   ticket: it never waits, so that case needs no co-residency at all.      */
/* ------------------------------------------------------------------------ */
tsm_status tsmttsm_d(tsm_plan p, int64_t K, const double *A, const double *B, double *C,
                     void *ws, size_t ws_bytes, tsm_stream stream);
tsm_status tsmttsm_z(tsm_plan p, int64_t K, const tsm_zcomplex *A, const tsm_zcomplex *B,
                     tsm_zcomplex *C, void *ws, size_t ws_bytes, tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* TSMM  B = A C                              */
/*   A: K x M device, C: M x N device, B: K x N device (overwritten).        */
/* ------------------------------------------------------------------------ */
tsm_status tsmm_d(tsm_plan p, int64_t K, const double *A, const double *C, double *B,
                  tsm_stream stream);
tsm_status tsmm_z(tsm_plan p, int64_t K, const tsm_zcomplex *A, const tsm_zcomplex *C,
                  tsm_zcomplex *B, tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* Strided row views (NEXT row N4; block vectors as column subsets of wider   */
/* arrays): row k of A starts at A + k*lda, of B at B + k*ldb (elements, lda  */
/* >= M, ldb >= N).  lda == M and ldb == N are the dense calls (any plan);    */
/* otherwise the plan needs a TSM_FLAG_STRIDED plan with a TMA kernel and     */
/* 16-byte row strides / bases, or a gather-capable plan (TSM_FLAG_GATHER,    */
/* or TSM_FLAG_STRIDED on a shape without a TMA kernel): any row stride, D    */
/* bases 8-byte aligned.  Other plans: TSM_ERR_UNSUPPORTED.  C stays dense.   */
/* ------------------------------------------------------------------------ */
tsm_status tsmttsm_ld_d(tsm_plan p, int64_t K, const double *A, int64_t lda, const double *B, int64_t ldb,
                        double *C, void *ws, size_t ws_bytes, tsm_stream stream);
tsm_status tsmttsm_ld_z(tsm_plan p, int64_t K, const tsm_zcomplex *A, int64_t lda,
                        const tsm_zcomplex *B, int64_t ldb, tsm_zcomplex *C, void *ws,
                        size_t ws_bytes, tsm_stream stream);
tsm_status tsmm_ld_d(tsm_plan p, int64_t K, const double *A, int64_t lda, const double *C, double *B,
                     int64_t ldb, tsm_stream stream);
tsm_status tsmm_ld_z(tsm_plan p, int64_t K, const tsm_zcomplex *A, int64_t lda, const tsm_zcomplex *C,
                     tsm_zcomplex *B, int64_t ldb, tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* TSMM update  B <- alpha * A C + beta * B   (SURVEY.md §8(f) NEXT row N1;  */
/* the TSMM step of classical Gram-Schmidt: B -= A C is    */
/* alpha = -1, beta = 1).  One pass over A and B:                            */
/*   beta = 0: B = alpha A C, written like tsmm_* (B is not read);            */
/*   beta = 1: the kernels add alpha A C into B with bulk / TMA reduce-add    */
/*             (cp.reduce.async.bulk .add.f64: B is read and written by the   */
/*             memory system, one rounding per element);                      */
/*   other beta: B is first scaled by beta (one extra pass over B), then as 1.*/
/* alpha multiplies C once per block (alpha = 1 leaves C bit-exact).  A plan */
/* with TSM_FLAG_CONJ uses conj(C).  Errors as tsmm_*.                        */
/* ------------------------------------------------------------------------ */
tsm_status tsmm_update_d(tsm_plan p, int64_t K, double alpha, const double *A, const double *C,
                         double beta, double *B, tsm_stream stream);
tsm_status tsmm_update_z(tsm_plan p, int64_t K, tsm_zcomplex alpha, const tsm_zcomplex *A,
                         const tsm_zcomplex *C, tsm_zcomplex beta, tsm_zcomplex *B,
                         tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* One block classical Gram-Schmidt projection (NEXT row N1) */
/* of the K x N block vector B against the K x M basis A:                    */
/*   C = A^T B        (p_tt: TSMTTSM plan (M, N); Z: create it with          */
/*                     TSM_FLAG_CONJ for A^H B),                              */
/*   B <- B - A C     (p_mm: TSMM plan (M, N), tsmm_update with alpha = -1,   */
/*                     beta = 1).                                             */
/* comm != NULL: K is this rank's K_local and C is summed over ranks (as      */
/* tsmttsm_allreduce_*) before the update; ws then needs the extra bytes of   */
/* tsm_comm_workspace_extra_bytes.  C (M x N, device) holds the coefficients  */
/* on return.                                                                 */
/* ------------------------------------------------------------------------ */
tsm_status tsm_cgs_step_d(tsm_plan p_tt, tsm_plan p_mm, tsm_comm comm, int64_t K, const double *A,
                          double *B, double *C, void *ws, size_t ws_bytes, tsm_stream stream);
tsm_status tsm_cgs_step_z(tsm_plan p_tt, tsm_plan p_mm, tsm_comm comm, int64_t K,
                          const tsm_zcomplex *A, tsm_zcomplex *B, tsm_zcomplex *C, void *ws,
                          size_t ws_bytes, tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* Device input generator (same counter-based generator as  */
/* the Python module tsminputs, implemented independently):                  */
/*   dst[i] = value(mix64(seed*0xD1B54A32D192ED03 + (mat_id<<48) + start+i))  */
/*   for i < n (n real values; a complex matrix of e elements is n = 2e).     */
/*   mode 0 = "fp" uniform [-1,1), mode 1 = "int" integers in [-1024,1023].   */
/* ------------------------------------------------------------------------ */
tsm_status tsm_fill(double *dst, int64_t n, uint64_t seed, int mat_id, int mode,
                    int64_t start, tsm_stream stream);

/* L2 flush helper for benchmarks: overwrite `bytes` of scratch device memory. */
tsm_status tsm_l2_flush(void *scratch, size_t bytes, tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* Roofline-denominator probes (measurement only, not part of the path).    */
/* "b_s is measured in the same run, following the paper's */
/* convention: read-only streaming for TSMTTSM, read +   */
/* write copy for TSMM"; "measure P_fp64 sustained; do not assume boost"    */
/* (PAPER.md:280-289 measures its peaks the same way).  One launch on       */
/* `stream`; the caller times it with events.  *work receives the launch's  */
/* work: bytes moved (READ: `bytes` read; COPY: bytes/2 read + bytes/2      */
/* written) or FP64 flops (DMMA: mma.sync.m8n8k4.f64 chains, `iters` loop   */
/* trips, 8 blocks x 4 warps per SM).  buf: caller-owned device memory,     */
/* 16-byte aligned; READ reads it, COPY overwrites its second half, DMMA    */
/* writes at most buf[0].  Errors: TSM_ERR_INVALID_VALUE (bad kind, buffer, */
/* iters), TSM_ERR_CUDA (launch).                                           */
/* ------------------------------------------------------------------------ */
#define TSM_PROBE_READ 0
#define TSM_PROBE_COPY 1
#define TSM_PROBE_DMMA 2
#define TSM_PROBE_CLOCK 3 /* one thread: SM cycles over `iters` ns of globaltimer -> MHz in buf[0] */
tsm_status tsm_probe(int kind, void *buf, size_t bytes, int64_t iters, tsm_stream stream, double *work);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: one process per GPU, K sharded by rows.      */
/* The 128-byte NCCL unique id is created on rank 0 with tsm_comm_unique_id  */
/* and exchanged by the caller (torch.distributed).  NCCL is loaded          */
/* dynamically (the libnccl.so.2 already in the process, e.g. torch's);      */
/* TSM_ERR_NCCL if unavailable.                                              */
/* ------------------------------------------------------------------------ */
#define TSM_COMM_DETERMINISTIC 1 /* allgather partials + fixed rank-order sum */

tsm_status tsm_comm_unique_id(void *uid128);
tsm_status tsm_comm_init(tsm_comm *out, const void *uid128, int nranks, int rank, int device,
                         int flags);
tsm_status tsm_comm_destroy(tsm_comm c);
/* Workspace for the sharded TSMTTSM: tsm_plan_workspace_bytes(p, K_local) plus
 * this many extra bytes (deterministic mode gathers nranks partial C's). */
tsm_status tsm_comm_workspace_extra_bytes(tsm_comm c, tsm_plan p, size_t *bytes);

/* Local TSMTTSM over this rank's K_local rows, then a sum of C over ranks
 * (ncclAllReduce, or allgather + fixed-order sum with TSM_COMM_DETERMINISTIC).
 * C ends replicated on every rank.  K_local may be 0 (contributes zeros). */
tsm_status tsmttsm_allreduce_d(tsm_plan p, tsm_comm c, int64_t K_local, const double *A,
                               const double *B, double *C, void *ws, size_t ws_bytes,
                               tsm_stream stream);
tsm_status tsmttsm_allreduce_z(tsm_plan p, tsm_comm c, int64_t K_local, const tsm_zcomplex *A,
                               const tsm_zcomplex *B, tsm_zcomplex *C, void *ws,
                               size_t ws_bytes, tsm_stream stream);

/* Broadcast C from `root` (in place; input on root, output elsewhere), then
 * the local TSMM B_local = A_local C.  K_local may be 0. */
tsm_status tsmm_bcast_d(tsm_plan p, tsm_comm c, int root, int64_t K_local, const double *A,
                        double *C, double *B, tsm_stream stream);
tsm_status tsmm_bcast_z(tsm_plan p, tsm_comm c, int root, int64_t K_local,
                        const tsm_zcomplex *A, tsm_zcomplex *C, tsm_zcomplex *B,
                        tsm_stream stream);

/* ------------------------------------------------------------------------ */
/* NEXT N3: TSMTTSM with the   */
/* grid reduction FUSED with the cross-GPU sum over peer memory -- no NCCL    */
/* call.  Each rank owns a symmetric "slot buffer" (device memory allocated   */
/* by tsm_peer_create, 256 B + 2 x 8 x 64*64*2 doubles = 1 MiB); the buffers  */
/* are mapped into every rank with CUDA IPC (NVLink / NVSwitch P2P).  The     */
/* finisher blocks of the TSMTTSM kernel store this rank's C cells into the   */
/* slot of every rank, signal with system-scope atomics, wait for all ranks   */
/* and sum the slots in rank order: C ends replicated on every rank and is    */
/* bitwise equal to the TSM_COMM_DETERMINISTIC (allgather + rank-order sum)   */
/* result.  Setup: tsm_peer_create on every rank, tsm_peer_export -> 64-byte  */
/* IPC handle, exchange all handles (e.g. torch.distributed all_gather), then */
/* tsm_peer_open with the nranks handles in rank order (the own handle is     */
/* ignored).  Ranks may share a device (separate processes).  Calls must be   */
/* issued in the same order on every rank, one stream per tsm_peer.  A rank   */
/* that never arrives makes the others give up after the timeout (default   */
/* 2 s, tsm_peer_set_timeout): C = NaN and tsm_peer_error reports 1 (after a  */
/* stream sync) -- no GPU hang.  Each slot carries the sequence number of the */
/* call that wrote it; a reader that finds another call's data (a rank that   */
/* timed out and ran ahead) also reports the error instead of summing it.     */
/* Once the error flag of a rank is set, every later fused call on it fails   */
/* fast (C = NaN, nothing stored to peers, no arrival signalled) until every  */
/* rank calls tsm_peer_reset.  The parity / arrival target / sequence number  */
/* are launch arguments: capturing a fused call in a CUDA graph and replaying */
/* it is NOT supported.  The kernel's finisher blocks spin on arrivals, so    */
/* every block of the launch must be able to become resident (true for the   */
/* persistent grids libtsm launches unless another kernel pins the SMs).      */
/* ------------------------------------------------------------------------ */
typedef struct tsm_peer_s *tsm_peer;
/* nranks in [1, 8], rank in [0, nranks); allocates and zeroes the slot buffer
 * on `device`.  TSM_ERR_CUDA on allocation failure. */
tsm_status tsm_peer_create(tsm_peer *out, int nranks, int rank, int device);
/* 64-byte cudaIpcMemHandle of this rank's slot buffer (host memory out). */
tsm_status tsm_peer_export(tsm_peer p, void *handle64);
/* handles: nranks x 64 bytes (host), rank order.  Opens every peer's buffer
 * (cudaIpcOpenMemHandle, lazy peer access).  TSM_ERR_CUDA if a handle cannot
 * be opened (e.g. no P2P path). */
tsm_status tsm_peer_open(tsm_peer p, const void *handles);
tsm_status tsm_peer_destroy(tsm_peer p);
/* 1 if a fused reduction on this tsm_peer timed out waiting for a rank or
 * found a slot written by another call (synchronous device read). */
tsm_status tsm_peer_error(tsm_peer p, int *err);
/* Bounded wait of later fused calls, in nanoseconds (> 0; default 2e9). */
tsm_status tsm_peer_set_timeout(tsm_peer p, uint64_t timeout_ns);
/* Collective recovery after an error: synchronizes `stream`, clears this
 * rank's counters, error flag and sequence numbers and restarts the call
 * count.  Every rank must call it (and the caller must barrier afterwards,
 * e.g. torch.distributed.barrier) before the next fused call. */
tsm_status tsm_peer_reset(tsm_peer p, tsm_stream stream);
/* C = sum over ranks of A_r^T B_r (plain transpose; A^H B with a conj plan),
 * replicated.  Arguments as tsmttsm_d / tsmttsm_z with K_local >= 0 (an
 * empty shard contributes zeros); the plan's workspace rules apply. */
tsm_status tsmttsm_peer_d(tsm_plan p, tsm_peer c, int64_t K_local, const double *A,
                          const double *B, double *C, void *ws, size_t ws_bytes,
                          tsm_stream stream);
tsm_status tsmttsm_peer_z(tsm_plan p, tsm_peer c, int64_t K_local, const tsm_zcomplex *A,
                          const tsm_zcomplex *B, tsm_zcomplex *C, void *ws, size_t ws_bytes,
                          tsm_stream stream);

/* Library / build information (JSON), e.g. the list of AOT instantiations. */
const char *tsm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* LIBTSM_H */
