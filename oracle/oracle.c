/*
 * oracle.c — CPU ORACLE for libtsm.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  The product path
 * (paper_1905_03136_b200/, libtsm.so) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (the plain definitions; PAPER.md is the authority):
 *
 *   TSMTTSM  C = A^T B      PAPER.md:64-68 (§1.1, "A^T B = C"),
 *            C[m][n] = sum_{k<K} A[k][m] * B[k][n]
 *                            PAPER.md:342-349 (Listing 1, naive MMM)
 *   TSMM     B = A C        PAPER.md:64-68 ("A C = B")
 *            B[k][n] = sum_{m<M} A[k][m] * C[m][n]   (reduction over the short M axis)
 *
 *   A is K x M, B is K x N, C is M x N, all row-major and contiguous
 *   ("Row-major tall & skinny matrices"; C row-major m*N+n is
 *   DESIGN.md reading R2).  Z = complex double stored as interleaved (re, im)
 *   pairs; the transpose is the PLAIN (non-conjugating) one (PAPER.md:66 writes
 *   A^T throughout; reading R1).
 *
 * Summation order (reading R5 — the paper leaves the order open):
 *   TSMTTSM sums K terms per cell.  A plain serial sum has a worst-case error
 *   of gamma_K * sum|terms| (1.9e-9 at K=2^24), too close to the 1e-12 parity
 *   tolerance for comfort, so the oracle evaluates the same sum as
 *     1. serial fma chains over chunks of ORACLE_CHUNK = 1024 consecutive rows
 *        (k increasing),
 *     2. Neumaier-compensated accumulation of the chunk sums in chunk order
 *        inside a block of ORACLE_BLOCK = 2^16 rows,
 *     3. Neumaier-compensated accumulation of the block sums in block order.
 *   The structure is fixed by K alone, so results are bitwise independent of
 *   the OpenMP thread count.  Steps 1-2 (oracle_tsmttsm_{d,z}_blocks) and
 *   step 3 (oracle_tsmttsm_{d,z}_combine) are also exported on their own:
 *   the streaming mode of SURVEY.md §8(c) feeds the rows segment by segment
 *   (segments of whole 2^16-row blocks, regenerated from the input generator)
 *   and combines all blocks at the end -- the same operations in the same
 *   order as the one-shot call, so the same result bit for bit, with no host
 *   copy of a K = 2^28 matrix.  Complex cells use the 4 fmas
 *     re += ar*br; re -= ai*bi; im += ar*bi; im += ai*br
 *   in that order (8 real flops per complex multiply-add).
 *   TSMM sums only M <= 64 terms: a serial fma chain over m increasing.
 *
 * Each function also returns the error-bound matrix the parity tolerance is
 * stated against (BASELINE.json north_star):
 *   TSMTTSM  bound[m][n] = sum_k |A[k][m]| |B[k][n]|
 *   TSMM     bound[k][n] = sum_m |A[k][m]| |C[m][n]|
 *   with |.| the complex modulus for Z.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): SPEC.md:370-372 worked examples,
 * hand-worked 2x2 complex cases (tests/golden/), exact Fraction brute force,
 * exact integer arithmetic, Walsh/orthonormal closed forms, K-split additivity,
 * numpy matmul cross-check, thread-count determinism.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * (explicit fma() only; no FTZ/DAZ).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_CHUNK 1024
#define ORACLE_BLOCK 65536 /* 64 chunks */

/* Neumaier compensated accumulation of x into (*s, *c). */
static inline void neumaier_add(double *s, double *c, double x) {
  double t = *s + x;
  if (fabs(*s) >= fabs(x))
    *c += (*s - t) + x;
  else
    *c += (x - t) + *s;
  *s = t;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------------ */
/* TSMTTSM, real double.  C = A^T B (Listing 1).           */
/* C and bound are M*N row-major outputs; bound may be NULL.                 */
/* ------------------------------------------------------------------------ */
/* Steps 1-2 for every 2^16-row block of rows [0, K): per block and cell the
 * compensated sum of its chunk sums (S, Cc) and the bound term (Bd), written
 * to bs[b][3][MN] (zeroed by the caller). */
void oracle_tsmttsm_d_blocks(int64_t K, int M, int N, const double *A, const double *B,
                             double *bs) {
  const int64_t MN = (int64_t)M * N;
  const int64_t nblk = (K + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
#pragma omp parallel
  {
    double *acc = (double *)malloc(sizeof(double) * (size_t)MN);
    double *accb = (double *)malloc(sizeof(double) * (size_t)MN);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < nblk; b++) {
      double *S = bs + b * MN * 3, *Cc = S + MN, *Bd = Cc + MN;
      const int64_t k0 = b * ORACLE_BLOCK;
      const int64_t k1 = (k0 + ORACLE_BLOCK < K) ? k0 + ORACLE_BLOCK : K;
      for (int64_t c0 = k0; c0 < k1; c0 += ORACLE_CHUNK) {
        const int64_t c1 = (c0 + ORACLE_CHUNK < k1) ? c0 + ORACLE_CHUNK : k1;
        memset(acc, 0, sizeof(double) * (size_t)MN);
        memset(accb, 0, sizeof(double) * (size_t)MN);
        for (int64_t k = c0; k < c1; k++) {
          const double *a = A + k * M, *bb = B + k * N;
          for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
              acc[m * N + n] = fma(a[m], bb[n], acc[m * N + n]);
              accb[m * N + n] += fabs(a[m]) * fabs(bb[n]);
            }
        }
        for (int64_t i = 0; i < MN; i++) {
          neumaier_add(&S[i], &Cc[i], acc[i]);
          Bd[i] += accb[i];
        }
      }
    }
    free(acc);
    free(accb);
  }
}

/* Step 3: the block results combined in block order (compensated). */
void oracle_tsmttsm_d_combine(int64_t nblk, int M, int N, const double *bs, double *C, double *bound) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t i = 0; i < MN; i++) {
    double s = 0, c = 0, bd = 0;
    for (int64_t b = 0; b < nblk; b++) {
      const double *S = bs + b * MN * 3;
      neumaier_add(&s, &c, S[i]);
      c += S[MN + i];
      bd += S[2 * MN + i];
    }
    C[i] = s + c;
    if (bound) bound[i] = bd;
  }
}

void oracle_tsmttsm_d(int64_t K, int M, int N, const double *A, const double *B,
                      double *C, double *bound) {
  const int64_t MN = (int64_t)M * N;
  const int64_t nblk = (K + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
  /* per block: sum, compensation, bound */
  double *bs = (double *)calloc((size_t)(nblk * MN * 3 + 1), sizeof(double));
  oracle_tsmttsm_d_blocks(K, M, N, A, B, bs);
  oracle_tsmttsm_d_combine(nblk, M, N, bs, C, bound);
  free(bs);
}

/* ------------------------------------------------------------------------ */
/* TSMTTSM, complex double (interleaved re,im).  Plain transpose (R1); with  */
/* conj = 1 the conjugate transpose C = A^H B (NEXT row N2: the complex      */
/* Gram-Schmidt use of PAPER.md:108-112 needs A^H): conj(a) = ar - i ai is   */
/* substituted for a, i.e. ai -> -ai in the same 4 fmas.                     */
/* ------------------------------------------------------------------------ */
/* Steps 1-2 per block (complex): bs[b][5][MN] = re sum, re comp, im sum,
 * im comp, bound (zeroed by the caller). */
void oracle_tsmttsm_z_blocks(int64_t K, int M, int N, const double *A, const double *B,
                             double *bs, int conj) {
  const int64_t MN = (int64_t)M * N;
  const int64_t nblk = (K + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
#pragma omp parallel
  {
    double *acc = (double *)malloc(sizeof(double) * (size_t)MN * 2);
    double *accb = (double *)malloc(sizeof(double) * (size_t)MN);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < nblk; b++) {
      double *Sr = bs + b * MN * 5, *Cr = Sr + MN, *Si = Cr + MN, *Ci = Si + MN,
             *Bd = Ci + MN;
      const int64_t k0 = b * ORACLE_BLOCK;
      const int64_t k1 = (k0 + ORACLE_BLOCK < K) ? k0 + ORACLE_BLOCK : K;
      for (int64_t c0 = k0; c0 < k1; c0 += ORACLE_CHUNK) {
        const int64_t c1 = (c0 + ORACLE_CHUNK < k1) ? c0 + ORACLE_CHUNK : k1;
        memset(acc, 0, sizeof(double) * (size_t)MN * 2);
        memset(accb, 0, sizeof(double) * (size_t)MN);
        for (int64_t k = c0; k < c1; k++) {
          const double *a = A + 2 * k * M, *bb = B + 2 * k * N;
          for (int m = 0; m < M; m++) {
            const double ar = a[2 * m], ai = conj ? -a[2 * m + 1] : a[2 * m + 1];
            const double am = hypot(ar, ai);
            for (int n = 0; n < N; n++) {
              const double br = bb[2 * n], bi = bb[2 * n + 1];
              double re = acc[2 * (m * N + n)], im = acc[2 * (m * N + n) + 1];
              re = fma(ar, br, re);
              re = fma(-ai, bi, re);
              im = fma(ar, bi, im);
              im = fma(ai, br, im);
              acc[2 * (m * N + n)] = re;
              acc[2 * (m * N + n) + 1] = im;
              accb[m * N + n] += am * hypot(br, bi);
            }
          }
        }
        for (int64_t i = 0; i < MN; i++) {
          neumaier_add(&Sr[i], &Cr[i], acc[2 * i]);
          neumaier_add(&Si[i], &Ci[i], acc[2 * i + 1]);
          Bd[i] += accb[i];
        }
      }
    }
    free(acc);
    free(accb);
  }
}

/* Step 3 (complex): block results in block order. */
void oracle_tsmttsm_z_combine(int64_t nblk, int M, int N, const double *bs, double *C, double *bound) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t i = 0; i < MN; i++) {
    double sr = 0, cr = 0, si = 0, ci = 0, bd = 0;
    for (int64_t b = 0; b < nblk; b++) {
      const double *S = bs + b * MN * 5;
      neumaier_add(&sr, &cr, S[i]);
      cr += S[MN + i];
      neumaier_add(&si, &ci, S[2 * MN + i]);
      ci += S[3 * MN + i];
      bd += S[4 * MN + i];
    }
    C[2 * i] = sr + cr;
    C[2 * i + 1] = si + ci;
    if (bound) bound[i] = bd;
  }
}

static void tsmttsm_z_impl(int64_t K, int M, int N, const double *A, const double *B,
                           double *C, double *bound, int conj) {
  const int64_t MN = (int64_t)M * N;
  const int64_t nblk = (K + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
  /* per block: re sum, re comp, im sum, im comp, bound */
  double *bs = (double *)calloc((size_t)(nblk * MN * 5 + 1), sizeof(double));
  oracle_tsmttsm_z_blocks(K, M, N, A, B, bs, conj);
  oracle_tsmttsm_z_combine(nblk, M, N, bs, C, bound);
  free(bs);
}


void oracle_tsmttsm_z(int64_t K, int M, int N, const double *A, const double *B,
                      double *C, double *bound) {
  tsmttsm_z_impl(K, M, N, A, B, C, bound, 0);
}

/* C = A^H B */
void oracle_tsmttsm_zc(int64_t K, int M, int N, const double *A, const double *B,
                       double *C, double *bound) {
  tsmttsm_z_impl(K, M, N, A, B, C, bound, 1);
}

/* ------------------------------------------------------------------------ */
/* TSMM, real double.  B = A C (reduction over M,            */
/* PAPER.md:372-375).  B and bound are K*N row-major; bound may be NULL.     */
/* ------------------------------------------------------------------------ */
void oracle_tsmm_d(int64_t K, int M, int N, const double *A, const double *C,
                   double *B, double *bound) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; k++) {
    const double *a = A + k * M;
    for (int n = 0; n < N; n++) {
      double s = 0, bd = 0;
      for (int m = 0; m < M; m++) {
        s = fma(a[m], C[m * N + n], s);
        bd += fabs(a[m]) * fabs(C[m * N + n]);
      }
      B[k * N + n] = s;
      if (bound) bound[k * N + n] = bd;
    }
  }
}

/* TSMM, complex double (interleaved).  C used as given (no conjugation). */
void oracle_tsmm_z(int64_t K, int M, int N, const double *A, const double *C,
                   double *B, double *bound) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; k++) {
    const double *a = A + 2 * k * M;
    for (int n = 0; n < N; n++) {
      double re = 0, im = 0, bd = 0;
      for (int m = 0; m < M; m++) {
        const double ar = a[2 * m], ai = a[2 * m + 1];
        const double cr = C[2 * (m * N + n)], ci = C[2 * (m * N + n) + 1];
        re = fma(ar, cr, re);
        re = fma(-ai, ci, re);
        im = fma(ar, ci, im);
        im = fma(ai, cr, im);
        bd += hypot(ar, ai) * hypot(cr, ci);
      }
      B[2 * (k * N + n)] = re;
      B[2 * (k * N + n) + 1] = im;
      if (bound) bound[k * N + n] = bd;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* TSMM update (NEXT row N1): B <- alpha * (A C) + beta * B.  PAPER.md:108-112: */
/* "both the TSMTTSM (A^T B) and TSMM (A C) occur in classical Gram-Schmidt   */
/* orthogonalization of a number of vectors represented by B against an       */
/* orthogonal basis A" -- the projection step is B <- B - A (A^T B), i.e.      */
/* alpha = -1, beta = 1.  Per (k, n): s = serial fma chain over m (as in       */
/* oracle_tsmm_*), then out = fma(alpha, s, beta * b_old) (D), and the complex */
/* products alpha*s + beta*b written out the same way (Z).  conj_c = 1 uses   */
/* conj(C) (N2).  bound = |alpha| sum_m |a||c| + |beta| |b_old|.               */
/* ------------------------------------------------------------------------ */
void oracle_tsmm_update_d(int64_t K, int M, int N, double alpha, const double *A,
                          const double *C, double beta, double *B, double *bound) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; k++) {
    const double *a = A + k * M;
    for (int n = 0; n < N; n++) {
      double s = 0, bd = 0;
      for (int m = 0; m < M; m++) {
        s = fma(a[m], C[m * N + n], s);
        bd += fabs(a[m]) * fabs(C[m * N + n]);
      }
      const double b = B[k * N + n];
      B[k * N + n] = fma(alpha, s, beta * b);
      if (bound) bound[k * N + n] = fabs(alpha) * bd + fabs(beta) * fabs(b);
    }
  }
}

void oracle_tsmm_update_z(int64_t K, int M, int N, double alpha_re, double alpha_im,
                          const double *A, const double *C, double beta_re, double beta_im,
                          double *B, double *bound, int conj_c) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; k++) {
    const double *a = A + 2 * k * M;
    for (int n = 0; n < N; n++) {
      double re = 0, im = 0, bd = 0;
      for (int m = 0; m < M; m++) {
        const double ar = a[2 * m], ai = a[2 * m + 1];
        const double cr = C[2 * (m * N + n)];
        const double ci = conj_c ? -C[2 * (m * N + n) + 1] : C[2 * (m * N + n) + 1];
        re = fma(ar, cr, re);
        re = fma(-ai, ci, re);
        im = fma(ar, ci, im);
        im = fma(ai, cr, im);
        bd += hypot(ar, ai) * hypot(cr, ci);
      }
      double *b = B + 2 * (k * N + n);
      const double br = b[0], bi = b[1];
      /* alpha * s + beta * b, each complex product as two fma chains */
      double orr = beta_re * br;
      orr = fma(-beta_im, bi, orr);
      orr = fma(alpha_re, re, orr);
      orr = fma(-alpha_im, im, orr);
      double oi = beta_re * bi;
      oi = fma(beta_im, br, oi);
      oi = fma(alpha_re, im, oi);
      oi = fma(alpha_im, re, oi);
      b[0] = orr;
      b[1] = oi;
      if (bound) bound[k * N + n] = hypot(alpha_re, alpha_im) * bd + hypot(beta_re, beta_im) * hypot(br, bi);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Parity comparison (north star tolerance): max |got-ref| / bound.          */
/* Z: complex modulus of the difference.  n = element count (complex count   */
/* for Z).  Returns max ratio, writes the worst index and max abs error.     */
/* bound==0 cells require got==ref exactly (ratio +inf otherwise).           */
/* ------------------------------------------------------------------------ */
double oracle_max_err_ratio(int64_t n, int is_complex, const double *got,
                            const double *ref, const double *bound,
                            int64_t *worst, double *max_abs) {
  double worst_r = 0, worst_a = 0;
  int64_t wi = 0;
  for (int64_t i = 0; i < n; i++) {
    double d;
    if (is_complex)
      d = hypot(got[2 * i] - ref[2 * i], got[2 * i + 1] - ref[2 * i + 1]);
    else
      d = fabs(got[i] - ref[i]);
    if (d != d) { /* NaN */
      if (worst) *worst = i;
      if (max_abs) *max_abs = d;
      return d;
    }
    double r = (d == 0) ? 0.0 : (bound[i] > 0 ? d / bound[i] : INFINITY);
    if (d > worst_a) worst_a = d;
    if (r > worst_r) {
      worst_r = r;
      wi = i;
    }
  }
  if (worst) *worst = wi;
  if (max_abs) *max_abs = worst_a;
  return worst_r;
}
