/*
 * gen.c -- fast host copy of the tsminputs counter-based generator.
 *
 * Holds NONE of the method's arithmetic: it only produces input values, the
 * same values tsminputs/__init__.py computes with numpy (tests check the two
 * agree element for element).  Used for full-size (K = 2^24 .. 2^28) parity
 * checks, where whole columns of A and B must be regenerated on the host
 * (SURVEY.md §8(c) streaming mode: "rows regenerated from the §8(d)
 * generator on the fly").
 *
 *   mix64(z): z += 0x9E3779B97F4A7C15
 *             z  = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
 *             z  = (z ^ (z >> 27)) * 0x94D049BB133111EB
 *             z ^= z >> 31
 *   h = mix64(key + i),  key = seed * 0xD1B54A32D192ED03 + (id << 48)
 *   fp : ((int64)(h >> 11) - 2^52) * 2^-52      int: (int64)(h >> 53) - 1024
 */
#include <stdint.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double value(uint64_t key, uint64_t i, int mode) {
  uint64_t h = mix64(key + i);
  if (mode == 0) return (double)((int64_t)(h >> 11) - ((int64_t)1 << 52)) * 0x1p-52;
  return (double)((int64_t)(h >> 53) - 1024);
}

/* out[j] = value(start + j * stride) for j < n (real streams). */
void tsmgen_strided(double *out, int64_t n, uint64_t start, uint64_t stride, uint64_t key, int mode) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; j++) out[j] = value(key, start + (uint64_t)j * stride, mode);
}

/* Rows [row0, row0 + K) x columns cols[0..ncol) of a matrix of `width`
 * columns, written row-major into out (K x ncol; complex: interleaved re, im,
 * element e -> indices 2e, 2e+1). */
void tsmgen_columns(double *out, int64_t row0, int64_t K, int64_t width, const int64_t *cols, int ncol,
                    uint64_t key, int mode, int cplx) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; k++) {
    for (int c = 0; c < ncol; c++) {
      uint64_t e = (uint64_t)(row0 + k) * (uint64_t)width + (uint64_t)cols[c];
      if (cplx) {
        out[2 * (k * ncol + c)] = value(key, 2 * e, mode);
        out[2 * (k * ncol + c) + 1] = value(key, 2 * e + 1, mode);
      } else {
        out[k * ncol + c] = value(key, e, mode);
      }
    }
  }
}
