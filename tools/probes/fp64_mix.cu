// Probe: do DFMA (FP64 pipe) and DMMA (tensor pipe, m8n8k4 f64) run
// concurrently on one SM sub-partition?  Warps of a block run either a DFMA
// loop or a DMMA loop (or both interleaved in one instruction stream); if the
// two pipes were independent, the mixed rate would exceed the ~37 TFLOP/s
// each reaches alone (profiles/r01_probe.txt).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd DFMA;
// 3: every warp interleaves 1 DMMA with `ratio` DFMA instructions
__global__ void mix_k(double* out, long iters, int mode, int dfma_per_iter) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0) || mode == 3;
  const bool do_fma = mode == 1 || (mode == 2 && (warp & 1)) || mode == 3;
  double acc[8][2];
  double f[16];
#pragma unroll
  for (int j = 0; j < 8; j++) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int j = 0; j < 16; j++) f[j] = 1.0 + j + threadIdx.x;
  const double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  for (long it = 0; it < iters; it++) {
    if (do_mma) {
#pragma unroll
      for (int j = 0; j < 8; j++) dmma(acc[j][0], acc[j][1], a, b);
    }
    if (do_fma) {
      // 8 DMMAs = 8 x 256 FMA per warp = 64 DFMA warp-instructions of equal work
      for (int r = 0; r < dfma_per_iter; r += 16) {
#pragma unroll
        for (int j = 0; j < 16; j++) f[j] = fma(f[j], 0.999999, 1e-9);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += acc[j][0] + acc[j][1];
#pragma unroll
  for (int j = 0; j < 16; j++) s += f[j];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int S = 0;
  CK(cudaDeviceGetAttribute(&S, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const long iters = 20000;
  const int threads = 256, bps = 4;
  for (int mode = 0; mode < 4; mode++) {
    for (int dpi : {16, 32, 64}) {
      if (mode == 0 && dpi != 64) continue;
      mix_k<<<S * bps, threads>>>(out, 10, mode, dpi);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      mix_k<<<S * bps, threads>>>(out, iters, mode, dpi);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double warps = (double)S * bps * threads / 32;
      const double mma_w = mode == 0 || mode == 3 ? warps : mode == 2 ? warps / 2 : 0;
      const double fma_w = mode == 1 || mode == 3 ? warps : mode == 2 ? warps / 2 : 0;
      const double fl_mma = mma_w * iters * 8 * 256 * 2.0;
      const double fl_fma = fma_w * iters * dpi * 32 * 2.0;
      printf("mode %d dfma/iter %2d: %.3f ms  dmma %.2f + dfma %.2f = %.2f TFLOP/s\n", mode, dpi, ms,
             fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
    }
  }
  return 0;
}
