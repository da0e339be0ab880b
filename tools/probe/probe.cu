// B200 roofline-denominator probe (PAPER.md:248-289 analogue):
// read-only and read+write HBM bandwidth, FP64 DFMA and DMMA.8x8x4 throughput.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void read_sum(const double2* __restrict__ p, size_t n2, double* out) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n2; i += 4 * st) {
    double2 a = __ldg(p + i), b = __ldg(p + i + st), c = __ldg(p + i + 2 * st), d = __ldg(p + i + 3 * st);
    s0 += a.x + a.y; s1 += b.x + b.y; s2 += c.x + c.y; s3 += d.x + d.y;
  }
  for (; i < n2; i += st) { double2 a = p[i]; s0 += a.x + a.y; }
  double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) out[0] = s;
}
__global__ void copy_k(const double2* __restrict__ p, double2* __restrict__ q, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + st < n2; i += 2 * st) { double2 a = p[i], b = p[i + st]; q[i] = a; q[i + st] = b; }
  for (; i < n2; i += st) q[i] = p[i];
}
__global__ void dfma_k(double* out, long iters, double x) {
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; j++) a[j] = x + j + threadIdx.x;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 16; j++) a[j] = fma(a[j], 0.999999, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; j++) s += a[j];
  if (s == 1.2345) out[0] = s;
}
__global__ void dmma_k(double* out, long iters) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; j++) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += acc[j][0] + acc[j][1];
  if (s == 1.2345) out[0] = s;
}
template <class F> float time_ms(F f, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a)); for (int r = 0; r < reps; r++) f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms / reps;
}
int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2\":%d,\"smem_optin\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d}\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize, pr.sharedMemPerBlockOptin, pr.regsPerMultiprocessor, clk);
  int S = pr.multiProcessorCount;
  size_t bytes = 4ull << 30; size_t n2 = bytes / 16;
  double2 *p, *q; double* out; CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&q, bytes)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(p, 0, bytes)); CK(cudaMemset(q, 0, bytes));
  for (int bps : {2, 4, 8, 16}) {
    float ms = time_ms([&] { read_sum<<<S * bps, 256>>>(p, n2, out); }, 10);
    printf("read_only blocks/SM=%d: %.1f GB/s\n", bps, bytes / ms / 1e6);
  }
  for (int bps : {4, 8, 16}) {
    float ms = time_ms([&] { copy_k<<<S * bps, 256>>>(p, q, n2 / 2); }, 10);
    printf("copy (r+w) blocks/SM=%d: %.1f GB/s\n", bps, bytes / ms / 1e6);
  }
  for (long iters : {2000L, 200000L}) {
    for (int bps : {4, 8}) {
      float ms = time_ms([&] { dfma_k<<<S * bps, 256>>>(out, iters, 1.0); }, 3);
      double fl = 2.0 * 16 * iters * 256.0 * S * bps;
      printf("dfma iters=%ld blocks/SM=%d: %.3f ms %.2f TFLOP/s\n", iters, bps, ms, fl / ms / 1e9);
    }
  }
  for (long iters : {2000L, 100000L}) {
    for (int bps : {4, 8}) {
      float ms = time_ms([&] { dmma_k<<<S * bps, 256>>>(out, iters); }, 3);
      double fl = 2.0 * 256 * 8 * iters * 8.0 * S * bps;  // 8 warps/block
      printf("dmma iters=%ld blocks/SM=%d: %.3f ms %.2f TFLOP/s\n", iters, bps, ms, fl / ms / 1e9);
    }
  }
  return 0;
}
