// Probe: does the TMA tensor reduce-add (cp.reduce.async.bulk.tensor .add) work on
// an FP64 tensor map on this GPU, and does the non-tensor bulk reduce (.add.f64)?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/probes/tma_reduce_f64.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void red_tensor(const __grid_constant__ CUtensorMap tm) {
  __shared__ alignas(1024) double s[16 * 8];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) s[i] = 1.0 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                 :: "l"(&tm), "r"(0), "r"(0), "r"(sa) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void red_bulk(double* g) {
  __shared__ alignas(128) double s[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) s[i] = 1.0 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                 :: "l"(g), "r"(sa), "r"(1024) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 1024 * 8);
  std::vector<double> h(1024, 0.5), o(1024);
  cudaMemcpy(d, h.data(), 1024 * 8, cudaMemcpyHostToDevice);
  red_bulk<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(o.data(), d, 1024 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128; i++) bad += o[i] != 0.5 + 1.0 + i;
  printf("bulk reduce add.f64: %s, %d bad\n", cudaGetErrorString(e), bad);

  cudaMemcpy(d, h.data(), 1024 * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {32, 32};        // 32 x 32 doubles, row-major
  cuuint64_t strides[1] = {32 * 8};
  cuuint32_t box[2] = {16, 8};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  red_tensor<<<1, 128>>>(tm);
  e = cudaDeviceSynchronize();
  cudaMemcpy(o.data(), d, 1024 * 8, cudaMemcpyDeviceToHost);
  double sum = 0;
  for (int i = 0; i < 1024; i++) sum += o[i];
  // 128 values 1..128 added (swizzled placement) on top of 0.5 everywhere
  printf("tensor reduce add (f64 map): %s, sum %.1f (expect %.1f)\n", cudaGetErrorString(e), sum,
         1024 * 0.5 + 128 * 129 / 2.0);
  return 0;
}
