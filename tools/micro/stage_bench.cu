// Micro-benchmark: global->shared staging of B bytes per CTA, three ways:
//  (0) one cp.async.bulk of B bytes   (1) cp.async.bulk in 16 KB chunks by 16 threads
//  (2) cooperative 16-B LDG + STS, 8 loads in flight per thread.
// Also measures mbarrier wait variants.  Development aid for the span kernels.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(bar)) : "memory");
}
template <int MODE, int WAIT>
__global__ void k(const double2* __restrict__ src, int elems, double* sink) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ uint64_t bar;
  const double2* s = src + (size_t)blockIdx.x * elems;
  if (MODE < 2) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(elems * 16) : "memory");
    }
    __syncthreads();
    if (MODE == 0) {
      if (threadIdx.x == 0) bulk(sm, s, elems * 16, &bar);
    } else {
      const int chunk = 1024;  // 16 KB
      for (int c = threadIdx.x; c * chunk < elems; c += blockDim.x) {
        int n = min(chunk, elems - c * chunk);
        bulk(sm + c * chunk, s + c * chunk, n * 16, &bar);
      }
    }
    if (WAIT == 0) {
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, 10000000;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su(&bar)) : "memory");
    } else {
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su(&bar)) : "memory");
    }
  } else {
    for (int i0 = threadIdx.x; i0 < elems; i0 += blockDim.x * 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) if (i0 + u * blockDim.x < elems) v[u] = __ldg(s + i0 + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 8; ++u) if (i0 + u * blockDim.x < elems) sm[i0 + u * blockDim.x] = v[u];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = sm[elems / 2].x;
}
int main() {
  const int maxe = 12800;
  double2* src; double* sink; char* flush;
  cudaMalloc(&src, (size_t)148 * maxe * 16); cudaMemset(src, 1, (size_t)148 * maxe * 16);
  cudaMalloc(&sink, 148 * 8); cudaMalloc(&flush, 512 << 20);
  cudaFuncSetAttribute(k<0,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxe * 16);
  cudaFuncSetAttribute(k<0,1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxe * 16);
  cudaFuncSetAttribute(k<1,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxe * 16);
  cudaFuncSetAttribute(k<2,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxe * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[4] = {"bulk1 suspend", "bulk1 spin", "bulk16KB", "ldg"};
  for (int grid : {1, 64, 148}) for (int e : {1024, 6400, 12800}) for (int m = 0; m < 4; ++m) {
    float tot = 0; int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      cudaMemsetAsync(flush, r, 512 << 20);
      cudaEventRecord(a);
      if (m == 0) k<0,0><<<grid, 256, e * 16>>>(src, e, sink);
      if (m == 1) k<0,1><<<grid, 256, e * 16>>>(src, e, sink);
      if (m == 2) k<1,0><<<grid, 256, e * 16>>>(src, e, sink);
      if (m == 3) k<2,0><<<grid, 256, e * 16>>>(src, e, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) tot += ms;
    }
    float us = tot / reps * 1e3;
    printf("grid %3d  %6d B/CTA  %-14s %8.2f us  %8.1f GB/s per CTA\n", grid, e * 16, names[m], us, e * 16 / us / 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
