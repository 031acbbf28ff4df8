// Launch / fence overheads of a persistent 296-CTA kernel with ~108 KB dynamic smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k_empty(unsigned* ctr, int iters, int fence) {
  extern __shared__ double sm[];
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 32) {
      if (fence) __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ctr + 1 + blockIdx.x), "r"(i) : "memory");
    }
  }
  if (threadIdx.x == 0) atomicAdd(ctr, 1u);
  if (threadIdx.x == 0 && iters < 0) sm[0] = 1;
}
int main() {
  unsigned* ctr; cudaMalloc(&ctr, 4096 * 4);
  char* flush; cudaMalloc(&flush, 256 << 20);
  const int smem = 108 * 1024;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int coop = 0; coop < 2; ++coop)
    for (int iters : {0, 8, 32})
      for (int fence : {0, 1}) {
        float tot = 0;
        for (int r = 0; r < 22; ++r) {
          cudaMemsetAsync(flush, r, 256 << 20);
          cudaEventRecord(a);
          if (coop) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(296); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_empty, ctr, iters, fence);
          } else {
            k_empty<<<296, 256, smem>>>(ctr, iters, fence);
          }
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) tot += ms;
        }
        printf("coop=%d iters=%2d fence=%d : %6.2f us\n", coop, iters, fence, tot / 20 * 1e3);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
