// Fixed-shape panel GEMV (compile-time R, w) to bound the achievable per-op latency.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
template <int R, int W>
__device__ __forceinline__ void panel_fixed(const double2* P, const double2* in, double2* out) {
  constexpr int WP = W <= 1 ? 1 : W <= 2 ? 2 : W <= 4 ? 4 : W <= 8 ? 8 : W <= 16 ? 16 : 32;
  constexpr int G = 32 / WP;
  const int lane = threadIdx.x & 31;
  const int g = lane / WP, c = lane % WP;
  double2 a = make_double2(0, 0);
  if (c < W) {
#pragma unroll
    for (int r = 0; r < (R + G - 1) / G; ++r) {
      const int rr = g + r * G;
      if (rr < R) cfma(a, P[rr * W + c], in[rr]);
    }
  }
#pragma unroll
  for (int m = WP; m < 32; m <<= 1) {
    a.x += __shfl_xor_sync(0xffffffffu, a.x, m);
    a.y += __shfl_xor_sync(0xffffffffu, a.y, m);
  }
  if (lane < W) out[lane] = a;
}
template <int R, int W, int MODE>
__global__ void k(int reps, long long* cycles, double* sink) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 11000; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double2* dst = sm + 10000 + warp * 64;
  const double2* P = sm + warp * 16;
  const double2* in = sm + 8000 + warp * 8;
  const long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    panel_fixed<R, W>(P, in, dst);
    if (MODE == 0) __syncthreads();
    else __syncwarp();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[0] = t1 - t0; sink[0] = dst[0].x; }
}
template <int R, int W>
void run(double* sink, long long* cyc_d) {
  cudaFuncSetAttribute(k<R, W, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  cudaFuncSetAttribute(k<R, W, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  long long cyc = 0;
  k<R, W, 0><<<1, 256, 12000 * 16>>>(100, cyc_d, sink);
  cudaMemcpy(&cyc, cyc_d, 8, cudaMemcpyDeviceToHost);
  printf("fixed R=%3d w=%3d : %6.0f cycles/op with __syncthreads, ", R, W, cyc / 100.0);
  k<R, W, 1><<<1, 256, 12000 * 16>>>(100, cyc_d, sink);
  cudaMemcpy(&cyc, cyc_d, 8, cudaMemcpyDeviceToHost);
  printf("%6.0f with __syncwarp only\n", cyc / 100.0);
}
int main() {
  double* sink; long long* cyc_d; cudaMalloc(&sink, 64); cudaMalloc(&cyc_d, 64);
  run<32, 5>(sink, cyc_d);
  run<10, 5>(sink, cyc_d);
  run<6, 32>(sink, cyc_d);
  run<1, 32>(sink, cyc_d);
}
