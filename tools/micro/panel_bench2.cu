// Break down the cost of one small panel GEMV op in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
template <int MODE>
__global__ void k(int R, int w, int reps, long long* cycles, double* sink) {
  extern __shared__ double2 sm[];
  __shared__ double2 red[256];
  for (int i = threadIdx.x; i < 11000; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* dst = sm + 10000 + warp * 64;
  const double2* P = sm + warp * 16;
  const double2* in = sm + 8000 + warp * 8;
  const long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    const int G = 32 / w;
    const int g = lane / w, c = lane - g * w;
    double2 a = make_double2(0.0, 0.0);
    if (MODE != 2 && g < G)
      for (int r = g; r < R; r += G) cfma(a, P[r * w + c], in[r]);
    if (MODE == 1) { dst[lane] = a; }
    if (MODE != 1) {
      red[threadIdx.x] = a;
      __syncwarp();
      if (lane < w) {
        double2 s = red[warp * 32 + lane];
        for (int gg = 1; gg < G; ++gg) { double2 v = red[warp * 32 + gg * w + lane]; s.x += v.x; s.y += v.y; }
        dst[lane] = s;
      }
      __syncwarp();
    }
    if (MODE != 3) __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[0] = t1 - t0; sink[0] = dst[0].x; }
}
int main() {
  double* sink; long long* cyc_d; cudaMalloc(&sink, 64); cudaMalloc(&cyc_d, 64);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  int shapes[][2] = {{32, 5}, {5, 10}, {64, 19}};
  const char* nm[4] = {"full", "loop only", "reduce only", "full, no bar"};
  for (auto& s : shapes) for (int m = 0; m < 4; ++m) {
    if (m == 0) k<0><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    if (m == 1) k<1><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    if (m == 2) k<2><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    if (m == 3) k<3><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    long long cyc = 0; cudaMemcpy(&cyc, cyc_d, 8, cudaMemcpyDeviceToHost);
    printf("R=%3d w=%3d %-12s: %6.0f cycles per op\n", s[0], s[1], nm[m], cyc / 100.0);
  }
}
