// Compare warp panel GEMV formulations (operands in shared memory), cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
// v2: power-of-two column groups, two accumulators, shuffle reduction
__device__ __forceinline__ void panel_v2(const double2* P, int R, int w, const double2* in, double2* out) {
  const int lane = threadIdx.x & 31;
  int wp = 1;
  while (wp < w) wp <<= 1;
  const int G = 32 / wp;  // wp <= 32 assumed
  const int g = lane / wp, c = lane & (wp - 1);
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  if (c < w) {
    int r = g;
    for (; r + G < R; r += 2 * G) {
      cfma(a0, P[r * w + c], in[r]);
      cfma(a1, P[(r + G) * w + c], in[r + G]);
    }
    if (r < R) cfma(a0, P[r * w + c], in[r]);
  }
  a0.x += a1.x; a0.y += a1.y;
  for (int m = wp; m < 32; m <<= 1) {
    a0.x += __shfl_xor_sync(0xffffffffu, a0.x, m);
    a0.y += __shfl_xor_sync(0xffffffffu, a0.y, m);
  }
  if (lane < w) out[lane] = a0;
}
template <int MODE>
__global__ void k(int R, int w, int reps, long long* cycles, double* sink) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 11000; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double2* dst = sm + 10000 + warp * 64;
  const double2* P = sm + warp * 16;
  const double2* in = sm + 8000 + warp * 8;
  const long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    panel_v2(P, R, w, in, dst);
    if (MODE == 1) panel_v2(P + 3000, R, w, in + 100, dst + 32);  // 2 ops per warp
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[0] = t1 - t0; sink[0] = dst[0].x; }
}
int main() {
  double* sink; long long* cyc_d; cudaMalloc(&sink, 64); cudaMalloc(&cyc_d, 64);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  int shapes[][2] = {{32, 5}, {32, 8}, {5, 10}, {10, 5}, {64, 19}, {6, 32}};
  for (auto& s : shapes) for (int m = 0; m < 2; ++m) {
    if (m == 0) k<0><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    else k<1><<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    long long cyc = 0; cudaMemcpy(&cyc, cyc_d, 8, cudaMemcpyDeviceToHost);
    printf("v2 R=%3d w=%3d ops/warp=%d: %6.0f cycles per level\n", s[0], s[1], m + 1, cyc / 100.0);
  }
}
