// Dependent-chain latencies: SHFL (64-bit value as two 32-bit halves), DADD, LDS.128
#include <cstdio>
__global__ void k(int n, double* out, long long* cyc) {
  __shared__ double2 s[64];
  s[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  __syncwarp();
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1.0000001;
  long long t2 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { double2 v = s[idx]; idx = (int)v.y + (threadIdx.x & 31) - 1; }
  long long t3 = clock64();
  out[threadIdx.x] = x + idx;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; long long h[3];
  cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(1000, o, c);
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("SHFL(f64) %.1f  DADD %.1f  LDS.128 %.1f cycles per dependent op\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
}
