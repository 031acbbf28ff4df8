// DFMA latency (dependent chain, 1 warp) and throughput (many warps) on this GPU, plus
// __syncthreads and an empty-loop baseline.
#include <cstdio>
__global__ void lat(double a, double b, int n, double* out, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
    x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr(double a, double b, int n, double* out, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void syncs(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long c;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 64);
  const int n = 1000;
  lat<<<1, 32>>>(1.0000001, 1e-9, n, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", c / (8.0 * n));
  for (int warps : {1, 4, 8, 16, 32}) {
    thr<<<1, 32 * warps>>>(1.0000001, 1e-9, n, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %2d warps on 1 SM: %.2f DFMA/clk/SM\n", warps, 32.0 * warps * 8 * n / c);
  }
  thr<<<148 * 2, 512>>>(1.0000001, 1e-9, n, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA throughput full chip, block 0: %.2f DFMA/clk/SM\n", 32.0 * 16 * 2 * 8 * n / c);
  for (int t : {32, 256, 1024}) {
    syncs<<<1, t>>>(n, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads (%4d threads): %.1f cycles\n", t, c / (double)n);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
