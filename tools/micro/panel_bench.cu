// Micro-benchmark: cycles per warp_panel op (operands in shared memory) for several shapes.
#include <cstdio>
#include "../../paper_1703_01175_b200/csrc/h2b_panel.cuh"
void h2b_set_error(const std::string&) {}
__global__ void k(int R, int w, int reps, long long* cycles, double* sink) {
  extern __shared__ double2 sm[];
  __shared__ double2 red[256];
  for (int i = threadIdx.x; i < 11000; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double2* dst = sm + 10000 + warp * 64;
  const double2* P = sm + warp * 16;
  const double2* in = sm + 8000 + warp * 8;
  auto inf = [in](int r) { return in[r]; };
  const long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    warp_panel<false>(P, R, w, inf, dst, red + warp * 32);
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cycles[0] = t1 - t0;
    sink[0] = dst[0].x;
  }
}
int main() {
  double* sink;
  long long* cyc_d;
  cudaMalloc(&sink, 64);
  cudaMalloc(&cyc_d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12000 * 16);
  int shapes[][2] = {{32, 5}, {32, 8}, {10, 5}, {5, 10}, {6, 32}, {64, 19}, {20, 64}};
  for (auto& s : shapes) {
    k<<<1, 256, 12000 * 16>>>(s[0], s[1], 100, cyc_d, sink);
    long long cyc = 0;
    cudaMemcpy(&cyc, cyc_d, 8, cudaMemcpyDeviceToHost);
    printf("R=%3d w=%3d : %6.0f cycles per op (incl. __syncthreads)\n", s[0], s[1], cyc / 100.0);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
