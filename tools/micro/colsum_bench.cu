// Latency of one tree level in shared memory on B200: 16 (32 x 6) complex panels, warp per
// panel, column sums (the leaf forward transform of the q=1 far field), then __syncthreads.
// Prints cycles per level for several code shapes.  nvcc -O3 -arch=sm_100a colsum_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1703_01175_b200/csrc/h2b_panel.cuh"

constexpr int NP = 12;
__device__ __forceinline__ int sh_of(int w) { return w <= 1 ? 0 : 32 - __clz(w - 1); }

template <int MODE>
__global__ void k_lvl(int reps, int R, int w, long long* out, double2* sink) {
  __shared__ double2 P[NP * 32 * 6];
  __shared__ double2 xin[NP * 32];
  __shared__ double2 o[NP * 8];
  for (int i = threadIdx.x; i < NP * 32 * 6; i += blockDim.x) P[i] = make_double2(1e-3 * i, 1.0);
  for (int i = threadIdx.x; i < NP * 32; i += blockDim.x) xin[i] = make_double2(1.0, 1e-3 * i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    for (int n = warp; n < NP; n += 8) {
      const double2* p = P + n * R * w;
      const double2* in = xin + n * R;
      if (MODE == 0) {  // h2b_panel warp_panel_sum
        auto inf = [in](int r) { return in[r]; };
        const double2 s = warp_panel_sum(p, R, w, sh_of(w), inf);
        if (lane < w) o[n * 8 + lane] = s;
      } else if (MODE == 1) {  // lane per column, serial over rows (no shuffles)
        if (lane < w) {
          double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
          for (int r = 0; r < R; r += 4) {
            cfma(a0, p[r * w + lane], in[r]);
            cfma(a1, p[(r + 1) * w + lane], in[r + 1]);
            cfma(a2, p[(r + 2) * w + lane], in[r + 2]);
            cfma(a3, p[(r + 3) * w + lane], in[r + 3]);
          }
          o[n * 8 + lane] = cadd(cadd(a0, a1), cadd(a2, a3));
        }
      } else if (MODE == 3) {  // the same FMAs on register operands (no shared loads)
        if (lane < w) {
          double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
          const double2 pv = make_double2(1e-3 * lane, 1.0), xv = make_double2(1.0, 1e-3 * n);
          for (int r = 0; r < R; r += 4) {
            cfma(a0, pv, xv);
            cfma(a1, pv, xv);
            cfma(a2, pv, xv);
            cfma(a3, pv, xv);
          }
          o[n * 8 + lane] = cadd(cadd(a0, a1), cadd(a2, a3));
        }
      } else if (MODE == 4) {  // the loads only (integer-ish use)
        if (lane < w) {
          double acc = 0;
          for (int r = 0; r < R; r += 4) {
            const double2 q0 = p[r * w + lane], q1 = p[(r + 1) * w + lane], q2 = p[(r + 2) * w + lane], q3 = p[(r + 3) * w + lane];
            const double2 i0 = in[r], i1 = in[r + 1], i2 = in[r + 2], i3 = in[r + 3];
            acc += q0.x + q1.x + q2.x + q3.x + i0.y + i1.y + i2.y + i3.y;
          }
          o[n * 8 + lane] = make_double2(acc, 0);
        }
      } else {  // empty body: barrier + loop overhead only
        if (lane < w && it < 0) o[n * 8 + lane] = p[lane];
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
  if (threadIdx.x < 8) sink[threadIdx.x] = o[threadIdx.x];
}

// dependent DFMA chain latency
__global__ void k_dfma_lat(int n, double* out, long long* cyc) {
  double a = threadIdx.x * 1e-9, b = 1.0000001, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
}
__global__ void k_lds_lat(int n, long long* cyc, int* sink) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int j = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = s[j];
  long long t1 = clock64();
  sink[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
}
__global__ void k_bar_lat(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
}

int main() {
  long long* d;
  double2* sink;
  double* dd;
  int* di;
  cudaMalloc(&d, 1024 * 8);
  cudaMalloc(&sink, 1024 * 16);
  cudaMalloc(&dd, 1024 * 8);
  cudaMalloc(&di, 1024 * 4);
  long long h[4];
  k_dfma_lat<<<1, 32>>>(1000, dd, d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency: %lld cycles\n", h[0]);
  k_lds_lat<<<1, 32>>>(1000, d, di);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("dependent LDS latency: %lld cycles\n", h[0]);
  k_bar_lat<<<1, 256>>>(1000, d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (256 thr): %lld cycles\n", h[0]);
  for (int w : {6}) {
    k_lvl<0><<<1, 256>>>(200, 32, w, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("level 16 x (32x%d) warp_panel_sum: %lld cycles\n", w, h[0]);
    k_lvl<1><<<1, 256>>>(200, 32, w, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("level 16 x (32x%d) lane-per-column: %lld cycles\n", w, h[0]);
    k_lvl<3><<<1, 256>>>(200, 32, w, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("level FMAs only: %lld cycles\n", h[0]);
    k_lvl<4><<<1, 256>>>(200, 32, w, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("level loads (+DADD) only: %lld cycles\n", h[0]);
    k_lvl<2><<<1, 256>>>(200, 32, w, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("level empty: %lld cycles\n", h[0]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
