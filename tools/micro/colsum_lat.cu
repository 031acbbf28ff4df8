// Latency (one warp, one node) of small complex panel ops in shared memory on B200.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1703_01175_b200/csrc/h2b_panel.cuh"

__device__ __forceinline__ int sh_of(int w) { return w <= 1 ? 0 : 32 - __clz(w - 1); }

// V3: compile-time-free fast path: lane (g, c), rows r = g + G*i, all rows loaded first
template <int MAXI>
__device__ __forceinline__ double2 colsum_v3(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  double2 pv[MAXI], xv[MAXI];
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int r = g + G * i;
    const bool ok = c < w && r < R;
    pv[i] = ok ? P[r * w + c] : make_double2(0.0, 0.0);
    xv[i] = ok ? in[r] : make_double2(0.0, 0.0);
  }
  double2 a = make_double2(0.0, 0.0), b = a;
#pragma unroll
  for (int i = 0; i < MAXI; i += 2) {
    cfma(a, pv[i], xv[i]);
    if (i + 1 < MAXI) cfma(b, pv[i + 1], xv[i + 1]);
  }
  a = cadd(a, b);
  for (int m = wp; m < 32; m <<= 1) a = cadd(a, shfl_xor2(a, m));
  return a;
}

template <int MODE>
__global__ void k(int R, int w, long long* out, double2* sink, int reps) {
  __shared__ double2 P[64 * 16];
  __shared__ double2 xin[64];
  __shared__ double2 o[32];
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) P[i] = make_double2(1e-3 * i, 1.0);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) xin[i] = make_double2(1.0, 1e-3 * i);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  long long best = 1 << 30;
  for (int it = 0; it < reps; ++it) {
    __syncwarp();
    long long t0 = clock64();
    double2 s;
    if (MODE == 0) {
      auto inf = [](int r) { return xin[r]; };
      s = warp_panel_sum(P, R, w, sh_of(w), inf);
    } else {
      s = colsum_v3<4>(P, R, w, sh_of(w), xin);
    }
    if (lane < w) o[lane] = s;
    __syncwarp();
    long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  if (lane == 0) out[0] = best;
  sink[lane] = o[lane];
}

int main() {
  long long* d;
  double2* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 32 * 16);
  long long h;
  for (int R : {12, 16, 32}) for (int w : {6, 8}) {
    k<0><<<1, 32>>>(R, w, d, sink, 20);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("R %2d w %d warp_panel_sum %lld cycles", R, w, h);
    k<1><<<1, 32>>>(R, w, d, sink, 20);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("  | loads-first v3 %lld cycles\n", h);
  }
}
