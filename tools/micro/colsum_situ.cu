// One-shot vs repeated latency of the tree kernel's colsum (h2b_tree.cu), 1 or 8 warps per CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1703_01175_b200/csrc/h2b_common.cuh"

__device__ __forceinline__ double2 colsum_sum(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  double2 a = make_double2(0.0, 0.0), b = a;
  for (int r0 = g; r0 < R; r0 += 4 * G) {
    double2 pv[4], xv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * G;
      const bool ok = c < w && r < R;
      pv[i] = ok ? P[r * w + c] : make_double2(0.0, 0.0);
      xv[i] = ok ? in[r] : make_double2(0.0, 0.0);
    }
    cfma(a, pv[0], xv[0]);
    cfma(b, pv[1], xv[1]);
    cfma(a, pv[2], xv[2]);
    cfma(b, pv[3], xv[3]);
  }
  a = cadd(a, b);
  for (int m = wp; m < 32; m <<= 1) a = cadd(a, shfl_xor2(a, m));
  return a;
}


// V2: unconditional loads from clamped (always valid) addresses, zeroed by a select afterwards
__device__ __forceinline__ double2 colsum_v2(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  const int cc = c < w ? c : w - 1;
  double2 a = make_double2(0.0, 0.0), b = a;
  for (int r0 = g; r0 < R; r0 += 4 * G) {
    double2 pv[4], xv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * G;
      const int rc = r < R ? r : R - 1;
      pv[i] = P[rc * w + cc];
      xv[i] = in[rc];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = c < w && r0 + i * G < R;
      if (!ok) pv[i] = make_double2(0.0, 0.0);
    }
    cfma(a, pv[0], xv[0]);
    cfma(b, pv[1], xv[1]);
    cfma(a, pv[2], xv[2]);
    cfma(b, pv[3], xv[3]);
  }
  a = cadd(a, b);
  for (int m = wp; m < 32; m <<= 1) a = cadd(a, shfl_xor2(a, m));
  return a;
}
__device__ __forceinline__ void lds4(const double2* p0, const double2* p1, const double2* p2, const double2* p3,
                                     double2& v0, double2& v1, double2& v2, double2& v3) {
  asm volatile(
      "ld.shared.v2.f64 {%0, %1}, [%8];\n\t"
      "ld.shared.v2.f64 {%2, %3}, [%9];\n\t"
      "ld.shared.v2.f64 {%4, %5}, [%10];\n\t"
      "ld.shared.v2.f64 {%6, %7}, [%11];"
      : "=d"(v0.x), "=d"(v0.y), "=d"(v1.x), "=d"(v1.y), "=d"(v2.x), "=d"(v2.y), "=d"(v3.x), "=d"(v3.y)
      : "r"((unsigned)__cvta_generic_to_shared(p0)), "r"((unsigned)__cvta_generic_to_shared(p1)),
        "r"((unsigned)__cvta_generic_to_shared(p2)), "r"((unsigned)__cvta_generic_to_shared(p3)));
}
// V3: V2 with the loads in one asm block (issue order forced)
__device__ __forceinline__ double2 colsum_v3(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  const int cc = c < w ? c : w - 1;
  double2 a = make_double2(0.0, 0.0), b = a;
  for (int r0 = g; r0 < R; r0 += 4 * G) {
    double2 pv[4], xv[4];
    int rc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * G;
      rc[i] = r < R ? r : R - 1;
    }
    lds4(P + rc[0] * w + cc, P + rc[1] * w + cc, P + rc[2] * w + cc, P + rc[3] * w + cc, pv[0], pv[1], pv[2], pv[3]);
    lds4(in + rc[0], in + rc[1], in + rc[2], in + rc[3], xv[0], xv[1], xv[2], xv[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = c < w && r0 + i * G < R;
      if (!ok) pv[i] = make_double2(0.0, 0.0);
    }
    cfma(a, pv[0], xv[0]);
    cfma(b, pv[1], xv[1]);
    cfma(a, pv[2], xv[2]);
    cfma(b, pv[3], xv[3]);
  }
  a = cadd(a, b);
  for (int m = wp; m < 32; m <<= 1) a = cadd(a, shfl_xor2(a, m));
  return a;
}

__device__ __forceinline__ double2 v4(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh;
  double2 a = make_double2(lane, 1.0);
  for (int m = wp; m < 32; m <<= 1) a = cadd(a, shfl_xor2(a, m));
  return a;
}
__device__ __forceinline__ double2 v5(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh;
  double2 a = make_double2(lane, 1.0);
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) if (m >= wp) a = cadd(a, shfl_xor2(a, m));
  return a;
}
// V6: column-serial (lane c < w sums its column over all rows; no shuffles), 4-row chunks
__device__ __forceinline__ double2 v6(const double2* P, int R, int w, int sh, const double2* in) {
  const int c = threadIdx.x & 31;
  double2 a0 = make_double2(0.0, 0.0), a1 = a0;
  if (c < w) {
    int r = 0;
    for (; r + 4 <= R; r += 4) {
      const double2 p0 = P[r * w + c], p1 = P[(r + 1) * w + c], p2 = P[(r + 2) * w + c], p3 = P[(r + 3) * w + c];
      const double2 x0 = in[r], x1 = in[r + 1], x2 = in[r + 2], x3 = in[r + 3];
      cfma(a0, p0, x0); cfma(a1, p1, x1); cfma(a0, p2, x2); cfma(a1, p3, x3);
    }
    for (; r < R; ++r) cfma(a0, P[r * w + c], in[r]);
  }
  return cadd(a0, a1);
}
// V7: column-serial, 8-row chunks, 4 accumulators
__device__ __forceinline__ double2 v7(const double2* P, int R, int w, int sh, const double2* in) {
  const int c = threadIdx.x & 31;
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  if (c < w) {
    int r = 0;
    for (; r + 8 <= R; r += 8) {
      double2 p[8], x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) { p[i] = P[(r + i) * w + c]; x[i] = in[r + i]; }
      cfma(a0, p[0], x[0]); cfma(a1, p[1], x[1]); cfma(a2, p[2], x[2]); cfma(a3, p[3], x[3]);
      cfma(a0, p[4], x[4]); cfma(a1, p[5], x[5]); cfma(a2, p[6], x[6]); cfma(a3, p[7], x[7]);
    }
    for (; r + 4 <= R; r += 4) {
      const double2 p0 = P[r * w + c], p1 = P[(r + 1) * w + c], p2 = P[(r + 2) * w + c], p3 = P[(r + 3) * w + c];
      const double2 x0 = in[r], x1 = in[r + 1], x2 = in[r + 2], x3 = in[r + 3];
      cfma(a0, p0, x0); cfma(a1, p1, x1); cfma(a2, p2, x2); cfma(a3, p3, x3);
    }
    for (; r < R; ++r) cfma(a0, P[r * w + c], in[r]);
  }
  return cadd(cadd(a0, a1), cadd(a2, a3));
}
template <int V>
__global__ void k(int R, int w, int sh, long long* out, double2* sink) {
  extern __shared__ double2 sm[];
  double2* P = sm + (threadIdx.x >> 5) * 1024;
  double2* xin = sm + 8 * 1024 + (threadIdx.x >> 5) * 64;
  double2* o = sm + 8 * 1024 + 8 * 64 + (threadIdx.x >> 5) * 32;
  for (int i = threadIdx.x & 31; i < 1024; i += 32) P[i] = make_double2(1e-3 * i, 1.0);
  for (int i = threadIdx.x & 31; i < 64; i += 32) xin[i] = make_double2(1.0, 1e-3 * i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  long long t[4];
  for (int it = 0; it < 4; ++it) {
    __syncwarp();
    const long long t0 = clock64();
    const double2 s = V == 1 ? colsum_sum(P, R, w, sh, xin) : V == 2 ? colsum_v2(P, R, w, sh, xin) : V == 3 ? colsum_v3(P, R, w, sh, xin) : V == 4 ? v4(P, R, w, sh, xin) : V == 5 ? v5(P, R, w, sh, xin) : V == 6 ? v6(P, R, w, sh, xin) : v7(P, R, w, sh, xin);
    if (lane < w) o[lane] = s;
    t[it] = clock64() - t0;
  }
  if (lane == 0 && threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) out[i] = t[i];
  sink[threadIdx.x] = o[lane];
}

int main() {
  long long* d;
  double2* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 256 * 16);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long h[4];
  int cases[][3] = {{4, 3, 2}, {14, 7, 3}, {24, 8, 3}, {32, 6, 3}, {48, 8, 3}};
  for (auto& c : cases)
    for (int v = 1; v <= 7; ++v) {
      if (v == 4 || v == 5) continue;
      const int nt = 256;
      if (v == 1) k<1><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 2) k<2><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 4) k<4><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 5) k<5><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 6) k<6><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 7) k<7><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      if (v == 3) k<3><<<1, nt, (8 * 1024 + 8 * 64 + 8 * 32) * 16>>>(c[0], c[1], c[2], d, sink);
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("R %2d w %d v%d: calls %lld %lld %lld %lld cycles\n", c[0], c[1], v, h[0], h[1], h[2], h[3]);
    }
  return 0;
}
