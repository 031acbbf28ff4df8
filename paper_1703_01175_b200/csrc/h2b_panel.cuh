// Panel GEMV building blocks shared by the far-field kernels.
//
// Every far-field product of the H² matvec is written as
//     out[c] (+)= Σ_{r<R} P[r*w + c] · in(r)          (P: R x w, row-major)
// so each thread owns a fixed output column c, accumulates in registers and
// reads P in coalesced rows.  Groups of threads split the rows r when w is
// narrower than the thread group; their partials are combined in a fixed
// order (deterministic results).
#pragma once

#include "h2b_common.cuh"

// warp: out[c] (+)= Σ_r P[r*w+c] in(r)   (q = 1; P/out in smem or global)
template <bool ACC, class InF>
__device__ __forceinline__ void warp_panel(const double2* P, int R, int w, InF in, double2* out,
                                           double2* red) {
  const int lane = threadIdx.x & 31;
  if (w <= 32) {
    const int G = 32 / w;
    const int g = lane / w, c = lane - (lane / w) * w;
    double2 a = make_double2(0.0, 0.0);
    if (g < G) {
#pragma unroll 4
      for (int r = g; r < R; r += G) cfma(a, P[(int64_t)r * w + c], in(r));
    }
    red[lane] = a;
    __syncwarp();
    if (lane < w) {
      double2 s = red[lane];
      for (int gg = 1; gg < G; ++gg) s = cadd(s, red[gg * w + lane]);
      out[lane] = ACC ? cadd(out[lane], s) : s;
    }
    __syncwarp();
  } else {
    for (int c = lane; c < w; c += 32) {
      double2 a = make_double2(0.0, 0.0);
#pragma unroll 4
      for (int r = 0; r < R; ++r) cfma(a, P[(int64_t)r * w + c], in(r));
      out[c] = ACC ? cadd(out[c], a) : a;
    }
  }
}

// warp: out[c] (+)= Σ_r P[r*w+c] in(r) with the column groups precomputed on the host:
// wp = 1 << sh is w rounded up to a power of two (<= 32), G = 32 / wp row groups.  Lane
// (g, c) walks rows g, g+G, ... with four independent accumulators (short FP64 dependency
// chains, loads hoisted), then the G partial sums meet through xor shuffles.  For w > 32
// lanes loop over columns.  Deterministic: the summation order depends on the shape only.
// w <= 32: the reduced column sum, valid in lanes c < w
template <class InF>
__device__ __forceinline__ double2 warp_panel_sum(const double2* P, int R, int w, int sh, InF in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  if (c < w) {
    int r = g;
    for (; r + 3 * G < R; r += 4 * G) {
      const double2 p0 = P[r * w + c], p1 = P[(r + G) * w + c], p2 = P[(r + 2 * G) * w + c],
                    p3 = P[(r + 3 * G) * w + c];
      const double2 i0 = in(r), i1 = in(r + G), i2 = in(r + 2 * G), i3 = in(r + 3 * G);
      cfma(a0, p0, i0);
      cfma(a1, p1, i1);
      cfma(a2, p2, i2);
      cfma(a3, p3, i3);
    }
    if (r < R) cfma(a0, P[r * w + c], in(r));
    if (r + G < R) cfma(a1, P[(r + G) * w + c], in(r + G));
    if (r + 2 * G < R) cfma(a2, P[(r + 2 * G) * w + c], in(r + 2 * G));
  }
  a0 = cadd(cadd(a0, a1), cadd(a2, a3));
  for (int m = wp; m < 32; m <<= 1) a0 = cadd(a0, shfl_xor2(a0, m));
  return a0;
}

template <bool ACC, class InF>
__device__ __forceinline__ void warp_panel_fast(const double2* P, int R, int w, int sh, InF in,
                                                double2* out) {
  const int lane = threadIdx.x & 31;
  if (w <= 32) {
    const double2 a0 = warp_panel_sum(P, R, w, sh, in);
    if (lane < w) out[lane] = ACC ? cadd(out[lane], a0) : a0;
  } else {
    for (int c = lane; c < w; c += 32) {
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
      int r = 0;
      for (; r + 3 < R; r += 4) {
        const double2 p0 = P[r * w + c], p1 = P[(r + 1) * w + c], p2 = P[(r + 2) * w + c],
                      p3 = P[(r + 3) * w + c];
        cfma(a0, p0, in(r));
        cfma(a1, p1, in(r + 1));
        cfma(a2, p2, in(r + 2));
        cfma(a3, p3, in(r + 3));
      }
      for (; r < R; ++r) cfma(a0, P[r * w + c], in(r));
      a0 = cadd(cadd(a0, a1), cadd(a2, a3));
      out[c] = ACC ? cadd(out[c], a0) : a0;
    }
  }
}

// One out-of-line copy of the warp panel GEMV for the persistent kernel, whose
// task bodies otherwise overflow the instruction cache when CTAs switch between
// task types.  mode 0: out = sum; 1: out += sum; 2: out += sum with out in global
// memory written by another SM in the same launch (read through L2); 3: atomic
// out += sum in global memory (another kernel adds into it concurrently).
static __device__ __noinline__ void panel_op(const double2* P, int R, int w, int sh, const double2* in,
                                      double2* out, int mode) {
  const int lane = threadIdx.x & 31;
  auto inf = [in](int r) { return in[r]; };
  if (w <= 32) {
    double2 prev = make_double2(0.0, 0.0);
    if (mode == 2 && lane < w) prev = __ldcg(out + lane);
    const double2 s = warp_panel_sum(P, R, w, sh, inf);
    if (lane < w) {
      if (mode == 3) {
        atomicAdd(&out[lane].x, s.x);
        atomicAdd(&out[lane].y, s.y);
        return;
      }
      if (mode == 1) prev = out[lane];
      out[lane] = mode ? cadd(prev, s) : s;
    }
    return;
  }
  for (int c = lane; c < w; c += 32) {
    double2 a0 = make_double2(0.0, 0.0), a1 = a0;
    int r = 0;
    for (; r + 1 < R; r += 2) {
      cfma(a0, P[r * w + c], in[r]);
      cfma(a1, P[(r + 1) * w + c], in[r + 1]);
    }
    if (r < R) cfma(a0, P[r * w + c], in[r]);
    a0 = cadd(a0, a1);
    if (mode == 3) {
      atomicAdd(&out[c].x, a0.x);
      atomicAdd(&out[c].y, a0.y);
      continue;
    }
    const double2 prev = mode == 2 ? __ldcg(out + c) : (mode == 1 ? out[c] : make_double2(0.0, 0.0));
    out[c] = mode ? cadd(prev, a0) : a0;
  }
}

__host__ __device__ inline int panel_shift(int w) {
  int s = 0;
  while ((1 << s) < w && s < 5) ++s;
  return s;
}

// CTA of NTH threads: out[c*q+col] (+)= Σ_r P[r*w+c] in(r, col) for all q columns
template <int NTH, class InF>
__device__ __forceinline__ void cta_panel_q(const double2* __restrict__ P, int64_t R, int w, InF in,
                                            double2* out, bool acc, int q, double2* red) {
  const int tid = threadIdx.x;
  if (w <= NTH) {
    const int G = NTH / w;
    const int g = tid / w, c = tid - (tid / w) * w;
    for (int col = 0; col < q; ++col) {
      double2 a = make_double2(0.0, 0.0);
      if (g < G) {
#pragma unroll 8
        for (int64_t r = g; r < R; r += G) cfma(a, P[r * w + c], in(r, col));
      }
      red[tid] = a;
      __syncthreads();
      if (tid < w) {
        double2 s = red[tid];
        for (int gg = 1; gg < G; ++gg) s = cadd(s, red[gg * w + tid]);
        double2* o = out + (int64_t)tid * q + col;
        *o = acc ? cadd(*o, s) : s;
      }
      __syncthreads();
    }
  } else {
    for (int c = tid; c < w; c += NTH)
      for (int col = 0; col < q; ++col) {
        double2 a = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int64_t r = 0; r < R; ++r) cfma(a, P[r * w + c], in(r, col));
        double2* o = out + (int64_t)c * q + col;
        *o = acc ? cadd(*o, a) : a;
      }
  }
}

// Table pointers used by the per-level (any q) kernels
struct Tabs {
  const int32_t *c_start, *c_size, *c_rank, *c_lo, *c_hi;
  const int64_t *c_xoff, *c_voff, *c_toff;
};
