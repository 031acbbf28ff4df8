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
