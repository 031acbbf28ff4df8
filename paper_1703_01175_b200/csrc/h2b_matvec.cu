// H² matvec kernels for sm_100a (B200).
//
// Restates the four phases of the reference `_apply_perm`
// (/root/reference/pkg/src/h2vie/arith.py:52-104) on the level-packed layout
// (paper_1703_01175_b200/pack.py):
//   (1) forward  x̂_c = V_cᵀ x_c (leaves), x̂_t = T_loᵀ x̂_lo + T_hiᵀ x̂_hi   arith.py:58-71
//   (2) coupling ŷ_t = Σ_s S^{t,s} x̂_s                                      arith.py:72-81
//   (3) backward ŷ_child += T_child ŷ_t ; y_c += V_c ŷ_c (leaves)           arith.py:82-99
//   (4) near     y_t += Σ_s D_{t,s} x_s                                      arith.py:100-104
// Plain transpose (not conjugate) in (1), as in the reference (arith.py:10-12).
//
// Execution plan: the near-field (the byte-dominant phase) runs on the
// caller's stream and overwrites y; the far-field chain (1)-(3) runs on a
// forked stream concurrently and the leaf back-transform joins it (it adds
// into y after the near-field finished).
#include <algorithm>

#include "h2b_common.cuh"

namespace {

constexpr int NT = 256;  // threads per CTA for all matvec kernels
constexpr int NWARP = NT / 32;

// ---------------------------------------------------------------------------
// near-field, q = 1, uniform leaf size NS (32 or 64): each lane streams
// 32-byte chunks (2 complex) of the contiguous row panel of its target leaf;
// partial sums stay in registers across all partner blocks and are reduced
// across the LPR lanes of a row once at the end.
// ---------------------------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(NT) k_near_q1(const int32_t* __restrict__ leaves,
                                                 const int32_t* __restrict__ c_start,
                                                 const int64_t* __restrict__ d_row_ptr,
                                                 const int32_t* __restrict__ d_col,
                                                 const int64_t* __restrict__ d_off,
                                                 const double2* __restrict__ dbuf,
                                                 const double2* __restrict__ x,
                                                 double2* __restrict__ y) {
  constexpr int LPR = NS / 2;          // lanes per row
  constexpr int RPW = 32 / LPR;        // rows per warp instruction
  constexpr int RSTEP = NWARP * RPW;   // row stride between a thread's rows
  constexpr int R = NS / RSTEP;        // rows per thread
  const int t = leaves[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = (lane % LPR) * 2;
  const int row0 = warp * RPW + lane / LPR;
  double2 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = make_double2(0.0, 0.0);
  const int64_t b0 = d_row_ptr[t], b1 = d_row_ptr[t + 1];
#pragma unroll 2
  for (int64_t b = b0; b < b1; ++b) {
    const double2* D = dbuf + d_off[b] + (int64_t)row0 * NS + col;
    const cd2 xv = ld_cached256(x + c_start[d_col[b]] + col);
    cd2 dv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) dv[r] = ld_stream256(D + (int64_t)r * RSTEP * NS);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cfma(acc[r], dv[r].a, xv.a);
      cfma(acc[r], dv[r].b, xv.b);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int m = LPR / 2; m > 0; m >>= 1) acc[r] = cadd(acc[r], shfl_xor2(acc[r], m));
  }
  if ((lane % LPR) == 0) {
    double2* yt = y + c_start[t] + row0;
#pragma unroll
    for (int r = 0; r < R; ++r) yt[r * RSTEP] = acc[r];
  }
}

// near-field, any sizes, any q: warp per (row, column)
__global__ void __launch_bounds__(NT) k_near_generic(const int32_t* __restrict__ leaves,
                                                      const int32_t* __restrict__ c_start,
                                                      const int32_t* __restrict__ c_size,
                                                      const int64_t* __restrict__ d_row_ptr,
                                                      const int32_t* __restrict__ d_col,
                                                      const int64_t* __restrict__ d_off,
                                                      const double2* __restrict__ dbuf,
                                                      const double2* __restrict__ x,
                                                      double2* __restrict__ y, int q) {
  const int t = leaves[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = c_size[t];
  const int64_t t0 = c_start[t];
  const int64_t b0 = d_row_ptr[t], b1 = d_row_ptr[t + 1];
  for (int i = warp; i < nt; i += NWARP) {
    for (int c = 0; c < q; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t b = b0; b < b1; ++b) {
        const int s = d_col[b];
        const int ns = c_size[s];
        const int64_t s0 = c_start[s];
        const double2* D = dbuf + d_off[b] + (int64_t)i * ns;
        for (int j = lane; j < ns; j += 32) cfma(acc, D[j], x[(s0 + j) * q + c]);
      }
      acc = warp_sum2(acc);
      if (lane == 0) y[(t0 + i) * q + c] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// small dense products used by the far field (CTA-cooperative)
// ---------------------------------------------------------------------------
// out[j*q+c] = Σ_i A[i*k+j] in[i*q+c]   (A row-major m x k; "Aᵀ in")
__device__ void cta_coldot(const double2* __restrict__ A, int m, int k,
                           const double2* __restrict__ in, int q, double2* __restrict__ out,
                           double2* smem) {
  const int tid = threadIdx.x;
  if (k <= NT) {
    const int G = NT / k;
    const int g = tid / k, j = tid % k;
    for (int c = 0; c < q; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      if (g < G)
        for (int i = g; i < m; i += G) cfma(acc, A[(int64_t)i * k + j], in[(int64_t)i * q + c]);
      if (g < G) smem[g * k + j] = acc;
      __syncthreads();
      for (int jj = tid; jj < k; jj += NT) {
        double2 s = smem[jj];
        for (int gg = 1; gg < G; ++gg) s = cadd(s, smem[gg * k + jj]);
        out[(int64_t)jj * q + c] = s;
      }
      __syncthreads();
    }
  } else {
    for (int j = tid; j < k; j += NT)
      for (int c = 0; c < q; ++c) {
        double2 acc = make_double2(0.0, 0.0);
        for (int i = 0; i < m; ++i) cfma(acc, A[(int64_t)i * k + j], in[(int64_t)i * q + c]);
        out[(int64_t)j * q + c] = acc;
      }
  }
}

// out[i*q+c] += Σ_j A[i*k+j] in[j*q+c]   (A row-major m x k; warp per row)
__device__ void cta_rowdot_acc(const double2* __restrict__ A, int m, int k,
                               const double2* __restrict__ in, int q, double2* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < m; i += NWARP)
    for (int c = 0; c < q; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = lane; j < k; j += 32) cfma(acc, A[(int64_t)i * k + j], in[(int64_t)j * q + c]);
      acc = warp_sum2(acc);
      if (lane == 0) out[(int64_t)i * q + c] = cadd(out[(int64_t)i * q + c], acc);
    }
}

// (1) forward transform of one level: leaves V_cᵀ x_c, non-leaves [T_lo;T_hi]ᵀ [x̂_lo;x̂_hi]
// (children are adjacent in their level list, so x̂_lo, x̂_hi are contiguous)
__global__ void __launch_bounds__(NT) k_up_level(int p_begin, const int32_t* __restrict__ c_start,
                                                 const int32_t* __restrict__ c_size,
                                                 const int32_t* __restrict__ c_rank,
                                                 const int32_t* __restrict__ c_lo,
                                                 const int32_t* __restrict__ c_hi,
                                                 const int64_t* __restrict__ c_xoff,
                                                 const int64_t* __restrict__ c_voff,
                                                 const int64_t* __restrict__ c_toff,
                                                 const double2* __restrict__ vbuf,
                                                 const double2* __restrict__ tbuf,
                                                 const double2* __restrict__ x, double2* xhat,
                                                 int q) {
  __shared__ double2 smem[NT];
  const int p = p_begin + blockIdx.x;
  const int k = c_rank[p];
  if (k == 0) return;
  const int lo = c_lo[p];
  if (lo < 0) {
    cta_coldot(vbuf + c_voff[p], c_size[p], k, x + (int64_t)c_start[p] * q, q,
               xhat + c_xoff[p] * q, smem);
  } else {
    const int m = c_rank[lo] + c_rank[c_hi[p]];
    cta_coldot(tbuf + c_toff[p], m, k, xhat + c_xoff[lo] * q, q, xhat + c_xoff[p] * q, smem);
  }
}

// (2) coupling: ŷ_t = Σ_b S_b x̂_{s_b}, overwrite (zeros when no block)
__global__ void __launch_bounds__(NT) k_coupling(const int32_t* __restrict__ c_rank,
                                                 const int64_t* __restrict__ c_xoff,
                                                 const int64_t* __restrict__ s_row_ptr,
                                                 const int32_t* __restrict__ s_col,
                                                 const int64_t* __restrict__ s_off,
                                                 const double2* __restrict__ sbuf,
                                                 const double2* __restrict__ xhat,
                                                 double2* __restrict__ yhat, int q) {
  const int t = blockIdx.x;
  const int kt = c_rank[t];
  if (kt == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = s_row_ptr[t], b1 = s_row_ptr[t + 1];
  double2* yt = yhat + c_xoff[t] * q;
  for (int i = warp; i < kt; i += NWARP)
    for (int c = 0; c < q; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t b = b0; b < b1; ++b) {
        const int s = s_col[b];
        const int ks = c_rank[s];
        const double2* S = sbuf + s_off[b] + (int64_t)i * ks;
        const double2* xs = xhat + c_xoff[s] * q;
        for (int j = lane; j < ks; j += 32) cfma(acc, S[j], xs[(int64_t)j * q + c]);
      }
      acc = warp_sum2(acc);
      if (lane == 0) yt[(int64_t)i * q + c] = acc;
    }
}

// (3a) backward transfer of one level: [ŷ_lo;ŷ_hi] += [T_lo;T_hi] ŷ_p
__global__ void __launch_bounds__(NT) k_down_level(int p_begin, const int32_t* __restrict__ c_rank,
                                                   const int32_t* __restrict__ c_lo,
                                                   const int32_t* __restrict__ c_hi,
                                                   const int64_t* __restrict__ c_xoff,
                                                   const int64_t* __restrict__ c_toff,
                                                   const double2* __restrict__ tbuf,
                                                   double2* yhat, int q) {
  const int p = p_begin + blockIdx.x;
  const int k = c_rank[p];
  const int lo = c_lo[p];
  if (k == 0 || lo < 0) return;
  const int m = c_rank[lo] + c_rank[c_hi[p]];
  if (m == 0) return;
  cta_rowdot_acc(tbuf + c_toff[p], m, k, yhat + c_xoff[p] * q, q, yhat + c_xoff[lo] * q);
}

// (3b) leaf back-transform: y_c += V_c ŷ_c
__global__ void __launch_bounds__(NT) k_leaf_back(const int32_t* __restrict__ leaves,
                                                  const int32_t* __restrict__ c_start,
                                                  const int32_t* __restrict__ c_size,
                                                  const int32_t* __restrict__ c_rank,
                                                  const int64_t* __restrict__ c_xoff,
                                                  const int64_t* __restrict__ c_voff,
                                                  const double2* __restrict__ vbuf,
                                                  const double2* __restrict__ yhat, double2* y,
                                                  int q) {
  const int p = leaves[blockIdx.x];
  const int k = c_rank[p];
  if (k == 0) return;
  cta_rowdot_acc(vbuf + c_voff[p], c_size[p], k, yhat + c_xoff[p] * q, q,
                 y + (int64_t)c_start[p] * q);
}

__global__ void k_gather(const int64_t* __restrict__ perm, int64_t n, const double2* __restrict__ in,
                         double2* __restrict__ out, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / q, c = e - i * q;
    out[e] = in[perm[i] * q + c];
  }
}

__global__ void k_scatter(const int64_t* __restrict__ perm, int64_t n, const double2* __restrict__ in,
                          double2* __restrict__ out, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / q, c = e - i * q;
    out[perm[i] * q + c] = in[e];
  }
}

int grid_for(int64_t tot) {
  int64_t g = (tot + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

}  // namespace

int h2b_launch_gather(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                      cudaStream_t st) {
  k_gather<<<grid_for(n * q), 256, 0, st>>>(perm, n, in, out, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_scatter(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                       cudaStream_t st) {
  k_scatter<<<grid_for(n * q), 256, 0, st>>>(perm, n, in, out, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_ensure_workspace(h2b_ctx* h, int q) {
  if (q <= h->ws_q) return H2B_OK;
  if (h->xhat) cudaFree(h->xhat);
  if (h->yhat) cudaFree(h->yhat);
  h->xhat = h->yhat = nullptr;
  h->device_bytes -= 2 * 16 * h->K * h->ws_q;
  h->ws_q = 0;
  const size_t bytes = (size_t)16 * std::max<int64_t>(h->K, 1) * q;
  H2B_CUDA_TRY(cudaMalloc(&h->xhat, bytes));
  H2B_CUDA_TRY(cudaMalloc(&h->yhat, bytes));
  h->ws_q = q;
  h->device_bytes += 2 * 16 * h->K * q;
  return H2B_OK;
}

int h2b_run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st) {
  int rc = h2b_ensure_workspace(h, q);
  if (rc) return rc;
  const double2 *vbuf = h->buf[H2B_SEC_V], *tbuf = h->buf[H2B_SEC_T], *sbuf = h->buf[H2B_SEC_S],
                *dbuf = h->buf[H2B_SEC_D];
  // (4) near-field: overwrites every row of y (each leaf owns its diagonal block)
  if (q == 1 && h->uniform_leaf == 32) {
    k_near_q1<32><<<h->n_leaves, NT, 0, st>>>(h->leaves, h->c_start, h->d_row_ptr, h->d_col,
                                                h->d_off, dbuf, xp, yp);
  } else if (q == 1 && h->uniform_leaf == 64) {
    k_near_q1<64><<<h->n_leaves, NT, 0, st>>>(h->leaves, h->c_start, h->d_row_ptr, h->d_col,
                                                h->d_off, dbuf, xp, yp);
  } else {
    k_near_generic<<<h->n_leaves, NT, 0, st>>>(h->leaves, h->c_start, h->c_size_d, h->d_row_ptr,
                                               h->d_col, h->d_off, dbuf, xp, yp, q);
  }
  H2B_CHECK_LAUNCH();
  if (h->K == 0) return H2B_OK;
  // (1) forward, deepest level first
  for (int l : h->up_levels) {
    const int p0 = h->level_ptr[l], np = h->level_ptr[l + 1] - p0;
    k_up_level<<<np, NT, 0, st>>>(p0, h->c_start, h->c_size_d, h->c_rank_d, h->c_lo, h->c_hi,
                                  h->c_xoff, h->c_voff, h->c_toff, vbuf, tbuf, xp, h->xhat, q);
    H2B_CHECK_LAUNCH();
  }
  // (2) coupling
  k_coupling<<<h->P, NT, 0, st>>>(h->c_rank_d, h->c_xoff, h->s_row_ptr, h->s_col, h->s_off, sbuf,
                                  h->xhat, h->yhat, q);
  H2B_CHECK_LAUNCH();
  // (3) backward, root level first
  for (int l : h->down_levels) {
    const int p0 = h->level_ptr[l], np = h->level_ptr[l + 1] - p0;
    k_down_level<<<np, NT, 0, st>>>(p0, h->c_rank_d, h->c_lo, h->c_hi, h->c_xoff, h->c_toff, tbuf,
                                    h->yhat, q);
    H2B_CHECK_LAUNCH();
  }
  k_leaf_back<<<h->n_leaves, NT, 0, st>>>(h->leaves, h->c_start, h->c_size_d, h->c_rank_d,
                                          h->c_xoff, h->c_voff, vbuf, h->yhat, yp, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}
