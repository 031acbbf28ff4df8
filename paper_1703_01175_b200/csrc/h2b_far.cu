// Far-field phases of the H² matvec (reference arith.py:58-99):
//   forward  x̂_c = V_cᵀ x_c, x̂_t = [T_lo;T_hi]ᵀ [x̂_lo; x̂_hi]      arith.py:58-71
//   coupling ŷ_t = Σ_s S^{t,s} x̂_s                                  arith.py:72-81
//   backward [ŷ_lo;ŷ_hi] += [T_lo;T_hi] ŷ_t ; y_c += V_c ŷ_c         arith.py:82-99
// (plain transposes, not conjugates: arith.py:10-12).
//
// q = 1 uses "span programs" (see SpanHead in h2b_common.cuh): one CTA per
// span stages its whole working set with TMA bulk copies (cp.async.bulk,
// one elected thread, completion on an mbarrier), then walks the levels of
// its span from shared memory with one __syncthreads per level, warp per
// cluster.  All addresses were resolved on the host, so a CTA issues no
// dependent global load.  Coupling is a gathered panel GEMV over the
// transposed coupling panels (one warp or one CTA per target).
// Any q: per-level kernels reading global memory (also the fallback for
// clusters whose working set does not fit in shared memory).
#include "h2b_span.cuh"

namespace {

constexpr int NT = 256;
constexpr int TOP_NT = 1024;

template <int NTH>
__global__ void __launch_bounds__(NTH) k_span(const SpanHead* __restrict__ heads, int head_base,
                                              const SpanCopy* __restrict__ copies,
                                              const SpanCopy* __restrict__ outs, SpanBases B) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double2 red[NTH];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  run_span<NTH>(heads + head_base + blockIdx.x, copies, outs, B, sm, red, &bar, 0);
}

// ---------------------------------------------------------------------------
// coupling, q = 1: ŷ_t = Σ_r Sᵀpanel_t[r, :] x̂[xcol[r]]  (overwrite)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_couple_warp(const CoupleItem* __restrict__ items, int n,
                                                    const double2* __restrict__ sbuf,
                                                    const int32_t* __restrict__ xcol,
                                                    const double2* __restrict__ xhat,
                                                    double2* __restrict__ yhat) {
  __shared__ double2 red[NT];
  const int warp = threadIdx.x >> 5;
  const int i = blockIdx.x * (NT / 32) + warp;
  if (i >= n) return;
  const CoupleItem it = items[i];
  double2* out = yhat + it.out;
  if (it.R == 0) {
    for (int c = threadIdx.x & 31; c < it.w; c += 32) out[c] = make_double2(0.0, 0.0);
    return;
  }
  const int32_t* xc = xcol + it.xcol;
  warp_panel<false>(sbuf + it.panel, it.R, it.w, [=](int r) { return xhat[xc[r]]; }, out,
                    red + warp * 32);
}

__global__ void __launch_bounds__(NT) k_couple_cta(const CoupleItem* __restrict__ items,
                                                   const double2* __restrict__ sbuf,
                                                   const int32_t* __restrict__ xcol,
                                                   const double2* __restrict__ xhat,
                                                   double2* __restrict__ yhat) {
  __shared__ double2 red[NT];
  const CoupleItem it = items[blockIdx.x];
  double2* out = yhat + it.out;
  if (it.R == 0) {
    for (int c = threadIdx.x; c < it.w; c += NT) out[c] = make_double2(0.0, 0.0);
    return;
  }
  const int32_t* xc = xcol + it.xcol;
  cta_panel_q<NT>(sbuf + it.panel, it.R, it.w,
                  [=] __device__(int64_t r, int) { return xhat[xc[r]]; }, out, false, 1, red);
}

// ---------------------------------------------------------------------------
// per-level / per-cluster kernels (any q; global memory)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_level_up(int p_begin, Tabs tb, const double2* __restrict__ vbuf,
                                                 const double2* __restrict__ tbuf,
                                                 const double2* __restrict__ x, double2* xhat, int q) {
  __shared__ double2 red[NT];
  const int p = p_begin + blockIdx.x;
  const int k = tb.c_rank[p];
  if (k == 0) return;
  const int lo = tb.c_lo[p];
  double2* out = xhat + tb.c_xoff[p] * q;
  if (lo < 0) {
    const double2* xs = x + (int64_t)tb.c_start[p] * q;
    cta_panel_q<NT>(vbuf + tb.c_voff[p], tb.c_size[p], k,
                    [=] __device__(int64_t r, int col) { return xs[r * q + col]; }, out, false, q, red);
  } else {
    const double2* xs = xhat + tb.c_xoff[lo] * q;
    const int m = tb.c_rank[lo] + tb.c_rank[tb.c_hi[p]];
    cta_panel_q<NT>(tbuf + tb.c_toff[p], m, k,
                    [=] __device__(int64_t r, int col) { return xs[r * q + col]; }, out, false, q, red);
  }
}

__global__ void __launch_bounds__(NT) k_level_down(int p_begin, Tabs tb, const double2* __restrict__ tT,
                                                   double2* yhat, int q) {
  __shared__ double2 red[NT];
  const int p = p_begin + blockIdx.x;
  const int k = tb.c_rank[p];
  const int lo = tb.c_lo[p];
  if (k == 0 || lo < 0) return;
  const int m = tb.c_rank[lo] + tb.c_rank[tb.c_hi[p]];
  if (m == 0) return;
  const double2* ys = yhat + tb.c_xoff[p] * q;
  cta_panel_q<NT>(tT + tb.c_toff[p], k, m,
                  [=] __device__(int64_t r, int col) { return ys[r * q + col]; },
                  yhat + tb.c_xoff[lo] * q, true, q, red);
}

// leaf back-transform y_c += V_c ŷ_c for the leaves of one level range
__global__ void __launch_bounds__(NT) k_leaf_back(const int32_t* __restrict__ leaves, Tabs tb,
                                                  const double2* __restrict__ vT,
                                                  const double2* __restrict__ yhat, double2* y, int q) {
  __shared__ double2 red[NT];
  const int p = leaves[blockIdx.x];
  const int k = tb.c_rank[p];
  if (k == 0) return;
  const double2* ys = yhat + tb.c_xoff[p] * q;
  cta_panel_q<NT>(vT + tb.c_voff[p], k, tb.c_size[p],
                  [=] __device__(int64_t r, int col) { return ys[r * q + col]; },
                  y + (int64_t)tb.c_start[p] * q, true, q, red);
}

// coupling, any q: ŷ_t = Σ_r Sᵀpanel_t[r,:] x̂[xcol[r]]
__global__ void __launch_bounds__(NT) k_coupling_q(const int32_t* __restrict__ targets, Tabs tb,
                                                   const int64_t* __restrict__ s_row_ptr,
                                                   const int64_t* __restrict__ s_off,
                                                   const int64_t* __restrict__ s_prow,
                                                   const int32_t* __restrict__ s_xcol,
                                                   const double2* __restrict__ sbuf,
                                                   const double2* __restrict__ xhat,
                                                   double2* __restrict__ yhat, int q) {
  __shared__ double2 red[NT];
  const int t = targets[blockIdx.x];
  const int kt = tb.c_rank[t];
  double2* out = yhat + tb.c_xoff[t] * q;
  const int64_t b0 = s_row_ptr[t], b1 = s_row_ptr[t + 1];
  const int64_t R = s_prow[t + 1] - s_prow[t];
  if (b0 == b1 || R == 0) {
    for (int e = threadIdx.x; e < kt * q; e += NT) out[e] = make_double2(0.0, 0.0);
    return;
  }
  const int32_t* xc = s_xcol + s_prow[t];
  cta_panel_q<NT>(sbuf + s_off[b0], R, kt,
                  [=] __device__(int64_t r, int col) { return xhat[(int64_t)xc[r] * q + col]; }, out,
                  false, q, red);
}

Tabs tabs_of(const h2b_ctx* h) {
  return Tabs{h->c_start_d, h->c_size_d, h->c_rank_d, h->c_lo, h->c_hi,
              h->c_xoff_d,  h->c_voff_d, h->c_toff_d};
}

SpanBases bases_of(const h2b_ctx* h, const double2* xp, double2* yp) {
  SpanBases B;
  B.src[SRC_V] = h->buf[H2B_SEC_V];
  B.src[SRC_T] = h->buf[H2B_SEC_T];
  B.src[SRC_VT] = h->vT;
  B.src[SRC_TT] = h->tT;
  B.src[SRC_X] = xp;
  B.src[SRC_XHAT] = h->xhat;
  B.src[SRC_YHAT] = h->yhat;
  B.src[SRC_OPS] = reinterpret_cast<const double2*>(h->span_ops);
  B.src[SRC_OUTS] = reinterpret_cast<const double2*>(h->span_outs);
  B.xhat = h->xhat;
  B.yhat = h->yhat;
  B.y = yp;
  B.ydeep = h->ydeep;
  return B;
}

}  // namespace

// dynamic shared memory cap of the span kernels (set once, process-wide)
int h2b_far_init_attributes(int smem_cap_bytes) {
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_span<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap_bytes));
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_span<TOP_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap_bytes));
  return H2B_OK;
}

// one launch of a span program (or the per-level fallback kernel it stands for)
int h2b_launch_span(h2b_ctx* h, const SpanLaunch& L, bool up, const double2* xp, double2* yp, int q,
                    cudaStream_t st) {
  const Tabs tb = tabs_of(h);
  if (L.level >= 0) {  // fallback: plain per-level kernel
    const int p0 = h->level_ptr[L.level], np = h->level_ptr[L.level + 1] - p0;
    if (up)
      k_level_up<<<np, NT, 0, st>>>(p0, tb, h->buf[H2B_SEC_V], h->buf[H2B_SEC_T], xp, h->xhat, q);
    else
      k_level_down<<<np, NT, 0, st>>>(p0, tb, h->tT, h->yhat, q);
    H2B_CHECK_LAUNCH();
    return H2B_OK;
  }
  const SpanBases B = bases_of(h, xp, yp);
  const size_t smem = 16 * (size_t)L.smem_elems;
  if (L.big)
    k_span<TOP_NT><<<L.n_heads, TOP_NT, smem, st>>>(h->span_heads, L.head_first, h->span_copies,
                                                     h->span_outs, B);
  else
    k_span<NT><<<L.n_heads, NT, smem, st>>>(h->span_heads, L.head_first, h->span_copies, h->span_outs,
                                            B);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

// q = 1 coupling on explicit work lists (plan handles): Sᵀ panels in `sbuf`, gathered x̂ rows
int h2b_launch_couple_list(const CoupleItem* items, int n, const double2* sbuf, const int32_t* xcol,
                           const double2* xhat, double2* yhat, int warp_mode, cudaStream_t st) {
  if (n <= 0) return H2B_OK;
  if (warp_mode)
    k_couple_warp<<<(n + NT / 32 - 1) / (NT / 32), NT, 0, st>>>(items, n, sbuf, xcol, xhat, yhat);
  else
    k_couple_cta<<<n, NT, 0, st>>>(items, sbuf, xcol, xhat, yhat);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_coupling(h2b_ctx* h, int q, cudaStream_t st) {
  const double2* sbuf = h->buf[H2B_SEC_S];
  if (q == 1) {
    if (h->n_couple_items == 0) return H2B_OK;
    if (h->couple_warp_mode)
      k_couple_warp<<<(h->n_couple_items + NT / 32 - 1) / (NT / 32), NT, 0, st>>>(
          h->couple_items, h->n_couple_items, sbuf, h->s_xcol, h->xhat, h->yhat);
    else
      k_couple_cta<<<h->n_couple_items, NT, 0, st>>>(h->couple_items, sbuf, h->s_xcol, h->xhat, h->yhat);
  } else {
    if (h->n_couple_targets == 0) return H2B_OK;
    k_coupling_q<<<h->n_couple_targets, NT, 0, st>>>(h->couple_targets, tabs_of(h), h->s_row_ptr_d,
                                                     h->s_off_d, h->s_prow, h->s_xcol, sbuf, h->xhat,
                                                     h->yhat, q);
  }
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

// generic (any q) far field: all levels up, coupling, all levels down (no leaf step)
int h2b_launch_far_levels_head(h2b_ctx* h, const double2* xp, int q, cudaStream_t st, int* nl) {
  const Tabs tb = tabs_of(h);
  for (int l : h->up_levels) {
    const int p0 = h->level_ptr[l], np = h->level_ptr[l + 1] - p0;
    k_level_up<<<np, NT, 0, st>>>(p0, tb, h->buf[H2B_SEC_V], h->buf[H2B_SEC_T], xp, h->xhat, q);
    H2B_CHECK_LAUNCH();
    ++*nl;
  }
  H2B_TRY(h2b_launch_coupling(h, q, st));
  ++*nl;
  for (int l : h->down_levels) {
    const int p0 = h->level_ptr[l], np = h->level_ptr[l + 1] - p0;
    k_level_down<<<np, NT, 0, st>>>(p0, tb, h->tT, h->yhat, q);
    H2B_CHECK_LAUNCH();
    ++*nl;
  }
  return H2B_OK;
}

int h2b_launch_leaf_back(h2b_ctx* h, double2* yp, int q, cudaStream_t st) {
  k_leaf_back<<<h->n_leaves, NT, 0, st>>>(h->leaves, tabs_of(h), h->vT, h->yhat, yp, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}
