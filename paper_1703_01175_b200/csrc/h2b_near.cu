// Near-field phase of the H² matvec: y_t = Σ_s D_{t,s} x_s over inadmissible
// leaf pairs (reference: /root/reference/pkg/src/h2vie/arith.py:100-104; the
// dense blocks come from build.py:321-324 and are kept row-major, the
// reference layout).  This phase holds 60-87 % of the operator's bytes
// (SURVEY.md §0 finding 3), so it decides the HBM roofline fraction.
//
// q = 1, uniform leaf size NS (32 or 64): `k_near_q1<NS, R>`.
//   * A CTA of 128 threads owns RB = R*128/(NS/2) consecutive rows of one
//     target leaf (work item), so both small and large operators give enough
//     CTAs to fill 148 SMs.
//   * Each thread owns R rows and one 2-column pair; it streams its 32-byte
//     row chunk of every partner block with a 256-bit non-allocating load
//     (LDG.E.ENL2.256), UNR = 8/R blocks per batch, i.e. 8 loads in flight
//     per thread.
//   * The partner list (block offset, x column) and the x segments of a
//     chunk of partners are staged in shared memory once per CTA, so the
//     streaming loop has no dependent global loads and x is read once per CTA.
//   * Partial sums stay in registers across all partners and are reduced once
//     across the NS/2 threads of a row.
// Any other shape / q: `k_near_generic` (warp per row, q loop).
#include "h2b_panel.cuh"

namespace {

constexpr int NEAR_NT = 128;
constexpr int NEAR_CHUNK = 32;  // partner blocks staged per pass

template <int NS, int R>
__global__ void __launch_bounds__(NEAR_NT, 4) k_near_q1(const NearItem* __restrict__ items,
                                                        const NearBlk* __restrict__ blks,
                                                        const double2* __restrict__ dbuf,
                                                        const double2* __restrict__ x,
                                                        double2* __restrict__ y) {
  constexpr int LPR = NS / 2;                 // threads per row
  constexpr int RPP = NEAR_NT / LPR;          // rows per pass of the CTA
  constexpr int UNR = 8 / R;                  // partner blocks per load batch
  __shared__ __align__(32) double2 xs[NEAR_CHUNK * NS];
  __shared__ int64_t sd[NEAR_CHUNK];
  const NearItem it = items[blockIdx.x];
  const int r0 = threadIdx.x / LPR;           // first row of this thread (within the item)
  const int col = (threadIdx.x % LPR) * 2;
  double2 acc[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < it.nb; c0 += NEAR_CHUNK) {
    const int nb = min(NEAR_CHUNK, it.nb - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * LPR; e += NEAR_NT) {
      const int b = e / LPR, j = (e - b * LPR) * 2;
      const NearBlk bl = blks[it.b_first + c0 + b];
      const cd2 v = ld_cached256(x + bl.x_off + j);
      xs[b * NS + j] = v.a;
      xs[b * NS + j + 1] = v.b;
      if (j == 0) sd[b] = bl.d_off;
    }
    __syncthreads();
    for (int i0 = 0; i0 < nb; i0 += UNR) {
      cd2 dv[UNR][R];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (i0 + u < nb) {
          const double2* D = dbuf + sd[i0 + u] + (int64_t)(it.row0 + r0) * NS + col;
#pragma unroll
          for (int r = 0; r < R; ++r) dv[u][r] = ld_stream256(D + (int64_t)r * RPP * NS);
        }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (i0 + u < nb) {
          const double2 xa = xs[(i0 + u) * NS + col], xb = xs[(i0 + u) * NS + col + 1];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            cfma(acc[r][0], dv[u][r].a, xa);
            cfma(acc[r][1], dv[u][r].b, xb);
          }
        }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double2 a = cadd(acc[r][0], acc[r][1]);
#pragma unroll
    for (int m = LPR / 2; m > 0; m >>= 1) a = cadd(a, shfl_xor2(a, m));
    if ((threadIdx.x % LPR) == 0) y[it.y_off + r0 + r * RPP] = a;
  }
}

// near-field, any sizes, any q: warp per row, q loop
constexpr int NT = 256;
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
  for (int i = warp; i < nt; i += NT / 32) {
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

template <int NS, int R>
void launch_q1(const h2b_ctx* h, const double2* xp, double2* yp, cudaStream_t st) {
  k_near_q1<NS, R><<<h->n_near_items, NEAR_NT, 0, st>>>(h->near_items, h->near_blks,
                                                        h->buf[H2B_SEC_D], xp, yp);
}

}  // namespace

// rows per CTA of the q=1 kernel for a leaf size (0 = not supported)
int h2b_near_rows_per_item(int ns, int r) { return (ns == 32 || ns == 64) ? r * NEAR_NT / (ns / 2) : 0; }

// the q=1 streaming kernel on explicit work lists (plan handles: one rank's near-field rows,
// x columns in the exchange buffer); y rows overwritten
int h2b_launch_near_list(const NearItem* items, int n_items, const NearBlk* blks, const double2* dbuf,
                         const double2* x, double2* y, int ns, int R, cudaStream_t st) {
  if (n_items <= 0) return H2B_OK;
#define NL(A, B)                                                                           \
  if (ns == A && R == B) k_near_q1<A, B><<<n_items, NEAR_NT, 0, st>>>(items, blks, dbuf, x, y); \
  else
  NL(32, 1) NL(32, 2) NL(32, 4) NL(64, 1) NL(64, 2) NL(64, 4) {
    h2b_set_error("h2b_launch_near_list: unsupported leaf size / rows per thread");
    return H2B_EINVAL;
  }
#undef NL
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_near(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st) {
  if (q == 1 && h->near_rb > 0) {
    const int ns = h->uniform_leaf, R = h->near_rb * (ns / 2) / NEAR_NT;
    if (ns == 32 && R == 1) launch_q1<32, 1>(h, xp, yp, st);
    else if (ns == 32 && R == 2) launch_q1<32, 2>(h, xp, yp, st);
    else if (ns == 32 && R == 4) launch_q1<32, 4>(h, xp, yp, st);
    else if (ns == 64 && R == 1) launch_q1<64, 1>(h, xp, yp, st);
    else if (ns == 64 && R == 2) launch_q1<64, 2>(h, xp, yp, st);
    else launch_q1<64, 4>(h, xp, yp, st);
  } else {
    k_near_generic<<<h->n_leaves, NT, 0, st>>>(h->leaves, h->c_start_d, h->c_size_d, h->d_row_ptr_d,
                                               h->d_col_d, h->d_off_d, h->buf[H2B_SEC_D], xp, yp, q);
  }
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}
