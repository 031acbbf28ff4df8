// Block GMRES(m) for q right-hand sides on device (sm_100a) — BASELINE config 5.
//
// New component (the reference has no GMRES, SURVEY.md §0 finding 1); restates the CPU oracle
// oracle/krylov_oracle.py::block_gmres_solve step for step: x0 = 0, block Arnoldi with block
// CGS2, a QR of every new block, restart after m blocks, converged when every column's TRUE
// relative residual is <= tol at the end of a cycle; `iterations` counts block Arnoldi steps and
// the history holds the max over columns of the least-squares residual relative to ||b_j||.
//
// Everything runs on libh2b kernels:
//   * the operator: the H² matvec with q columns (h2b_mrhs.cu, FP64 tensor pipe);
//   * tall-skinny complex products V^H W (k_bgram + k_breduce: row chunks x basis blocks, then a
//     fixed-order sum of the chunk partials: deterministic) and W -= V C (k_bupdate), register-
//     tiled DFMA kernels (on B200 the FP64 CUDA-core rate equals the DMMA rate, 37 TF measured);
//   * the QR of each N x q block as CholQR2 (Gram on device, k_chol_small: Cholesky + triangular
//     inverse of the q x q Gram matrix in one CTA, W R^-1 by k_bupdate, twice);
//   * the small least-squares problem min ||E0 - H_j Y|| without host work: the block columns of
//     the block Hessenberg H are orthonormalised incrementally in the small (m+1)q-dimensional
//     space with the same kernels (block CGS2 + CholQR2: H_j = Qs_j Rs_j), the projected
//     residual Eres = E0 - Qs Qs^H E0 is updated per step and its column norms give the exact
//     least-squares residual; k_bres writes max_c ||Eres_c|| / ||b_c|| into mapped pinned memory.
//     The host reads it one step behind the GPU (the next step is already queued) and solves
//     Rs Y = Qs^H E0 by block back substitution on the device only at the end of a cycle.
#include <math.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "h2b_common.cuh"

namespace {

constexpr int BQ = 64;        // max right-hand sides per block
constexpr int GT = 256;       // threads of the GEMM kernels
constexpr int KR = 16;        // rows per smem tile of k_bgram / k-slice of k_bupdate
constexpr int MROWS = 32;     // output rows per CTA of k_bupdate
constexpr int CHOL_SMEM = 3 * BQ * (BQ + 1) * 16;  // k_chol_small: G (updated), R and R^-1

// ---------------------------------------------------------------------------------------------
// k_bgram: partial[(blk * nchunk + c)] (q x q) = Σ_{r in chunk c} conj(A_blk[r][a]) B[r][b]
// A_blk = A + blk * astride (rows x q, row-major), B rows x q.  Thread (ta, tb) owns outputs
// a = ta*4 .. +3, b = tb*4 .. +3 (16 x 16 threads cover 64 x 64).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(GT) k_bgram(const double2* __restrict__ A, int64_t astride,
                                              const double2* __restrict__ B, int64_t rows, int q,
                                              int64_t chunk, int nchunk, double2* __restrict__ part) {
  __shared__ double2 As[KR][BQ + 1], Bs[KR][BQ + 1];
  const int blk = blockIdx.y, c = blockIdx.x;
  const double2* Ab = A + blk * astride;
  const int64_t r0 = (int64_t)c * chunk, r1 = rows < r0 + chunk ? rows : r0 + chunk;
  const int tid = threadIdx.x, ta = tid >> 4, tb = tid & 15;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  for (int64_t rt = r0; rt < r1; rt += KR) {
    const int nr = (int)(r1 - rt < KR ? r1 - rt : KR);
    for (int e = tid; e < KR * BQ; e += GT) {
      const int r = e / BQ, col = e % BQ;
      const bool ok = r < nr && col < q;
      As[r][col] = ok ? Ab[(rt + r) * q + col] : make_double2(0.0, 0.0);
      Bs[r][col] = ok ? B[(rt + r) * q + col] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < KR; ++r) {
      double2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[r][ta * 4 + i];
        b[i] = Bs[r][tb * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma_conj(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  double2* out = part + ((int64_t)blk * nchunk + c) * q * q;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = ta * 4 + i, b = tb * 4 + j;
      if (a < q && b < q) out[a * q + b] = acc[i][j];
    }
}

// C[blk] (q x q, block row blk of a (nblk q) x q matrix) (+)= alpha Σ_c partial[blk][c], fixed order
__global__ void k_breduce(const double2* __restrict__ part, int nblk, int nchunk, int q, double2* C,
                          int accumulate) {
  const int64_t tot = (int64_t)nblk * q * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = e / ((int64_t)q * q), o = e % ((int64_t)q * q);
    double2 s = make_double2(0.0, 0.0);
    for (int c = 0; c < nchunk; ++c) s = cadd(s, part[(blk * nchunk + c) * q * q + o]);
    C[e] = accumulate ? cadd(C[e], s) : s;
  }
}

// ---------------------------------------------------------------------------------------------
// k_bupdate: Out[r][b] = beta * In[r][b] + alpha * Σ_blk Σ_a A_blk[r][a] C_blk[a][b]
// A_blk = A + blk * astride (rows x q), C_blk = C + blk * q * q (q x q).  One CTA: 64 rows;
// thread (tr, tb) owns rows tr*4..+3, columns tb*4..+3.  In may alias Out.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(GT) k_bupdate(const double2* __restrict__ A, int64_t astride, int nblk,
                                                const double2* __restrict__ C, const double2* In,
                                                double2* Out, int64_t rows, int q, double alpha,
                                                double beta) {
  __shared__ double2 As[MROWS][KR + 1], Cs[KR][BQ + 1];
  const int64_t r0 = (int64_t)blockIdx.x * MROWS;
  const int tid = threadIdx.x, tr = tid >> 4, tb = tid & 15;
  constexpr int RPT = MROWS / 16;  // rows per thread
  double2 acc[RPT][4];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  const int K = nblk * q;
  for (int k0 = 0; k0 < K; k0 += KR) {
    for (int e = tid; e < MROWS * KR; e += GT) {
      const int r = e / KR, kk = e % KR, k = k0 + kk;
      const int64_t row = r0 + r;
      double2 v = make_double2(0.0, 0.0);
      if (row < rows && k < K) {
        const int blk = k / q, a = k % q;
        v = A[blk * astride + row * q + a];
      }
      As[r][kk] = v;
    }
    for (int e = tid; e < KR * BQ; e += GT) {
      const int kk = e / BQ, b = e % BQ, k = k0 + kk;
      double2 v = make_double2(0.0, 0.0);
      if (k < K && b < q) {
        const int blk = k / q, a = k % q;
        v = C[(int64_t)blk * q * q + a * q + b];
      }
      Cs[kk][b] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KR; ++kk) {
      double2 a[RPT], c[4];
#pragma unroll
      for (int i = 0; i < RPT; ++i) a[i] = As[tr * RPT + i][kk];
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = Cs[kk][tb * 4 + i];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma(acc[i][j], a[i], c[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t row = r0 + tr * RPT + i;
      const int b = tb * 4 + j;
      if (row < rows && b < q) {
        const double2 v = acc[i][j];
        double2 o = make_double2(alpha * v.x, alpha * v.y);
        if (beta != 0.0) {
          const double2 w = In[row * q + b];
          o.x = fma(beta, w.x, o.x);
          o.y = fma(beta, w.y, o.y);
        }
        Out[row * q + b] = o;
      }
    }
}

// ---------------------------------------------------------------------------------------------
// k_chol_small (one CTA): G (q x q, Hermitian) = R^H R with R upper triangular, positive real
// diagonal; Rinv = R^-1.  status[0] = 1 on a NaN pivot.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(GT) k_chol_small(const double2* __restrict__ G, int q, double2* Rout,
                                                   double2* RinvOut, int* status) {
  extern __shared__ __align__(16) double2 chol_sm[];
  auto S = reinterpret_cast<double2(*)[BQ + 1]>(chol_sm);                  // G, becoming R (upper)
  auto X = reinterpret_cast<double2(*)[BQ + 1]>(chol_sm + BQ * (BQ + 1));  // R^-1
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < q * q; e += GT) S[e / q][e % q] = G[e];
  __syncthreads();
  // right-looking Cholesky, upper: for each k, R[k][k] = sqrt(S[k][k]), R[k][j] = S[k][j] / R[k][k],
  // then S[i][j] -= conj(R[k][i]) R[k][j] for k < i <= j.  A negligible pivot (a column that is
  // zero or dependent on the previous ones: an all-zero right-hand side, a converged direction)
  // deflates: R row k = 0, and the inverse is taken of R with a unit pivot there, so that column
  // of Q = W R^-1 is the (zero) remainder of W — the oracle's Householder QR gives R[k][k] = 0 too.
  __shared__ double thr;
  __shared__ unsigned char defl[BQ];
  if (tid == 0) {
    double mx = 0.0;
    for (int k = 0; k < q; ++k) mx = fmax(mx, S[k][k].x);
    thr = 1e-28 * mx;
  }
  __syncthreads();
  // One barrier per step: row k is scaled into R (a separate array) while the trailing update
  // reads the unscaled row (S[i][j] -= conj(S[k][i]) S[k][j] / d^2), so no thread writes what
  // another reads within a step; 1/d from one reciprocal square root (no per-element divides).
  auto Rm = reinterpret_cast<double2(*)[BQ + 1]>(chol_sm + 2 * BQ * (BQ + 1));
  for (int k = 0; k < q; ++k) {
    const double d2 = S[k][k].x;
    if (tid == 0 && !(d2 == d2)) bad = 1;  // NaN
    const bool dk = !(d2 > thr);
    const double inv_d = dk ? 1.0 : rsqrt(d2);
    const double inv_d2 = inv_d * inv_d;
    if (tid == 0) defl[k] = dk;
    for (int j = tid; j < q; j += GT) {
      const double2 v = S[k][j];
      Rm[k][j] = j < k ? make_double2(0.0, 0.0)
                 : dk  ? make_double2(j == k ? 1.0 : 0.0, 0.0)
                       : (j == k ? make_double2(d2 * inv_d, 0.0) : make_double2(v.x * inv_d, v.y * inv_d));
    }
    // trailing update on a 16 x 16 thread grid (no integer division per element)
    if (!dk)
      for (int i = k + 1 + (tid >> 4); i < q; i += 16) {
        const double2 a = S[k][i];
        for (int j = i + ((tid & 15) - i % 16 + 16) % 16; j < q; j += 16) {
          const double2 b = S[k][j];
          // S[i][j] -= conj(a) b / d^2
          S[i][j].x -= (a.x * b.x + a.y * b.y) * inv_d2;
          S[i][j].y -= (a.x * b.y - a.y * b.x) * inv_d2;
        }
      }
    __syncthreads();
  }
  // X = R^-1 by Gauss-Jordan from the last row up, one barrier per step: rows r < i take
  // X[r] -= (R[r][i] / R[i][i]) X[i] with row i left unscaled until the end (row i is not
  // written in its own step)
  for (int e = tid; e < q * q; e += GT) {
    const int i = e / q, j = e % q;
    X[i][j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int i = q - 1; i >= 0; --i) {
    const double irr = 1.0 / Rm[i][i].x;  // 1 for a deflated pivot
    for (int r = tid >> 4; r < i; r += 16) {
      const double2 f0 = Rm[r][i];
      const double2 f = make_double2(f0.x * irr, f0.y * irr);
      for (int c = i + (tid & 15); c < q; c += 16) {
        const double2 x = X[i][c];
        X[r][c].x -= f.x * x.x - f.y * x.y;
        X[r][c].y -= f.x * x.y + f.y * x.x;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < q * q; e += GT) {
    const int i = e / q;
    const double irr = 1.0 / Rm[i][i].x;
    X[i][e % q] = make_double2(X[i][e % q].x * irr, X[i][e % q].y * irr);
  }
  __syncthreads();
  for (int e = tid; e < q * q; e += GT) {
    const int i = e / q, j = e % q;
    Rout[e] = defl[i] ? make_double2(0.0, 0.0) : Rm[i][j];  // deflated rows of R are zero
    RinvOut[e] = X[i][j];
  }
  if (tid == 0 && bad && status) status[0] = 1;
}

// the step's record from the column residuals: rec = {max_c colres[c], status}
__global__ void k_bres(const double* __restrict__ colres, int q, const int* status, double2* rec, int slot) {
  double mx = 0.0;
  for (int c = threadIdx.x; c < q; c += 32) mx = fmax(mx, colres[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (threadIdx.x == 0) {
    rec[slot] = make_double2(mx, status ? (double)status[0] : 0.0);
    __threadfence_system();
  }
}

// column norms of a rows x q block (relative to bn): out[c] = ||A_c|| / bn_c
__global__ void k_colnorm(const double2* __restrict__ Am, int64_t rows, int q, const double* bn, double* out) {
  __shared__ double red[GT];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += GT) {
    const double2 v = Am[r * q + c];
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = GT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = sqrt(red[0]) / (bn ? bn[c] : 1.0);
}

__global__ void k_add_inplace(double2* a, const double2* b, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    a[e] = cadd(a[e], b[e]);
}

__global__ void k_sub2(const double2* a, const double2* b, double2* out, int64_t n) {  // out = a - b
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = make_double2(a[e].x - b[e].x, a[e].y - b[e].y);
}

// ------------------------------------------------------------------------------------------------
// host-side composition
// ------------------------------------------------------------------------------------------------
struct Bk {
  cudaStream_t st;
  int q;
  double2* part;     // gram partials
  int64_t part_cap;  // elements
  int sms;

  // C (nblk q x q) (+)= Σ_blk A_blk^H B over `rows` rows
  int gram(const double2* A, int64_t astride, int nblk, const double2* B, int64_t rows, double2* C,
           bool accumulate) {
    int nchunk = std::max(1, (2 * sms) / std::max(1, nblk));
    const int64_t min_rows = 4 * KR;
    nchunk = (int)std::min<int64_t>(nchunk, std::max<int64_t>(1, rows / min_rows));
    while ((int64_t)nblk * nchunk * q * q > part_cap && nchunk > 1) --nchunk;
    if ((int64_t)nblk * nchunk * q * q > part_cap) {
      h2b_set_error("h2b_block_gmres: gram scratch too small");
      return H2B_EINVAL;
    }
    const int64_t chunk = ((rows + nchunk - 1) / nchunk + KR - 1) / KR * KR;
    nchunk = (int)((rows + chunk - 1) / chunk);
    k_bgram<<<dim3(nchunk, nblk), GT, 0, st>>>(A, astride, B, rows, q, chunk, nchunk, part);
    H2B_CHECK_LAUNCH();
    const int64_t tot = (int64_t)nblk * q * q;
    k_breduce<<<(int)std::min<int64_t>((tot + 255) / 256, 4 * sms), 256, 0, st>>>(part, nblk, nchunk, q, C,
                                                                                   accumulate ? 1 : 0);
    H2B_CHECK_LAUNCH();
    return H2B_OK;
  }
  // Out = beta In + alpha Σ_blk A_blk C_blk
  int update(const double2* A, int64_t astride, int nblk, const double2* C, const double2* In, double2* Out,
             int64_t rows, double alpha, double beta) {
    if (nblk <= 0) return H2B_OK;
    k_bupdate<<<(int)((rows + MROWS - 1) / MROWS), GT, 0, st>>>(A, astride, nblk, C, In, Out, rows, q, alpha, beta);
    H2B_CHECK_LAUNCH();
    return H2B_OK;
  }
  // CholQR2 of W (rows x q) -> Q (rows x q), R = R2 R1 (q x q) and, when Rinv is given,
  // R^-1 = R1^-1 R2^-1; T is scratch (rows x q); G, R1, R1i, R2, R2i scratch q x q
  int cholqr2(const double2* W, double2* Q, double2* T, int64_t rows, double2* R, double2* Rinv, double2* G,
              double2* R1, double2* R1i, double2* R2, double2* R2i, int* status) {
    H2B_TRY(gram(W, 0, 1, W, rows, G, false));
    k_chol_small<<<1, GT, CHOL_SMEM, st>>>(G, q, R1, R1i, status);
    H2B_CHECK_LAUNCH();
    H2B_TRY(update(W, 0, 1, R1i, nullptr, T, rows, 1.0, 0.0));  // T = W R1^-1
    H2B_TRY(gram(T, 0, 1, T, rows, G, false));
    k_chol_small<<<1, GT, CHOL_SMEM, st>>>(G, q, R2, R2i, status);
    H2B_CHECK_LAUNCH();
    H2B_TRY(update(T, 0, 1, R2i, nullptr, Q, rows, 1.0, 0.0));  // Q = T R2^-1
    H2B_TRY(update(R2, 0, 1, R1, nullptr, R, q, 1.0, 0.0));     // R = R2 R1
    if (Rinv) H2B_TRY(update(R1i, 0, 1, R2i, nullptr, Rinv, q, 1.0, 0.0));
    return H2B_OK;
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// =================================================================================================
// h2b_block_gmres: B_perm, X_perm are N x q row-major complex128 device arrays (permuted order)
// =================================================================================================
extern "C" int h2b_block_gmres(h2b_handle h, const void* B_perm, void* X_perm, int q, int restart, double tol,
                               int max_iter, double* history, h2b_report* report, void* stream) {
  if (!h || !B_perm || !X_perm || !report) {
    h2b_set_error("h2b_block_gmres: null argument");
    return H2B_EINVAL;
  }
  if (!(tol > 0.0 && tol < 1.0) || max_iter < 1 || restart < 1 || q < 1 || q > BQ) {
    h2b_set_error("h2b_block_gmres: need 0 < tol < 1, max_iter >= 1, restart >= 1, 1 <= q <= 64");
    return H2B_EINVAL;
  }
  const double t0 = now_s();
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  H2B_TRY(h2b_order_begin(h, st));
  struct OrderEnd {
    h2b_ctx* h;
    cudaStream_t st;
    ~OrderEnd() { h2b_order_end(h, st); }
  } order_end{h, st};
  const int64_t n = h->n;
  const int m = restart;
  const int64_t L = (int64_t)(m + 1) * q;  // rows of the small space
  const int64_t nq = n * q, qq = (int64_t)q * q;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  const int64_t part_cap = (int64_t)std::max(2 * sms, m + 2) * qq + (int64_t)(m + 1) * qq;
  // workspace layout (complex128 elements)
  const int64_t sz_V = (int64_t)(m + 1) * nq;  // basis blocks V_0..V_m
  const int64_t sz_big = 3 * nq;               // W, T, R (residual / scratch)
  const int64_t sz_Qs = (int64_t)m * L * q;    // small-space orthonormal blocks
  const int64_t sz_small = 3 * L * q;          // hcol, hs scratch, Eres
  const int64_t sz_C = 2 * (int64_t)(m + 1) * qq;     // CGS coefficients (two passes)
  const int64_t sz_Rs = (int64_t)m * m * qq;          // block upper triangular Rs (m x m grid)
  const int64_t sz_Rsi = (int64_t)m * qq;             // inverses of its diagonal blocks
  const int64_t sz_Z = (int64_t)m * qq;               // Qs^H E0 blocks, then Y
  const int64_t sz_qq = 12 * qq;                      // G, R1, R1i, R, Rinv, R0, ...
  const int64_t tot = sz_V + sz_big + sz_Qs + sz_small + sz_C + sz_Rs + sz_Rsi + sz_Z + sz_qq + part_cap + 2 * q + 64;
  double2* ws = nullptr;
  H2B_TRY(h2b_krylov_workspace(h, sizeof(double2) * (size_t)tot, &ws));
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize, CHOL_SMEM));
  double2* V = ws;
  double2* W = V + sz_V;
  double2* T = W + nq;
  double2* Rr = T + nq;
  double2* Qs = Rr + nq;
  double2* hcol = Qs + sz_Qs;
  double2* hs = hcol + L * q;
  double2* Eres = hs + L * q;
  double2* C1 = Eres + L * q;
  double2* C2 = C1 + (int64_t)(m + 1) * qq;
  double2* Rs = C2 + (int64_t)(m + 1) * qq;
  double2* Rsi = Rs + sz_Rs;
  double2* Z = Rsi + sz_Rsi;
  double2* G = Z + sz_Z;
  double2* R1 = G + qq;
  double2* R1i = R1 + qq;
  double2* Rq = R1i + qq;   // R of the current CholQR2
  double2* Rqi = Rq + qq;
  double2* R0 = Rqi + qq;
  double2* R2 = R0 + qq;    // CholQR2 scratch (second pass)
  double2* R2i = R2 + qq;
  double2* part = G + sz_qq;
  double* bn = reinterpret_cast<double*>(part + part_cap);
  double* colres = bn + q;
  int* status = reinterpret_cast<int*>(colres + q);
  Bk bk{st, q, part, part_cap, sms};
  const double2* Bm = (const double2*)B_perm;
  double2* X = (double2*)X_perm;
  // pinned, mapped records: one {max residual, status} per step (two rows of m), the column norms
  static thread_local double2* rec_h = nullptr;
  static thread_local int rec_cap = 0;
  if (rec_cap < 2 * m + 2 * BQ) {
    if (rec_h) cudaFreeHost(rec_h);
    H2B_CUDA_TRY(cudaHostAlloc(&rec_h, sizeof(double2) * (2 * m + 2 * BQ),
                               cudaHostAllocMapped | cudaHostAllocPortable));
    rec_cap = 2 * m + 2 * BQ;
  }
  double2* rec_d = nullptr;
  H2B_CUDA_TRY(cudaHostGetDevicePointer((void**)&rec_d, rec_h, 0));
  double* cn_h = reinterpret_cast<double*>(rec_h + 2 * m);  // q column norms
  double* cn_d = reinterpret_cast<double*>(rec_d + 2 * m);

  *report = h2b_report{0, 0, 0, 0, 0.0};
  H2B_CUDA_TRY(cudaMemsetAsync(X, 0, sizeof(double2) * nq, st));
  // ||b_c||: zero columns count as 1 (oracle: bn = where(bn == 0, 1, bn))
  k_colnorm<<<q, GT, 0, st>>>(Bm, n, q, nullptr, cn_d);
  H2B_CHECK_LAUNCH();
  H2B_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<double> bnh(q);
  bool all_zero = true;
  for (int c = 0; c < q; ++c) {
    bnh[c] = cn_h[c] == 0.0 ? 1.0 : cn_h[c];
    all_zero &= cn_h[c] == 0.0;
  }
  if (all_zero) {
    report->converged = 1;
    report->wall_time = now_s() - t0;
    return H2B_OK;
  }
  H2B_CUDA_TRY(cudaMemcpyAsync(bn, bnh.data(), sizeof(double) * q, cudaMemcpyHostToDevice, st));
  H2B_CUDA_TRY(cudaMemcpyAsync(Rr, Bm, sizeof(double2) * nq, cudaMemcpyDeviceToDevice, st));
  H2B_TRY(h2b_prepare(h));
  H2B_TRY(h2b_ensure_workspace(h, q));

  cudaEvent_t ev[2];
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
  } guard{ev};

  // one block Arnoldi step j (everything after is queued asynchronously)
  auto step = [&](int j) -> int {
    double2* Vj = V + (int64_t)j * nq;
    double2* Vn = V + (int64_t)(j + 1) * nq;
    H2B_TRY(h2b_run_matvec(h, Vj, W, q, st));
    // block CGS2 against V_0..V_j: Hc = C1 + C2
    H2B_TRY(bk.gram(V, nq, j + 1, W, n, C1, false));
    H2B_TRY(bk.update(V, nq, j + 1, C1, W, W, n, -1.0, 1.0));
    H2B_TRY(bk.gram(V, nq, j + 1, W, n, C2, false));
    H2B_TRY(bk.update(V, nq, j + 1, C2, W, W, n, -1.0, 1.0));
    // V_{j+1} R_j = W (CholQR2)
    H2B_TRY(bk.cholqr2(W, Vn, T, n, Rq, nullptr, G, R1, R1i, R2, R2i, status));
    // the new block column of H in the small space: hcol = [C1 + C2 ; R_j ; 0]
    H2B_CUDA_TRY(cudaMemsetAsync(hcol, 0, sizeof(double2) * L * q, st));
    H2B_CUDA_TRY(cudaMemcpyAsync(hcol, C1, sizeof(double2) * (j + 1) * qq, cudaMemcpyDeviceToDevice, st));
    {  // hcol[0:(j+1)q] += C2
      const int64_t e = (int64_t)(j + 1) * qq;
      k_add_inplace<<<(int)std::min<int64_t>((e + 255) / 256, 4 * sms), 256, 0, st>>>(hcol, C2, e);
      H2B_CHECK_LAUNCH();
    }
    H2B_CUDA_TRY(cudaMemcpyAsync(hcol + (int64_t)(j + 1) * qq, Rq, sizeof(double2) * qq, cudaMemcpyDeviceToDevice, st));
    // small space: block CGS2 of hcol against Qs_0..Qs_{j-1}, then CholQR2 -> Qs_j, Rs_jj
    double2* Rcol = Rs + (int64_t)j * m * qq;  // block column j of Rs: blocks i = 0..j (i*qq)
    if (j > 0) {
      H2B_TRY(bk.gram(Qs, L * q, j, hcol, L, Rcol, false));
      H2B_TRY(bk.update(Qs, L * q, j, Rcol, hcol, hcol, L, -1.0, 1.0));
      H2B_TRY(bk.gram(Qs, L * q, j, hcol, L, C2, false));
      H2B_TRY(bk.update(Qs, L * q, j, C2, hcol, hcol, L, -1.0, 1.0));
      k_add_inplace<<<(int)std::min<int64_t>((j * qq + 255) / 256, 4 * sms), 256, 0, st>>>(Rcol, C2, (int64_t)j * qq);
      H2B_CHECK_LAUNCH();
    }
    double2* Qsj = Qs + (int64_t)j * L * q;
    H2B_TRY(bk.cholqr2(hcol, Qsj, hs, L, Rcol + (int64_t)j * qq, Rsi + (int64_t)j * qq, G, R1, R1i, R2, R2i,
                       status));
    // Z_j = Qs_j^H E0 = Qs_j[0:q]^H R0 ; Eres -= Qs_j Z_j
    H2B_TRY(bk.gram(Qsj, 0, 1, R0, q, Z + (int64_t)j * qq, false));
    H2B_TRY(bk.update(Qsj, 0, 1, Z + (int64_t)j * qq, Eres, Eres, L, -1.0, 1.0));
    k_colnorm<<<q, GT, 0, st>>>(Eres, L, q, bn, colres);
    H2B_CHECK_LAUNCH();
    k_bres<<<1, 32, 0, st>>>(colres, q, status, rec_d, j);
    H2B_CHECK_LAUNCH();
    return H2B_OK;
  };

  int it = 0, nh = 0, matvecs = 0;
  bool converged = false;
  while (it < max_iter) {
    // V_0 R0 = R (CholQR2); Eres = [R0; 0]
    H2B_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), st));
    H2B_TRY(bk.cholqr2(Rr, V, T, n, R0, nullptr, G, R1, R1i, R2, R2i, status));
    H2B_CUDA_TRY(cudaMemsetAsync(Eres, 0, sizeof(double2) * L * q, st));
    H2B_CUDA_TRY(cudaMemcpyAsync(Eres, R0, sizeof(double2) * qq, cudaMemcpyDeviceToDevice, st));
    // steps run one ahead of the host's check (a speculative step writes only V_{j+2}, the
    // small-space block j+1, Z_{j+1} and Eres — Eres is not used by the back substitution)
    const int it0 = it;
    int j_done = 0;
    H2B_TRY(step(0));
    ++matvecs;
    H2B_CUDA_TRY(cudaEventRecord(ev[0], st));
    for (int j = 0; j < m; ++j) {
      if (j + 1 < m && it0 + j + 1 < max_iter) {
        H2B_TRY(step(j + 1));
        ++matvecs;
        H2B_CUDA_TRY(cudaEventRecord(ev[(j + 1) & 1], st));
      }
      H2B_CUDA_TRY(cudaEventSynchronize(ev[j & 1]));
      ++it;
      const double res = rec_h[j].x;
      const int bad = rec_h[j].y != 0.0;
      if (history && nh < max_iter) history[nh] = res;
      ++nh;
      j_done = j + 1;
      if (res <= tol || it >= max_iter || bad) break;
    }
    // Y = Rs^-1 Z by block back substitution (Z overwritten), then X += V Y
    for (int i = j_done - 1; i >= 0; --i) {
      // Y_i = Rs_ii^-1 Z_i (into C1 block i), then Z_{0..i-1} -= Rs_{0..i-1, i} Y_i
      H2B_TRY(bk.update(Rsi + (int64_t)i * qq, 0, 1, Z + (int64_t)i * qq, nullptr, C1 + (int64_t)i * qq, q, 1.0, 0.0));
      if (i > 0)
        H2B_TRY(bk.update(Rs + (int64_t)i * m * qq, 0, 1, C1 + (int64_t)i * qq, Z, Z, (int64_t)i * q, -1.0, 1.0));
    }
    // X += Σ_i V_i Y_i — Y_i is a q x q block: V (n x q blocks) times the stacked Y
    H2B_TRY(bk.update(V, nq, j_done, C1, X, X, n, 1.0, 1.0));
    // true residual R = B - A X, column norms relative to ||b_c||
    H2B_TRY(h2b_run_matvec(h, X, T, q, st));
    ++matvecs;
    {
      k_sub2<<<(int)std::min<int64_t>((nq + 255) / 256, 8 * sms), 256, 0, st>>>(Bm, T, Rr, nq);
      H2B_CHECK_LAUNCH();
    }
    k_colnorm<<<q, GT, 0, st>>>(Rr, n, q, bn, cn_d);
    H2B_CHECK_LAUNCH();
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    double mx = 0.0;
    for (int c = 0; c < q; ++c) mx = std::max(mx, cn_h[c]);
    if (mx <= tol) {
      converged = true;
      break;
    }
  }
  report->iterations = it;
  report->converged = converged ? 1 : 0;
  report->n_history = nh < max_iter ? nh : max_iter;
  report->matvecs = matvecs;
  report->wall_time = now_s() - t0;
  return H2B_OK;
}

