// Stage II of the H² builder on the device (first step): nested cluster bases,
// transfer matrices and couplings from the Stage-I grouped factors.
//
// Restates the reference's build_bases / build_coupling (/root/reference/pkg/src/h2vie/
// build.py:228-309) with linalg.trunc_eig_hermitian (linalg.py:207-231):
//   * cluster c's Gram matrix G_c = Σ_j X_j M_j X_j^H over the Stage-I factors j of c and of its
//     ancestors (build.py:_gram_terms), X_j = A_j restricted to c's rows for a leaf, and the
//     children-projected [V_lo^H A_j|lo ; V_hi^H A_j|hi] for a non-leaf (basis.apply_vh), M_j =
//     B_j^T conj(B_j); G_c <- (G_c + G_c^H) / 2;
//   * its accuracy-truncated eigendecomposition: the k leading eigenvectors with
//     sqrt(lambda / lambda_1) > eps_acc — the leaf basis V_c, or the transfers [T_lo; T_hi];
//   * couplings S_{t,s} = (V_t^H A_t)(V_s^H B_t|s)^T (build.py:build_coupling).
// The Hermitian eigenproblem is a parallel cyclic Jacobi in one CTA (tournament ordering: all
// m/2 rotations of a round at once; complex rotations reduced to real ones by a phase),
// matrix and eigenvectors in shared memory (m <= 80).  The flattened bases V_c (n_c x k_c,
// V_c = [V_lo T_lo ; V_hi T_hi]) are kept in HBM, so every projection is one small product.
// Eigenvectors are unique only up to phase (and rotations inside degenerate eigenspaces), so the
// bases differ from the reference's by unitary factors; the operator V_t S V_s^T is the same up
// to the truncation tolerance, which is what the tests check (dense operator, reference matvec).
#include <math.h>

#include <algorithm>
#include <vector>

#include "h2b_common.cuh"

namespace {

constexpr int BT = 256;     // threads per builder CTA
constexpr int JMAX = 80;    // largest Gram matrix (leaf size or k_lo + k_hi)
constexpr int JSMEM = 2 * JMAX * (JMAX + 1) * 16 + 8 * JMAX * 16;

constexpr int JBIG = 256;   // largest Gram matrix at all (beyond JMAX: G and eigenvectors in HBM)

struct Mat {               // a matrix in shared or global memory, row stride ld
  double2* p;
  int ld;
  __device__ __forceinline__ double2& operator()(int i, int j) const { return p[(int64_t)i * ld + j]; }
};

struct BTerm {             // one Stage-I factor feeding a cluster's Gram matrix
  int64_t a_off;           // element offset of A_j's first row restricted to the cluster
  int64_t m_off;           // element offset of M_j = B_j^T conj(B_j) (r x r)
  int32_t r, pad;          // rank of the factor
};
struct BClu {              // one cluster of a level step
  int32_t c, m, n, leaf;   // packed index, Gram size, points, leaf flag
  int32_t t_first, nt;     // terms
  int32_t lo, hi;          // children (packed) or -1
  int32_t klo, khi, pad0, pad1;
  int64_t x_off;           // scratch (m x rmax) for X and Y
  int64_t out_off;         // result slot (m x m): eigenvectors, sorted, leading k columns used
  int64_t j_off;           // m > JMAX: G and the eigenvectors in HBM (2 m^2 elements), else -1
};

// G (m x m) in smem <- Σ_terms X M X^H, X computed into global scratch
__device__ void gram(const BClu& C, const BTerm* terms, const double2* __restrict__ A, const double2* __restrict__ Mb,
                     const double2* __restrict__ Vf, const int64_t* __restrict__ vf_off, const int32_t* c_size,
                     double2* scratch, Mat G) {
  const int tid = threadIdx.x, m = C.m;
  for (int e = tid; e < m * m; e += BT) G(e / m, e % m) = make_double2(0.0, 0.0);
  __syncthreads();
  for (int ti = 0; ti < C.nt; ++ti) {
    const BTerm T = terms[C.t_first + ti];
    const int r = T.r;
    const double2* Aj = A + T.a_off;  // rows of the cluster, r columns (row-major, ld r)
    double2* X = scratch + C.x_off;     // m x r
    double2* Y = X + (int64_t)m * r;    // m x r
    if (C.leaf) {
      for (int e = tid; e < m * r; e += BT) X[e] = Aj[e];
    } else {
      // X = [Vf_lo^H A|lo ; Vf_hi^H A|hi]
      const int nlo = c_size[C.lo];
      for (int e = tid; e < m * r; e += BT) {
        const int i = e / r, j = e % r;
        const bool lo = i < C.klo;
        const int ch = lo ? C.lo : C.hi, ii = lo ? i : i - C.klo, kk = lo ? C.klo : C.khi;
        const int nch = c_size[ch], r0 = lo ? 0 : nlo;
        const double2* V = Vf + vf_off[ch];  // nch x kk
        double2 s = make_double2(0.0, 0.0);
        for (int p = 0; p < nch; ++p) cfma_conj(s, V[(int64_t)p * kk + ii], Aj[(int64_t)(r0 + p) * r + j]);
        X[e] = s;
      }
    }
    __syncthreads();
    // Y = X M
    const double2* Mj = Mb + T.m_off;
    for (int e = tid; e < m * r; e += BT) {
      const int i = e / r, j = e % r;
      double2 s = make_double2(0.0, 0.0);
      for (int l = 0; l < r; ++l) cfma(s, X[(int64_t)i * r + l], Mj[(int64_t)l * r + j]);
      Y[e] = s;
    }
    __syncthreads();
    // G += Y X^H
    for (int e = tid; e < m * m; e += BT) {
      const int i = e / m, j = e % m;
      double2 s = make_double2(0.0, 0.0);
      for (int l = 0; l < r; ++l) cfma_conj(s, X[(int64_t)j * r + l], Y[(int64_t)i * r + l]);  // Y[i,l] conj(X[j,l])
      G(i, j) = cadd(G(i, j), s);
    }
    __syncthreads();
  }
  // symmetrise: G <- (G + G^H) / 2
  for (int e = tid; e < m * m; e += BT) {
    const int i = e / m, j = e % m;
    if (i < j) {
      const double2 a = G(i, j), b = G(j, i);
      const double2 h = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      G(i, j) = h;
      G(j, i) = make_double2(h.x, -h.y);
    } else if (i == j) {
      G(i, i).y = 0.0;
    }
  }
  __syncthreads();
}

// one level step: Gram, Jacobi eigendecomposition, sorted eigenvectors and rank
__global__ void __launch_bounds__(BT, 1) k_stage2_level(const BClu* __restrict__ clus, const BTerm* __restrict__ terms,
                                                        const double2* __restrict__ A, const double2* __restrict__ Mb,
                                                        const double2* __restrict__ Vf, const int64_t* __restrict__ vf_off,
                                                        const int32_t* __restrict__ c_size, double2* scratch,
                                                        double2* out, int32_t* rank_out, double eps_acc,
                                                        double2* jwork) {
  extern __shared__ __align__(16) double2 bsm[];
  __shared__ double2 rot[JBIG];  // per pair: {c, s}, {e^{-i phi}}
  __shared__ int pp[JBIG / 2], qq[JBIG / 2];
  __shared__ double lam[JBIG];
  __shared__ int order[JBIG];
  __shared__ double offn, totn;
  const BClu C = clus[blockIdx.x];
  const int tid = threadIdx.x, m = C.m;
  // G and its eigenvectors E: shared memory up to JMAX, else this cluster's HBM slot
  const Mat G = C.j_off < 0 ? Mat{bsm, JMAX + 1} : Mat{jwork + C.j_off, m};
  const Mat E = C.j_off < 0 ? Mat{bsm + JMAX * (JMAX + 1), JMAX + 1} : Mat{jwork + C.j_off + (int64_t)m * m, m};
  if (C.nt == 0 || m == 0) {
    if (tid == 0) rank_out[C.c] = 0;
    return;
  }
  gram(C, terms, A, Mb, Vf, vf_off, c_size, scratch, G);
  for (int e = tid; e < m * m; e += BT) E(e / m, e % m) = make_double2(e / m == e % m ? 1.0 : 0.0, 0.0);
  const int me = m + (m & 1);  // even tournament size (a dummy index pairs with the odd one out)
  __syncthreads();
  for (int sweep = 0; sweep < 30; ++sweep) {
    // convergence: off-diagonal norm vs total
    if (tid == 0) {
      offn = 0.0;
      totn = 0.0;
    }
    __syncthreads();
    double o = 0.0, t = 0.0;
    for (int e = tid; e < m * m; e += BT) {
      const double2 v = G(e / m, e % m);
      const double a2 = v.x * v.x + v.y * v.y;
      t += a2;
      if (e / m != e % m) o += a2;
    }
    atomicAdd(&offn, o);
    atomicAdd(&totn, t);
    __syncthreads();
    if (!(offn > 1e-32 * totn)) break;
    for (int round = 0; round < me - 1; ++round) {
      // tournament pairs: position 0 fixed, the others rotate
      if (tid < me / 2) {
        auto at = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (me - 1); };
        int p = at(tid), q = at(me - 1 - tid);
        if (p > q) { const int w = p; p = q; q = w; }
        pp[tid] = p;
        qq[tid] = q;
        double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
        if (q < m) {
          const double2 b = G(p, q);
          const double ab = hypot(b.x, b.y);
          if (ab > 1e-300) {
            const double a = G(p, p).x, d = G(q, q).x;
            const double tau = (d - a) / (2.0 * ab);
            const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = tt * c;
            er = b.x / ab;   // e^{-i phi} = conj(b) / |b|
            ei = -b.y / ab;
          }
        }
        rot[2 * tid] = make_double2(c, s);
        rot[2 * tid + 1] = make_double2(er, ei);
      }
      __syncthreads();
      // columns: G <- G J, E <- E J with J = [[c, s], [-s e, c e]], e = e^{-i phi}
      for (int w = tid; w < (me / 2) * m; w += BT) {
        const int i = w / m, r = w % m;
        const int p = pp[i], q = qq[i];
        if (q >= m) continue;
        const double c = rot[2 * i].x, s = rot[2 * i].y;
        const double2 e = rot[2 * i + 1];
        const double2 j10 = make_double2(-s * e.x, -s * e.y), j11 = make_double2(c * e.x, c * e.y);
#pragma unroll
        for (int mat = 0; mat < 2; ++mat) {
          const Mat Mx = mat == 0 ? G : E;
          const double2 gp = Mx(r, p), gq = Mx(r, q);
          double2 np_ = make_double2(c * gp.x, c * gp.y), nq = make_double2(s * gp.x, s * gp.y);
          cfma(np_, gq, j10);
          cfma(nq, gq, j11);
          Mx(r, p) = np_;
          Mx(r, q) = nq;
        }
      }
      __syncthreads();
      // rows: G <- J^H G
      for (int w = tid; w < (me / 2) * m; w += BT) {
        const int i = w / m, col = w % m;
        const int p = pp[i], q = qq[i];
        if (q >= m) continue;
        const double c = rot[2 * i].x, s = rot[2 * i].y;
        const double2 e = rot[2 * i + 1];
        const double2 cj10 = make_double2(-s * e.x, s * e.y), cj11 = make_double2(c * e.x, -c * e.y);  // conj
        const double2 gp = G(p, col), gq = G(q, col);
        double2 np_ = make_double2(c * gp.x, c * gp.y), nq = make_double2(s * gp.x, s * gp.y);
        cfma(np_, cj10, gq);
        cfma(nq, cj11, gq);
        G(p, col) = np_;
        G(q, col) = nq;
      }
      __syncthreads();
    }
  }
  // eigenvalues, descending order, truncation rank
  for (int i = tid; i < m; i += BT) lam[i] = fmax(G(i, i).x, 0.0);
  __syncthreads();
  for (int i = tid; i < m; i += BT) {
    int rk = 0;
    for (int j = 0; j < m; ++j) rk += (lam[j] > lam[i]) || (lam[j] == lam[i] && j < i);
    order[rk] = i;
  }
  __syncthreads();
  __shared__ int s_k;
  if (tid == 0) {
    const double l1 = lam[order[0]];
    int k = 0;
    if (l1 > 0.0)
      for (int i = 0; i < m; ++i) k += sqrt(lam[order[i]] / l1) > eps_acc;
    s_k = k;
    rank_out[C.c] = k;
  }
  __syncthreads();
  // the leading k eigenvectors, row-major m x k
  const int k = s_k;
  double2* o = out + C.out_off;
  for (int e = tid; e < m * k; e += BT) o[e] = E(e / k, order[e % k]);
}

// flattened bases of one level: leaf V_c = p; non-leaf V_c = [Vf_lo T_lo ; Vf_hi T_hi]
__global__ void k_stage2_flatten(const BClu* __restrict__ clus, const double2* __restrict__ out,
                                 const int32_t* __restrict__ rank, const int32_t* __restrict__ c_size,
                                 double2* Vf, const int64_t* __restrict__ vf_off) {
  const BClu C = clus[blockIdx.x];
  const int k = rank[C.c];
  if (k == 0 || C.nt == 0) return;
  const double2* p = out + C.out_off;  // m x k
  double2* V = Vf + vf_off[C.c];       // n x k
  if (C.leaf) {
    for (int e = threadIdx.x; e < C.n * k; e += blockDim.x) V[e] = p[e];
    return;
  }
  const int nlo = c_size[C.lo];
  for (int e = threadIdx.x; e < C.n * k; e += blockDim.x) {
    const int row = e / k, j = e % k;
    const bool lo = row < nlo;
    const int ch = lo ? C.lo : C.hi, kk = lo ? C.klo : C.khi, r0 = lo ? 0 : C.klo;
    const int rr = lo ? row : row - nlo;
    const double2* Vc = Vf + vf_off[ch];
    double2 s = make_double2(0.0, 0.0);
    for (int l = 0; l < kk; ++l) cfma(s, Vc[(int64_t)rr * kk + l], p[(int64_t)(r0 + l) * k + j]);
    V[e] = s;
  }
}

struct SBlk {               // one admissible block (t, s)
  int32_t t, s, kt, ks;
  int32_t r, nt_, ns, pad;
  int64_t p_off;            // P_t = Vf_t^H A_t (kt x r), shared by t's blocks
  int64_t b_off;            // B_t rows of s (n_s x r)
  int64_t out_off;          // S (kt x ks)
};
struct PTgt {              // one target: P_t = Vf_t^H A_t
  int32_t t, kt, r, nt_;
  int64_t a_off, p_off;
};

// P_t = Vf_t^H A_t (kt x r) for every target with couplings
__global__ void k_stage2_proj(const PTgt* __restrict__ tg, const double2* __restrict__ A, const double2* __restrict__ Vf,
                              const int64_t* __restrict__ vf_off, double2* Pbuf) {
  const PTgt T = tg[blockIdx.x];
  const double2* Vt = Vf + vf_off[T.t];
  for (int e = threadIdx.x; e < T.kt * T.r; e += blockDim.x) {
    const int i = e / T.r, j = e % T.r;
    double2 s = make_double2(0.0, 0.0);
    for (int p = 0; p < T.nt_; ++p) cfma_conj(s, Vt[(int64_t)p * T.kt + i], A[T.a_off + (int64_t)p * T.r + j]);
    Pbuf[T.p_off + e] = s;
  }
}

// S = P_t (Vf_s^H B_t|s)^T, the inner dimension r in chunks of 32: Q chunk (ks x 32) in shared
// memory, S accumulated in global memory (each thread owns fixed elements)
constexpr int QCH = 8;
__global__ void k_stage2_couple(const SBlk* __restrict__ blks, const double2* __restrict__ Pbuf,
                                const double2* __restrict__ B, const double2* __restrict__ Vf,
                                const int64_t* __restrict__ vf_off, double2* S) {
  __shared__ double2 Q[JBIG * QCH];
  const SBlk b = blks[blockIdx.x];
  const int kt = b.kt, ks = b.ks, r = b.r;
  if (kt == 0 || ks == 0) return;
  const double2* Vs = Vf + vf_off[b.s];
  const double2* P = Pbuf + b.p_off;
  double2* So = S + b.out_off;
  for (int e = threadIdx.x; e < kt * ks; e += blockDim.x) So[e] = make_double2(0.0, 0.0);
  for (int l0 = 0; l0 < r; l0 += QCH) {
    const int lc = min(QCH, r - l0);
    __syncthreads();
    for (int e = threadIdx.x; e < ks * lc; e += blockDim.x) {
      const int j = e / lc, l = e % lc;
      double2 s = make_double2(0.0, 0.0);
      for (int p = 0; p < b.ns; ++p) cfma_conj(s, Vs[(int64_t)p * ks + j], B[b.b_off + (int64_t)p * r + l0 + l]);
      Q[j * QCH + l] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kt * ks; e += blockDim.x) {
      const int i = e / ks, j = e % ks;
      double2 s = So[e];
      for (int l = 0; l < lc; ++l) cfma(s, P[(int64_t)i * r + l0 + l], Q[j * QCH + l]);
      So[e] = s;
    }
  }
}

template <typename T>
int up(T** d, const T* h, size_t n) {  // h: host or device memory (unified addressing)
  H2B_CUDA_TRY(cudaMalloc((void**)d, sizeof(T) * std::max<size_t>(n, 1)));
  if (n) H2B_CUDA_TRY(cudaMemcpy(*d, h, sizeof(T) * n, cudaMemcpyDefault));
  return H2B_OK;
}

}  // namespace

struct h2b_builder_ctx {
  int P = 0, device = 0;
  std::vector<int32_t> rank;
  std::vector<int64_t> res_off;   // per cluster: result slot (V for leaves, T for non-leaves)
  std::vector<int64_t> s_off;     // per admissible block
  double2 *res = nullptr, *S = nullptr;
  std::vector<int32_t> m_of;      // Gram size per cluster
};

// Stage II on the device.  Inputs (host, packed order): the tree tables, the Stage-I factors
// (A_c, M_c = B_c^T conj(B_c), B_c with its partners' row offsets) and the admissible blocks in
// CSR by target (s_row_ptr / s_col).  Outputs stay on the device until fetched.
extern "C" int h2b_builder_create(int P, int depth, const int32_t* level_ptr, const int32_t* c_start,
                                  const int32_t* c_size, const int32_t* c_child_lo, const int32_t* c_child_hi,
                                  const int32_t* c_parent, const int32_t* s1_rank, const int64_t* s1_a_off,
                                  const void* s1_a, const int64_t* s1_m_off, const void* s1_m,
                                  const int64_t* s1_b_off, const void* s1_b, const int64_t* s1_part_ptr,
                                  const int32_t* s1_partner, const int64_t* s1_prow, const int64_t* s_row_ptr,
                                  const int32_t* s_col, double eps_acc, int device, void** out) {
  if (!level_ptr || !c_start || !c_size || !c_child_lo || !c_child_hi || !c_parent || !s1_rank || !out || P < 1) {
    h2b_set_error("h2b_builder_create: null argument");
    return H2B_EINVAL;
  }
  *out = nullptr;
  H2B_CUDA_TRY(cudaSetDevice(device));
  h2b_builder_ctx* B = new h2b_builder_ctx();
  B->P = P;
  B->device = device;
  B->rank.assign(P, 0);
  B->m_of.assign(P, 0);
  B->res_off.assign(P + 1, 0);
  // device copies of the Stage-I factors and tables
  const int64_t na = s1_a_off[P], nm = s1_m_off[P], nb = s1_b_off[P];
  double2 *dA = nullptr, *dM = nullptr, *dB = nullptr, *Vf = nullptr, *scratch = nullptr;
  int32_t *dsize = nullptr, *drank = nullptr;
  int64_t* dvf = nullptr;
  int rc = up(&dA, (const double2*)s1_a, (size_t)na);
  if (!rc) rc = up(&dM, (const double2*)s1_m, (size_t)nm);
  if (!rc) rc = up(&dB, (const double2*)s1_b, (size_t)nb);
  if (!rc) rc = up(&dsize, c_size, (size_t)P);
  if (!rc) rc = up(&drank, B->rank.data(), (size_t)P);
  std::vector<int64_t> vf_off(P + 1, 0);
  // flattened bases: sized per level as ranks become known (upper bound: n_c x m_c)
  int64_t vf_cap = 0;
  for (int p = 0; p < P; ++p) vf_cap += (int64_t)c_size[p] * std::min<int64_t>(c_size[p], JBIG);
  if (!rc) {
    const cudaError_t e = cudaMalloc(&Vf, sizeof(double2) * std::max<int64_t>(vf_cap, 1));
    if (e != cudaSuccess) rc = H2B_ENOMEM;
  }
  if (!rc) rc = up(&dvf, vf_off.data(), (size_t)P + 1);
  int64_t res_total = 0;
  if (!rc) H2B_CUDA_TRY(cudaFuncSetAttribute(k_stage2_level, cudaFuncAttributeMaxDynamicSharedMemorySize, JSMEM));
  // level by level, bottom-up
  int64_t vf_used = 0;
  std::vector<double2*> res_parts;
  for (int l = depth - 1; l >= 0 && !rc; --l) {
    std::vector<BClu> clus;
    std::vector<BTerm> terms;
    int64_t x_total = 0, o_total = 0, j_total = 0;
    double2* jwork = nullptr;
    for (int c = level_ptr[l]; c < level_ptr[l + 1]; ++c) {
      BClu C{};
      C.c = c;
      C.n = c_size[c];
      C.leaf = c_child_lo[c] < 0;
      C.lo = c_child_lo[c];
      C.hi = c_child_hi[c];
      C.klo = C.leaf ? 0 : B->rank[C.lo];
      C.khi = C.leaf ? 0 : B->rank[C.hi];
      C.m = C.leaf ? C.n : C.klo + C.khi;
      if (C.m > JBIG) {
        h2b_set_error("h2b_builder_create: a Gram matrix exceeds " + std::to_string(JBIG) +
                      " (leaf size or k_lo + k_hi): not supported by the device Stage II");
        rc = H2B_EINVAL;
        break;
      }
      C.j_off = -1;
      if (C.m > JMAX) {
        C.j_off = j_total;
        j_total += 2 * (int64_t)C.m * C.m;
      }
      C.t_first = (int)terms.size();
      int rmax = 0;
      for (int j = c; j >= 0; j = c_parent[j]) {  // the cluster itself, then its ancestors
        if (s1_rank[j] <= 0) continue;
        BTerm T{};
        T.r = s1_rank[j];
        T.a_off = s1_a_off[j] + (int64_t)(c_start[c] - c_start[j]) * T.r;
        T.m_off = s1_m_off[j];
        terms.push_back(T);
        rmax = std::max(rmax, T.r);
      }
      C.nt = (int)terms.size() - C.t_first;
      if (C.m == 0) C.nt = 0;
      C.x_off = x_total;
      x_total += 2 * (int64_t)C.m * rmax;
      C.out_off = o_total;
      o_total += (int64_t)C.m * C.m;
      B->m_of[c] = C.m;
      clus.push_back(C);
    }
    if (rc) break;
    BClu* dclus = nullptr;
    BTerm* dterms = nullptr;
    double2* res = nullptr;
    rc = up(&dclus, clus.data(), clus.size());
    if (!rc) rc = up(&dterms, terms.data(), terms.size());
    if (!rc) {
      cudaError_t e1 = cudaMalloc(&scratch, sizeof(double2) * std::max<int64_t>(x_total, 1));
      cudaError_t e2 = cudaMalloc(&res, sizeof(double2) * std::max<int64_t>(o_total, 1));
      cudaError_t e3 = cudaMalloc(&jwork, sizeof(double2) * std::max<int64_t>(j_total, 1));
      if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) rc = H2B_ENOMEM;
    }
    if (!rc) {
      k_stage2_level<<<(int)clus.size(), BT, JSMEM>>>(dclus, dterms, dA, dM, Vf, dvf, dsize, scratch, res, drank,
                                                      eps_acc, jwork);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        h2b_set_error(std::string("h2b_builder_create: level kernel: ") + cudaGetErrorString(e));
        rc = H2B_ECUDA;
      }
    }
    if (!rc) {
      H2B_CUDA_TRY(cudaMemcpy(B->rank.data(), drank, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
      for (const BClu& C : clus) {
        vf_off[C.c] = vf_used;
        vf_used += (int64_t)C.n * B->rank[C.c];
      }
      if (vf_used > vf_cap) {
        h2b_set_error("h2b_builder_create: flattened bases exceed their allocation");
        rc = H2B_EINVAL;
      }
    }
    if (!rc) {
      H2B_CUDA_TRY(cudaMemcpy(dvf, vf_off.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice));
      k_stage2_flatten<<<(int)clus.size(), 256>>>(dclus, res, drank, dsize, Vf, dvf);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        h2b_set_error(std::string("h2b_builder_create: flatten: ") + cudaGetErrorString(e));
        rc = H2B_ECUDA;
      }
    }
    // keep this level's results (eigenvector slots, m x m each) for the fetch
    if (!rc) {
      for (const BClu& C : clus) B->res_off[C.c] = res_total + C.out_off;
      res_total += o_total;
      res_parts.push_back(res);
    } else if (res) {
      cudaFree(res);
    }
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    if (jwork) cudaFree(jwork);
    if (dclus) cudaFree(dclus);
    if (dterms) cudaFree(dterms);
  }
  // gather the per-level result slots into one buffer (offsets in res_off)
  if (!rc) {
    H2B_CUDA_TRY(cudaMalloc(&B->res, sizeof(double2) * std::max<int64_t>(res_total, 1)));
    int64_t o = 0;
    int li = 0;
    for (int l = depth - 1; l >= 0 && li < (int)res_parts.size(); --l, ++li) {
      int64_t sz = 0;
      for (int c = level_ptr[l]; c < level_ptr[l + 1]; ++c) sz += (int64_t)B->m_of[c] * B->m_of[c];
      H2B_CUDA_TRY(cudaMemcpy(B->res + o, res_parts[li], sizeof(double2) * sz, cudaMemcpyDeviceToDevice));
      o += sz;
    }
  }
  for (double2* p : res_parts) cudaFree(p);
  // couplings: P_t once per target, then one CTA per block
  if (!rc) {
    std::vector<SBlk> blks;
    std::vector<PTgt> tgs;
    std::vector<int64_t> p_of(P, -1);
    int64_t ptot = 0;
    for (int t = 0; t < P; ++t) {
      if (s_row_ptr[t + 1] == s_row_ptr[t] || B->rank[t] == 0 || s1_rank[t] == 0) continue;
      PTgt T{t, B->rank[t], s1_rank[t], c_size[t], s1_a_off[t], ptot};
      p_of[t] = ptot;
      ptot += (int64_t)T.kt * T.r;
      tgs.push_back(T);
    }
    B->s_off.assign((size_t)s_row_ptr[P] + 1, 0);
    int64_t st = 0;
    for (int t = 0; t < P; ++t)
      for (int64_t b = s_row_ptr[t]; b < s_row_ptr[t + 1]; ++b) {
        const int s = s_col[b];
        SBlk K{};
        K.t = t;
        K.s = s;
        K.kt = B->rank[t];
        K.ks = B->rank[s];
        K.r = s1_rank[t];
        K.nt_ = c_size[t];
        K.ns = c_size[s];
        K.p_off = std::max<int64_t>(p_of[t], 0);
        int64_t prow = -1;
        for (int64_t j = s1_part_ptr[t]; j < s1_part_ptr[t + 1]; ++j)
          if (s1_partner[j] == s) prow = s1_prow[j];
        if (prow < 0 && K.kt > 0 && K.ks > 0 && K.r > 0) {
          h2b_set_error("h2b_builder_create: admissible block without its Stage-I partner");
          rc = H2B_EINVAL;
        }
        K.b_off = s1_b_off[t] + std::max<int64_t>(prow, 0) * K.r;
        K.out_off = st;
        B->s_off[(size_t)b] = st;
        st += (int64_t)K.kt * K.ks;
        blks.push_back(K);
      }
    B->s_off[(size_t)s_row_ptr[P]] = st;
    SBlk* dblk = nullptr;
    PTgt* dtg = nullptr;
    double2* dP = nullptr;
    if (!rc) rc = up(&dblk, blks.data(), blks.size());
    if (!rc) rc = up(&dtg, tgs.data(), tgs.size());
    if (!rc) {
      cudaError_t e1 = cudaMalloc(&B->S, sizeof(double2) * std::max<int64_t>(st, 1));
      cudaError_t e2 = cudaMalloc(&dP, sizeof(double2) * std::max<int64_t>(ptot, 1));
      if (e1 != cudaSuccess || e2 != cudaSuccess) rc = H2B_ENOMEM;
    }
    if (!rc) H2B_CUDA_TRY(cudaMemset(B->S, 0, sizeof(double2) * std::max<int64_t>(st, 1)));
    if (!rc && !tgs.empty()) {
      k_stage2_proj<<<(int)tgs.size(), 256>>>(dtg, dA, Vf, dvf, dP);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        h2b_set_error(std::string("h2b_builder_create: projections: ") + cudaGetErrorString(e));
        rc = H2B_ECUDA;
      }
    }
    // blocks whose target has no Stage-I factor keep S = 0 (the reference's zero coupling)
    if (!rc) {
      std::vector<SBlk> live;
      for (const SBlk& K : blks)
        if (K.r > 0 && p_of[K.t] >= 0 && K.kt > 0 && K.ks > 0) live.push_back(K);
      if (dblk) cudaFree(dblk);
      dblk = nullptr;
      rc = up(&dblk, live.data(), live.size());
      if (!rc && !live.empty()) {
        k_stage2_couple<<<(int)live.size(), 256>>>(dblk, dP, dB, Vf, dvf, B->S);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          h2b_set_error(std::string("h2b_builder_create: couplings: ") + cudaGetErrorString(e));
          rc = H2B_ECUDA;
        }
      }
    }
    if (dblk) cudaFree(dblk);
    if (dtg) cudaFree(dtg);
    if (dP) cudaFree(dP);
  }
  void* ptrs[] = {dA, dM, dB, dsize, drank, dvf, Vf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (rc) {
    if (B->res) cudaFree(B->res);
    if (B->S) cudaFree(B->S);
    delete B;
    return rc;
  }
  *out = B;
  return H2B_OK;
}

extern "C" int h2b_builder_ranks(void* b, int32_t* k) {
  h2b_builder_ctx* B = (h2b_builder_ctx*)b;
  if (!B || !k) {
    h2b_set_error("h2b_builder_ranks: null argument");
    return H2B_EINVAL;
  }
  std::copy(B->rank.begin(), B->rank.end(), k);
  return H2B_OK;
}

// what 0: leaf bases V_c (n_c x k_c) for every leaf, in packed order, concatenated;
//      1: transfers [T_lo; T_hi] ((k_lo + k_hi) x k_c) for every non-leaf, concatenated;
//      2: couplings S (k_t x k_s) in the CSR order of the admissible blocks.
// dst: host buffer of the concatenated size (complex128); c_child_lo: leaf test.
extern "C" int h2b_builder_fetch(void* b, int what, const int32_t* c_child_lo, void* dst) {
  h2b_builder_ctx* B = (h2b_builder_ctx*)b;
  if (!B || !dst || (what != 2 && !c_child_lo)) {
    h2b_set_error("h2b_builder_fetch: null argument");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(B->device));
  double2* o = (double2*)dst;
  if (what == 2) {
    H2B_CUDA_TRY(cudaMemcpy(o, B->S, sizeof(double2) * B->s_off.back(), cudaMemcpyDeviceToHost));
    return H2B_OK;
  }
  for (int c = 0; c < B->P; ++c) {
    const bool leaf = c_child_lo[c] < 0;
    if ((what == 0) != leaf) continue;
    const int64_t e = (int64_t)B->m_of[c] * B->rank[c];
    if (e) H2B_CUDA_TRY(cudaMemcpy(o, B->res + B->res_off[c], sizeof(double2) * e, cudaMemcpyDeviceToHost));
    o += e;
  }
  return H2B_OK;
}

extern "C" int h2b_builder_destroy(void* b) {
  h2b_builder_ctx* B = (h2b_builder_ctx*)b;
  if (!B) return H2B_OK;
  cudaSetDevice(B->device);
  if (B->res) cudaFree(B->res);
  if (B->S) cudaFree(B->S);
  delete B;
  return H2B_OK;
}

// =================================================================================================
// Stage I on the device: partially pivoted adaptive cross approximation of every cluster's
// grouped admissible block row (the cluster's points x all its partners' points), restating
// linalg.aca_factorize (/root/reference/pkg/src/h2vie/linalg.py:87-178) with the reference's
// pivoting, Frobenius estimate and stopping rule; entries sampled on the fly from the geometry
// (kernel.py:190-210: S[m, n] = -chi_n (k0^2 V / 4 pi r) e^{-j k0 r}, admissible blocks never
// hold the diagonal).  One CTA per cluster.  The SVD trim of the reference (recompress_lowrank)
// is skipped: the Gram matrices and couplings of Stage II depend on the block A B^T only, and
// Stage II's truncated eigendecomposition trims at eps_acc.
// =================================================================================================
namespace {

constexpr int AT = 256;

struct ACAClu {
  int32_t c, nr, ncols, cap;
  int64_t cols_off;   // into the column index list (original point indices, partners in CSR order)
  int64_t ws_a, ws_b; // workspace: a (nr x cap), b (ncols x cap), row-major
  int64_t ws_f;       // flags: used rows (nr) then used cols (ncols), one byte each
};

__device__ __forceinline__ double2 sys_entry(int64_t m, int64_t n, const double* __restrict__ ctr,
                                             const double2* __restrict__ chi, double k0, double coef) {
  const double dx = ctr[3 * m] - ctr[3 * n], dy = ctr[3 * m + 1] - ctr[3 * n + 1], dz = ctr[3 * m + 2] - ctr[3 * n + 2];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  const double amp = coef / r;
  double sn, cs;
  sincos(k0 * r, &sn, &cs);
  const double ar = amp * cs, ai = -(amp * sn);
  const double2 cn = chi[n];
  return make_double2(-(cn.x * ar - cn.y * ai), -(cn.x * ai + cn.y * ar));
}

// block-wide argmax of v (value, index), ties to the lowest index (np.argmax)
__device__ void bmax(double v, int i, double* sv, int* si, double* out_v, int* out_i) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_down_sync(0xffffffffu, v, o);
    const int i2 = __shfl_down_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
  if (lane == 0) { sv[w] = v; si[w] = i; }
  __syncthreads();
  if (tid == 0) {
    double bv = sv[0];
    int bi = si[0];
    for (int k = 1; k < AT / 32; ++k)
      if (sv[k] > bv || (sv[k] == bv && si[k] < bi)) { bv = sv[k]; bi = si[k]; }
    *out_v = bv;
    *out_i = bi;
  }
  __syncthreads();
}

__device__ double bsum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < AT / 32; ++k) s += red[k];
    red[AT / 32] = s;
  }
  __syncthreads();
  s = red[AT / 32];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(AT) k_aca(const ACAClu* __restrict__ clus, const int32_t* __restrict__ c_start,
                                            const int64_t* __restrict__ perm, const int64_t* __restrict__ cols_all,
                                            const double* __restrict__ ctr, const double2* __restrict__ chi, double k0,
                                            double coef, double eps_aca, double2* ws, unsigned char* flags,
                                            int32_t* rank_out, int32_t* err) {
  __shared__ double sv[AT / 32 + 1];
  __shared__ int si[AT / 32];
  __shared__ double s_v;
  __shared__ int s_i, s_next, s_stop;
  __shared__ double2 s_piv;
  __shared__ double2 dots[2][200];
  const ACAClu C = clus[blockIdx.x];
  const int tid = threadIdx.x, nr = C.nr, nc = C.ncols, cap = C.cap;
  const int64_t r0 = c_start[C.c];
  const int64_t* cols = cols_all + C.cols_off;
  double2* a = ws + C.ws_a;
  double2* b = ws + C.ws_b;
  unsigned char* ur = flags + C.ws_f;
  unsigned char* uc = ur + nr;
  for (int i = tid; i < nr; i += AT) ur[i] = 0;
  for (int j = tid; j < nc; j += AT) uc[j] = 0;
  if (tid == 0) { s_next = 0; s_stop = 0; }
  __syncthreads();
  const int full = min(nr, nc);
  double fro2 = 0.0;
  int k = 0;
  for (;;) {
    // residual row at the pivot row, skipping rows that are already resolved
    bool found = false;
    while (s_next >= 0) {
      const int i = s_next;
      if (tid == 0) ur[i] = 1;
      const int64_t m = perm[r0 + i];
      double best = -1.0;
      int bj = 0x7fffffff;
      for (int j = tid; j < nc; j += AT) {
        double2 r = make_double2(0.0, 0.0);
        if (!uc[j]) {
          r = sys_entry(m, cols[j], ctr, chi, k0, coef);
          for (int l = 0; l < k; ++l) {  // r -= a_l[i] b_l[j]
            const double2 al = a[(int64_t)i * cap + l], bl = b[(int64_t)j * cap + l];
            r.x -= al.x * bl.x - al.y * bl.y;
            r.y -= al.x * bl.y + al.y * bl.x;
          }
        }
        b[(int64_t)j * cap + k] = r;  // the candidate row, scaled below
        const double ab = hypot(r.x, r.y);
        if (ab > best) { best = ab; bj = j; }
      }
      bmax(best, bj, sv, si, &s_v, &s_i);
      if (s_v > 0.0) { found = true; break; }
      if (tid == 0) {  // first free row, or none
        int nx = -1;
        for (int q = 0; q < nr; ++q)
          if (!ur[q]) { nx = q; break; }
        s_next = nx;
      }
      __syncthreads();
    }
    if (!found) break;
    const int j = s_i;
    if (tid == 0) { s_piv = b[(int64_t)j * cap + k]; uc[j] = 1; }
    __syncthreads();
    const double2 pv = s_piv;
    const double pn = pv.x * pv.x + pv.y * pv.y;
    double nb2 = 0.0;
    for (int q = tid; q < nc; q += AT) {  // b_new = row / pivot
      const double2 r = b[(int64_t)q * cap + k];
      const double2 v = make_double2((r.x * pv.x + r.y * pv.y) / pn, (r.y * pv.x - r.x * pv.y) / pn);
      b[(int64_t)q * cap + k] = v;
      nb2 += v.x * v.x + v.y * v.y;
    }
    const int64_t nj = cols[j];
    double na2 = 0.0;
    for (int q = tid; q < nr; q += AT) {  // a_new = column j - sum b_l[j] a_l
      double2 c = sys_entry(perm[r0 + q], nj, ctr, chi, k0, coef);
      for (int l = 0; l < k; ++l) {
        const double2 bl = b[(int64_t)j * cap + l], al = a[(int64_t)q * cap + l];
        c.x -= bl.x * al.x - bl.y * al.y;
        c.y -= bl.x * al.y + bl.y * al.x;
      }
      a[(int64_t)q * cap + k] = c;
      na2 += c.x * c.x + c.y * c.y;
    }
    __syncthreads();
    nb2 = bsum(nb2, sv);
    na2 = bsum(na2, sv);
    // cross = sum_l Re(<a_l, a_new> <b_l, b_new>), l = 0 .. k-1 (k < cap <= 200)
    for (int l = tid; l < k; l += AT) {
      double2 da = make_double2(0.0, 0.0), db = da;
      for (int q = 0; q < nr; ++q) cfma_conj(da, a[(int64_t)q * cap + l], a[(int64_t)q * cap + k]);
      for (int q = 0; q < nc; ++q) cfma_conj(db, b[(int64_t)q * cap + l], b[(int64_t)q * cap + k]);
      dots[0][l] = da;
      dots[1][l] = db;
    }
    __syncthreads();
    double cross = 0.0;
    if (tid == 0) {
      for (int l = 0; l < k; ++l) {
        const double2 da = dots[0][l], db = dots[1][l];
        cross += da.x * db.x - da.y * db.y;
      }
      double f2 = fro2 + na2 * nb2 + 2.0 * cross;
      f2 = f2 > 0.0 ? f2 : 0.0;
      if (na2 * nb2 <= eps_aca * eps_aca * f2) {
        s_stop = 1;  // converged: the terminating cross is dropped
      } else {
        fro2 = f2;
        s_stop = 0;
      }
    }
    __syncthreads();
    if (s_stop) break;
    ++k;
    if (k >= full) break;
    if (k >= cap) {
      if (tid == 0) atomicExch(err, C.c + 1);
      break;
    }
    // next pivot row: the largest |a_new| over unused rows, else the first free row
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int q = tid; q < nr; q += AT) {
      const double2 v = a[(int64_t)q * cap + k - 1];
      const double ab = ur[q] ? 0.0 : hypot(v.x, v.y);
      if (ab > best || (ab == best && q < bi)) { best = ab; bi = q; }
    }
    bmax(best, bi, sv, si, &s_v, &s_i);
    if (tid == 0) {
      if (s_v > 0.0) {
        s_next = s_i;
      } else {
        int nx = -1;
        for (int q = 0; q < nr; ++q)
          if (!ur[q]) { nx = q; break; }
        s_next = nx;
      }
    }
    __syncthreads();
    if (s_next < 0) break;
  }
  if (tid == 0) rank_out[C.c] = k;
}

}  // namespace

namespace {
// compacted Stage-I factors of one cluster: A (nr x r), B (ncols x r), M = B^T conj(B) (r x r)
__global__ void k_stage1_pack(const ACAClu* __restrict__ clus, const int32_t* __restrict__ rank,
                              const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off,
                              const int64_t* __restrict__ m_off, const double2* __restrict__ ws, double2* A,
                              double2* B, double2* M) {
  const ACAClu C = clus[blockIdx.x];
  const int r = rank[C.c], cap = C.cap;
  if (r == 0) return;
  const double2* a = ws + C.ws_a;
  const double2* b = ws + C.ws_b;
  for (int e = threadIdx.x; e < C.nr * r; e += blockDim.x) A[a_off[C.c] + e] = a[(int64_t)(e / r) * cap + e % r];
  for (int e = threadIdx.x; e < C.ncols * r; e += blockDim.x) B[b_off[C.c] + e] = b[(int64_t)(e / r) * cap + e % r];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < C.ncols; ++q) cfma_conj(s, b[(int64_t)q * cap + j], b[(int64_t)q * cap + i]);  // B[q,i] conj(B[q,j])
    M[m_off[C.c] + e] = s;
  }
}
}  // namespace

struct h2b_stage1_ctx {
  int P = 0, device = 0;
  double2 *A = nullptr, *B = nullptr, *M = nullptr;
  int64_t na = 0, nb = 0, nm = 0;
};

// Stage I on the device for the admissible block structure (s_row_ptr / s_col, packed CSR) of a
// cluster tree (c_start / c_size, perm) over a voxel geometry.  Outputs: per-cluster ACA rank,
// the offsets of the compacted factors (a_off / b_off / m_off, P + 1 each), the partner lists in
// CSR order with each partner's first row in B (part_ptr P + 1, partner / prow one per block);
// the factors themselves via h2b_stage1_fetch.
extern "C" int h2b_stage1_run(int P, const int32_t* c_start, const int32_t* c_size, const int64_t* perm, int64_t n,
                              const int64_t* s_row_ptr, const int32_t* s_col, const double* centers, const void* chi,
                              double k0, double volume, double eps_aca, int max_rank, int device, int32_t* rank_out,
                              int64_t* a_off, int64_t* b_off, int64_t* m_off, int64_t* part_ptr, int32_t* partner,
                              int64_t* prow, void** out) {
  if (!c_start || !c_size || !perm || !s_row_ptr || !centers || !chi || !rank_out || !out || P < 1) {
    h2b_set_error("h2b_stage1_run: null argument");
    return H2B_EINVAL;
  }
  *out = nullptr;
  H2B_CUDA_TRY(cudaSetDevice(device));
  // partner lists (CSR order) and each partner's first row in the grouped B
  std::vector<int64_t> ncols(P, 0);
  part_ptr[0] = 0;
  for (int c = 0; c < P; ++c) {
    int64_t nc = 0;
    for (int64_t b = s_row_ptr[c]; b < s_row_ptr[c + 1]; ++b) {
      partner[b] = s_col[b];
      prow[b] = nc;
      nc += c_size[s_col[b]];
    }
    ncols[c] = nc;
    part_ptr[c + 1] = s_row_ptr[c + 1];
  }
  h2b_stage1_ctx* S = new h2b_stage1_ctx();
  S->P = P;
  S->device = device;
  int32_t *dstart = nullptr, *drank = nullptr, *derr = nullptr;
  int64_t* dperm = nullptr;
  double* dctr = nullptr;
  double2* dchi = nullptr;
  std::vector<int32_t> zeros(P, 0);
  int rc = up(&dstart, c_start, (size_t)P);
  if (!rc) rc = up(&dperm, perm, (size_t)n);
  if (!rc) rc = up(&dctr, centers, (size_t)(3 * n));
  if (!rc) rc = up(&dchi, (const double2*)chi, (size_t)n);
  if (!rc) rc = up(&drank, zeros.data(), (size_t)P);
  if (!rc) rc = up(&derr, zeros.data(), 1);
  const double coef = k0 * k0 * volume / (4.0 * 3.14159265358979323846);
  // clusters in batches of bounded ACA workspace (packed order, so the compacted factors come out
  // in packed order): the workspace holds cap columns per cluster, the factors only their rank
  struct Part {
    double2 *A = nullptr, *B = nullptr, *M = nullptr;
    int64_t na = 0, nb = 0, nm = 0;
  };
  std::vector<Part> parts;
  a_off[0] = b_off[0] = m_off[0] = 0;
  const int64_t WS_MAX = (int64_t)1 << 31;  // complex elements of ACA workspace per batch (32 GB)
  int c0 = 0;
  while (c0 < P && !rc) {
    std::vector<ACAClu> clus;
    std::vector<int64_t> cols;
    int64_t ws = 0, fl = 0;
    int c1 = c0;
    for (; c1 < P; ++c1) {
      const int64_t nc = ncols[c1];
      if (nc == 0) continue;
      ACAClu C{};
      C.c = c1;
      C.nr = c_size[c1];
      C.ncols = (int32_t)nc;
      C.cap = (int32_t)std::min<int64_t>(std::min<int64_t>(max_rank, 200), std::min<int64_t>(C.nr, nc));
      const int64_t need = ((int64_t)C.nr + nc) * C.cap;
      if (!clus.empty() && ws + need > WS_MAX) break;
      C.cols_off = (int64_t)cols.size();
      for (int64_t b = s_row_ptr[c1]; b < s_row_ptr[c1 + 1]; ++b) {
        const int s = s_col[b];
        for (int q = 0; q < c_size[s]; ++q) cols.push_back(perm[c_start[s] + q]);
      }
      C.ws_a = ws;
      ws += (int64_t)C.nr * C.cap;
      C.ws_b = ws;
      ws += nc * C.cap;
      C.ws_f = fl;
      fl += C.nr + nc;
      clus.push_back(C);
    }
    ACAClu* dclus = nullptr;
    int64_t *dcols = nullptr, *dao = nullptr, *dbo = nullptr, *dmo = nullptr;
    double2* dws = nullptr;
    unsigned char* dfl = nullptr;
    Part pt;
    rc = up(&dclus, clus.data(), clus.size());
    if (!rc) rc = up(&dcols, cols.data(), cols.size());
    if (!rc) {
      cudaError_t e1 = cudaMalloc(&dws, sizeof(double2) * std::max<int64_t>(ws, 1));
      cudaError_t e2 = cudaMalloc(&dfl, std::max<int64_t>(fl, 1));
      if (e1 != cudaSuccess || e2 != cudaSuccess) {
        h2b_set_error("h2b_stage1_run: ACA workspace allocation failed");
        rc = H2B_ENOMEM;
      }
    }
    if (!rc && !clus.empty()) {
      k_aca<<<(int)clus.size(), AT>>>(dclus, dstart, dperm, dcols, dctr, dchi, k0, coef, eps_aca, dws, dfl, drank,
                                      derr);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        h2b_set_error(std::string("h2b_stage1_run: ACA kernel: ") + cudaGetErrorString(e));
        rc = H2B_ECUDA;
      }
    }
    if (!rc) {
      int32_t err = 0;
      H2B_CUDA_TRY(cudaMemcpy(rank_out, drank, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
      H2B_CUDA_TRY(cudaMemcpy(&err, derr, sizeof(int32_t), cudaMemcpyDeviceToHost));
      if (err) {
        h2b_set_error("h2b_stage1_run: ACA reached its rank cap at cluster " + std::to_string(err - 1) +
                      " (the reference raises ClusterCompressionError)");
        rc = H2B_EINVAL;
      }
    }
    if (!rc) {
      // batch-local offsets for clusters c0 .. c1-1, then the global ones
      std::vector<int64_t> la(P + 1, 0), lb(P + 1, 0), lm(P + 1, 0);
      for (int c = c0; c < c1; ++c) {
        const int64_t r = rank_out[c];
        la[c + 1] = la[c] + (int64_t)c_size[c] * r;
        lb[c + 1] = lb[c] + ncols[c] * r;
        lm[c + 1] = lm[c] + r * r;
        a_off[c + 1] = a_off[c] + (int64_t)c_size[c] * r;
        b_off[c + 1] = b_off[c] + ncols[c] * r;
        m_off[c + 1] = m_off[c] + r * r;
      }
      pt.na = la[c1];
      pt.nb = lb[c1];
      pt.nm = lm[c1];
      rc = up(&dao, la.data(), (size_t)P + 1);
      if (!rc) rc = up(&dbo, lb.data(), (size_t)P + 1);
      if (!rc) rc = up(&dmo, lm.data(), (size_t)P + 1);
      if (!rc) {
        cudaError_t e1 = cudaMalloc(&pt.A, sizeof(double2) * std::max<int64_t>(pt.na, 1));
        cudaError_t e2 = cudaMalloc(&pt.B, sizeof(double2) * std::max<int64_t>(pt.nb, 1));
        cudaError_t e3 = cudaMalloc(&pt.M, sizeof(double2) * std::max<int64_t>(pt.nm, 1));
        if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) rc = H2B_ENOMEM;
      }
      if (!rc && !clus.empty()) {
        k_stage1_pack<<<(int)clus.size(), 256>>>(dclus, drank, dao, dbo, dmo, dws, pt.A, pt.B, pt.M);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          h2b_set_error(std::string("h2b_stage1_run: pack: ") + cudaGetErrorString(e));
          rc = H2B_ECUDA;
        }
      }
      parts.push_back(pt);
    }
    void* ptrs[] = {dclus, dcols, dao, dbo, dmo, dws, dfl};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    c0 = c1;
  }
  // one buffer per factor kind, batches in order (packed order)
  if (!rc) {
    S->na = a_off[P];
    S->nb = b_off[P];
    S->nm = m_off[P];
    cudaError_t e1 = cudaMalloc(&S->A, sizeof(double2) * std::max<int64_t>(S->na, 1));
    cudaError_t e2 = cudaMalloc(&S->B, sizeof(double2) * std::max<int64_t>(S->nb, 1));
    cudaError_t e3 = cudaMalloc(&S->M, sizeof(double2) * std::max<int64_t>(S->nm, 1));
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) rc = H2B_ENOMEM;
    int64_t oa = 0, ob = 0, om = 0;
    for (const Part& pt : parts) {
      if (rc) break;
      if (pt.na) H2B_CUDA_TRY(cudaMemcpy(S->A + oa, pt.A, sizeof(double2) * pt.na, cudaMemcpyDeviceToDevice));
      if (pt.nb) H2B_CUDA_TRY(cudaMemcpy(S->B + ob, pt.B, sizeof(double2) * pt.nb, cudaMemcpyDeviceToDevice));
      if (pt.nm) H2B_CUDA_TRY(cudaMemcpy(S->M + om, pt.M, sizeof(double2) * pt.nm, cudaMemcpyDeviceToDevice));
      oa += pt.na;
      ob += pt.nb;
      om += pt.nm;
    }
  }
  for (const Part& pt : parts) {
    if (pt.A) cudaFree(pt.A);
    if (pt.B) cudaFree(pt.B);
    if (pt.M) cudaFree(pt.M);
  }
  void* ptrs[] = {dstart, drank, derr, dperm, dctr, dchi};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (rc) {
    if (S->A) cudaFree(S->A);
    if (S->B) cudaFree(S->B);
    if (S->M) cudaFree(S->M);
    delete S;
    return rc;
  }
  *out = S;
  return H2B_OK;
}

// device pointers of the Stage-I factors (for h2b_builder_create without a host round trip)
extern "C" int h2b_stage1_device_ptrs(void* h, void** a, void** b, void** m) {
  h2b_stage1_ctx* S = (h2b_stage1_ctx*)h;
  if (!S || !a || !b || !m) {
    h2b_set_error("h2b_stage1_device_ptrs: null argument");
    return H2B_EINVAL;
  }
  *a = S->A;
  *b = S->B;
  *m = S->M;
  return H2B_OK;
}

extern "C" int h2b_stage1_fetch(void* h, void* a, void* b, void* m) {
  h2b_stage1_ctx* S = (h2b_stage1_ctx*)h;
  if (!S) {
    h2b_set_error("h2b_stage1_fetch: null handle");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(S->device));
  if (a && S->na) H2B_CUDA_TRY(cudaMemcpy(a, S->A, sizeof(double2) * S->na, cudaMemcpyDeviceToHost));
  if (b && S->nb) H2B_CUDA_TRY(cudaMemcpy(b, S->B, sizeof(double2) * S->nb, cudaMemcpyDeviceToHost));
  if (m && S->nm) H2B_CUDA_TRY(cudaMemcpy(m, S->M, sizeof(double2) * S->nm, cudaMemcpyDeviceToHost));
  return H2B_OK;
}

extern "C" int h2b_stage1_destroy(void* h) {
  h2b_stage1_ctx* S = (h2b_stage1_ctx*)h;
  if (!S) return H2B_OK;
  cudaSetDevice(S->device);
  if (S->A) cudaFree(S->A);
  if (S->B) cudaFree(S->B);
  if (S->M) cudaFree(S->M);
  delete S;
  return H2B_OK;
}
