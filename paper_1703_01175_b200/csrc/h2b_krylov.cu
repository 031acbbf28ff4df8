// Krylov solvers around the H² matvec, on device (sm_100a).
//
// * GMRES(m) with CGS2 Arnoldi — new component (the reference has no GMRES,
//   SURVEY.md §0 finding 1); restates oracle/krylov_oracle.py::gmres_solve.
// * BiCGStab — restates the reference's own solver line by line
//   (/root/reference/pkg/src/h2vie/arith.py:605-689).
//
// Vector work is done by fused reduction kernels with a deterministic
// two-stage (per-CTA partial, then fixed-order final sum) reduction, so the
// same inputs always produce the same bits.  The Givens rotations of each
// Arnoldi step run on the device (givens_update); the host reads each step's
// residual from mapped pinned memory one step behind the GPU and does the
// cycle's (<= 63 x 63) back substitution.
#include <math.h>

#include <algorithm>
#include <chrono>
#include <complex>
#include <map>
#include <vector>

#include <cooperative_groups.h>

#include "h2b_common.cuh"

namespace {

constexpr int RT = 256;      // threads per reduction CTA
constexpr int RB_MAX = 296;  // max reduction CTAs (2 per SM)
constexpr int MAXV = 8;      // max pairs per fused dot launch

__device__ __forceinline__ double2 block_sum2(double2 v, double2* sm) {
  v = warp_sum2(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int w = 0; w < RT / 32; ++w) s = cadd(s, sm[w]);
  return s;  // valid in thread 0
}

struct DotPairs {
  const double2* a[MAXV];
  const double2* b[MAXV];
  int np;
};

// partial[j*gridDim + block] = Σ_{i in block's slice} conj(a_j[i]) b_j[i]
__global__ void __launch_bounds__(RT) k_dots_partial(DotPairs d, int64_t n, double2* partial) {
  __shared__ double2 sm[RT / 32];
  for (int j = 0; j < d.np; ++j) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT)
      cfma_conj(acc, d.a[j][i], d.b[j][i]);
    double2 s = block_sum2(acc, sm);
    if (threadIdx.x == 0) partial[j * gridDim.x + blockIdx.x] = s;
  }
}

// multi-dot against the rows of a basis: partial[j*nb+blk] = Σ conj(V[j*ldv+i]) w[i]; one grid
// row (blockIdx.y) per basis vector, so all j run in parallel (fixed per-block summation order)
__global__ void __launch_bounds__(RT) k_basis_dots_partial(const double2* __restrict__ V, int64_t ldv,
                                                           int nv, const double2* __restrict__ w,
                                                           int64_t n, double2* partial) {
  __shared__ double2 sm[RT / 32];
  const int j = blockIdx.y;
  if (j >= nv) return;
  const double2* vj = V + j * ldv;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT)
    cfma_conj(acc, vj[i], w[i]);
  double2 s = block_sum2(acc, sm);
  if (threadIdx.x == 0) partial[j * gridDim.x + blockIdx.x] = s;
}

// out[j] = Σ_blk partial[j*nb + blk] in fixed order (one warp per j)
__global__ void k_reduce_partials(const double2* __restrict__ partial, int nb, int nv,
                                  double2* __restrict__ out) {
  const int j = blockIdx.x;
  if (j >= nv) return;
  const int lane = threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  for (int b = lane; b < nb; b += 32) acc = cadd(acc, partial[j * nb + b]);
  acc = warp_sum2(acc);
  if (lane == 0) out[j] = acc;
}

// w[i] -= Σ_j V[j*ldv+i] h[j]; optional partial of ||w||^2 (stored in .x)
__global__ void __launch_bounds__(RT) k_basis_sub(const double2* __restrict__ V, int64_t ldv, int nv,
                                                  const double2* __restrict__ hcoef, double2* w,
                                                  int64_t n, double2* nrm_partial) {
  __shared__ double2 sm[RT / 32];
  __shared__ double2 hs[64];
  for (int j = threadIdx.x; j < nv && j < 64; j += RT) hs[j] = hcoef[j];
  __syncthreads();
  double2 nrm = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < nv; ++j) cfma(acc, V[j * ldv + i], j < 64 ? hs[j] : hcoef[j]);
    double2 wi = w[i];
    wi.x -= acc.x;
    wi.y -= acc.y;
    w[i] = wi;
    nrm.x = fma(wi.x, wi.x, nrm.x);
    nrm.x = fma(wi.y, wi.y, nrm.x);
  }
  if (nrm_partial) {
    double2 s = block_sum2(nrm, sm);
    if (threadIdx.x == 0) nrm_partial[blockIdx.x] = s;
  }
}

struct Lin3 {
  double2 c[3];
  const double2* x[3];
  int nx;
};

// out = Σ c_k x_k (x_k may alias out); optional partial ||out||^2
__global__ void __launch_bounds__(RT) k_lincomb(Lin3 L, double2* out, int64_t n, double2* nrm_partial) {
  __shared__ double2 sm[RT / 32];
  double2 nrm = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < L.nx; ++k) cfma(acc, L.c[k], L.x[k][i]);
    out[i] = acc;
    nrm.x = fma(acc.x, acc.x, nrm.x);
    nrm.x = fma(acc.y, acc.y, nrm.x);
  }
  if (nrm_partial) {
    double2 s = block_sum2(nrm, sm);
    if (threadIdx.x == 0) nrm_partial[blockIdx.x] = s;
  }
}

int nblocks(int64_t n) {
  int64_t b = (n + RT - 1) / RT;  // small n: one element per thread (latency-bound)
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, RB_MAX));
}

typedef std::complex<double> cplx;

// Scratch of the reductions: partials (RB_MAX * 64), device scalars (256) and pinned, mapped
// host scalars (SCR_HOST).  Solvers use the scratch of their handle (allocated on the handle's
// device, never reallocated, so captured step graphs stay valid); the handle-less exported
// vector kernels use one scratch per (thread, device).  Host slots: [0, 128) general (fetched
// dot products, back-substitution coefficients), [128, 256) GMRES (res_j, hn_j) records,
// [256, 260) BiCGStab iteration records.
constexpr int SCR_HOST = 512, SCR_GMRES = 128, SCR_BICG = 256;
struct Scratch {
  double2* partial = nullptr;
  double2* vals = nullptr;
  double2* host = nullptr;
};

int scratch_alloc(Scratch* s) {
  H2B_CUDA_TRY(cudaMalloc(&s->partial, sizeof(double2) * RB_MAX * 64));
  H2B_CUDA_TRY(cudaMalloc(&s->vals, sizeof(double2) * 256));
  H2B_CUDA_TRY(cudaHostAlloc(&s->host, sizeof(double2) * SCR_HOST, cudaHostAllocMapped));
  return H2B_OK;
}

int handle_scratch(h2b_ctx* h, Scratch* out) {
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  if (!h->ks_partial) {
    Scratch s;
    const int rc = scratch_alloc(&s);
    if (rc) {
      if (s.partial) cudaFree(s.partial);
      if (s.vals) cudaFree(s.vals);
      return rc;
    }
    h->ks_partial = s.partial;
    h->ks_vals = s.vals;
    h->ks_host = s.host;
  }
  out->partial = h->ks_partial;
  out->vals = h->ks_vals;
  out->host = h->ks_host;
  return H2B_OK;
}

int thread_scratch(Scratch* out) {
  static thread_local std::map<int, Scratch> per_device;
  int dev = 0;
  H2B_CUDA_TRY(cudaGetDevice(&dev));
  auto it = per_device.find(dev);
  if (it == per_device.end()) {
    Scratch s;
    H2B_TRY(scratch_alloc(&s));
    it = per_device.emplace(dev, s).first;
  }
  *out = it->second;
  return H2B_OK;
}

// ---- device-side building blocks used by the solvers -----------------------
struct Ops {
  cudaStream_t st;
  int64_t n;
  int nb;
  double2 *partial, *vals, *host;

  // vals[0..np) = vdot(a_j, b_j); copies back to host[0..np) when `fetch`
  int dots(std::initializer_list<std::pair<const double2*, const double2*>> pairs, bool fetch) {
    DotPairs d;
    d.np = 0;
    for (auto& pr : pairs) {
      d.a[d.np] = pr.first;
      d.b[d.np] = pr.second;
      ++d.np;
    }
    k_dots_partial<<<nb, RT, 0, st>>>(d, n, partial);
    H2B_CHECK_LAUNCH();
    k_reduce_partials<<<d.np, 32, 0, st>>>(partial, nb, d.np, vals);
    H2B_CHECK_LAUNCH();
    if (fetch) return fetch_vals(d.np);
    return H2B_OK;
  }
  int fetch_vals(int cnt) {
    H2B_CUDA_TRY(cudaMemcpyAsync(host, vals, sizeof(double2) * cnt, cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    return H2B_OK;
  }
  // out = Σ c_k x_k ; if nrm: vals[slot] = ||out||^2
  int lincomb(double2* out, std::initializer_list<std::pair<cplx, const double2*>> terms, int nrm_slot) {
    Lin3 L;
    L.nx = 0;
    for (auto& t : terms) {
      L.c[L.nx] = make_double2(t.first.real(), t.first.imag());
      L.x[L.nx] = t.second;
      ++L.nx;
    }
    k_lincomb<<<nb, RT, 0, st>>>(L, out, n, nrm_slot >= 0 ? partial : nullptr);
    H2B_CHECK_LAUNCH();
    if (nrm_slot >= 0) {
      k_reduce_partials<<<1, 32, 0, st>>>(partial, nb, 1, vals + nrm_slot);
      H2B_CHECK_LAUNCH();
    }
    return H2B_OK;
  }
};

#define TRY(x)          \
  do {                  \
    int _rc = (x);      \
    if (_rc) return _rc; \
  } while (0)

struct KryWs {
  double2* base = nullptr;
  size_t bytes = 0;
};

int krylov_ws(h2b_ctx* h, size_t bytes, double2** out) {
  if (h->kry_bytes < bytes) {
    for (auto& kv : h->gmres_graphs) cudaGraphExecDestroy(kv.second);  // they point into kry
    h->gmres_graphs.clear();
    if (h->kry) cudaFree(h->kry);
    h->device_bytes -= h->kry_bytes;
    h->kry = nullptr;
    h->kry_bytes = 0;
    H2B_CUDA_TRY(cudaMalloc(&h->kry, bytes));
    h->kry_bytes = bytes;
    h->device_bytes += bytes;
  }
  *out = (double2*)h->kry;
  return H2B_OK;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}


}  // namespace

// the handle's Krylov workspace (grown on demand; the cached GMRES step graphs point into it)
int h2b_krylov_workspace(h2b_ctx* h, size_t bytes, double2** out) { return krylov_ws(h, bytes, out); }

namespace {

// ---- GMRES: Givens rotations on the device --------------------------------------------------
struct GivensState {
  double2* H;       // (m+1) x m, row-major: H[i*m + j]
  double2* g;       // m+1: rotated right-hand side
  double2* cs_sn;   // m: {c_i, 0}
  double2* res_hn;  // 2m: {res_j, 0}, {hn_j, 0}
  double2* scale;   // 1: 1 / hn of the last step (0 on breakdown)
  double2* bnrm;    // 1: {||b||, 0} of the current solve (written per solve, read by the graphs)
  double2* host_res = nullptr;  // optional: mapped pinned copy of res_hn (stored by the kernel itself)
};

// Restates the host recurrence of oracle/krylov_oracle.py::gmres_solve for step j:
// hc = h1 + h2 (CGS2), apply rotations 0..j-1, new rotation zeroing hn, update g.  The cosines
// c_i live in cs_sn[i].x, the complex sines s_i in the spare last row of H (H[m*m + i]), which
// never holds a Hessenberg entry (the sub-diagonal is rotated away, never stored).
__device__ __noinline__ void givens_update(int j, int m, const double2* hv, GivensState S) {
  const double bnrm = S.bnrm[0].x;
  double2 hc[64];
  for (int i = 0; i <= j; ++i) hc[i] = make_double2(hv[i].x + hv[64 + i].x, hv[i].y + hv[64 + i].y);
  const double hn = sqrt(hv[128].x);
  double2* sn = S.H + (size_t)m * m;  // row m of H: the complex sines
  for (int i = 0; i < j; ++i) {
    const double c = S.cs_sn[i].x;
    const double2 s = sn[i];
    const double2 a = hc[i], bb = hc[i + 1];
    // hc[i] = c a + s bb ; hc[i+1] = -conj(s) a + c bb
    hc[i] = make_double2(c * a.x + (s.x * bb.x - s.y * bb.y), c * a.y + (s.x * bb.y + s.y * bb.x));
    hc[i + 1] = make_double2(-(s.x * a.x + s.y * a.y) + c * bb.x, -(s.x * a.y - s.y * a.x) + c * bb.y);
  }
  double c;
  double2 s, rr;
  const double ahj = hypot(hc[j].x, hc[j].y);
  if (hn == 0.0) {
    c = 1.0; s = make_double2(0.0, 0.0); rr = hc[j];
  } else if (ahj == 0.0) {
    c = 0.0; s = make_double2(1.0, 0.0); rr = make_double2(hn, 0.0);
  } else {
    const double t = hypot(ahj, hn);
    const double2 ph = make_double2(hc[j].x / ahj, hc[j].y / ahj);
    c = ahj / t;
    s = make_double2(ph.x * hn / t, ph.y * hn / t);
    rr = make_double2(ph.x * t, ph.y * t);
  }
  S.cs_sn[j] = make_double2(c, 0.0);
  sn[j] = s;
  for (int i = 0; i <= j; ++i) S.H[(size_t)i * m + j] = hc[i];
  S.H[(size_t)j * m + j] = rr;
  const double2 gj = S.g[j];
  S.g[j + 1] = make_double2(-(s.x * gj.x + s.y * gj.y), -(s.x * gj.y - s.y * gj.x));  // -conj(s) gj
  S.g[j] = make_double2(c * gj.x, c * gj.y);
  const double2 gn = S.g[j + 1];
  S.res_hn[2 * j] = make_double2(hypot(gn.x, gn.y) / bnrm, 0.0);
  S.res_hn[2 * j + 1] = make_double2(hn, 0.0);
  if (S.host_res) {  // straight into the host's pinned buffer (no copy node in the step graph)
    S.host_res[2 * j] = S.res_hn[2 * j];
    S.host_res[2 * j + 1] = S.res_hn[2 * j + 1];
    __threadfence_system();
  }
  S.scale[0] = make_double2(hn == 0.0 ? 0.0 : 1.0 / hn, 0.0);
}

__global__ void k_givens_step(int j, int m, const double2* __restrict__ hv, GivensState S) {
  if (threadIdx.x == 0) givens_update(j, m, hv, S);
}

// out = {sqrt(v[0].x), 0}: a norm from a reduced squared norm
__global__ void k_set_norm(const double2* __restrict__ v, double2* out) {
  out[0] = make_double2(sqrt(v[0].x), 0.0);
}

// ---------------------------------------------------------------------------
// One Arnoldi step after the matvec (CGS2 against V[0..nv), normalisation, Givens update) in
// ONE launch of one thread-block cluster, for small n: CTA c owns rows [cR, cR + R) and keeps
// its rows of the basis and of w in shared memory (the basis is read once per step instead of
// four times); the per-CTA partial dot products meet through distributed shared memory, summed
// in CTA order by every CTA (deterministic, the same bits in all CTAs), at three cluster
// barriers.  Replaces nine launches of the multi-kernel step (dots / reduce / subtract twice,
// norm, Givens, scale), whose launch latencies dominate at these sizes.
// ---------------------------------------------------------------------------
constexpr int AC_T = 256;
struct ArnoldiArgs {
  const double2* V;
  int64_t n;
  int nv, R;
  double2* w;
  double2* hv;  // [0, nv): pass-1 coefficients, [64, 64 + nv): pass 2, [128]: ||w||^2
  GivensState S;
  int j, m;
};

__global__ void __launch_bounds__(AC_T) k_arnoldi_cluster(ArnoldiArgs A) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = AC_T / 32;
  extern __shared__ __align__(16) double2 dsm[];
  __shared__ double2 part[3][64];  // this CTA's partials: pass-1 dots, pass-2 dots, ||w||^2
  __shared__ double2 hs[64];
  __shared__ double2 red[NW];
  __shared__ double s_hn2;
  const int R = A.R, nv = A.nv;
  const int64_t row0 = (int64_t)c * R;
  const int64_t left = A.n - row0;
  const int rows = left <= 0 ? 0 : (left < R ? (int)left : R);
  double2* Vs = dsm;                // nv x R (vector-major)
  double2* ws = dsm + (size_t)nv * R;
  // this CTA's rows of the nv basis vectors and of w: one bulk copy per vector (a thread-strided
  // copy loop would serialise its global loads), rows past n zeroed
  __shared__ __align__(8) uint64_t bar;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(&bar, 16u * (uint32_t)(nv + 1) * (uint32_t)rows);
  }
  __syncthreads();
  if (tid <= nv && rows > 0)
    bulk_g2s(tid < nv ? Vs + (size_t)tid * R : ws, tid < nv ? A.V + (int64_t)tid * A.n + row0 : A.w + row0,
             16u * (uint32_t)rows, &bar);
  for (int idx = tid; idx < (nv + 1) * (R - rows); idx += AC_T) {
    const int i = idx / (R - rows), r = rows + (idx - i * (R - rows));
    (i < nv ? Vs + (size_t)i * R : ws)[r] = make_double2(0.0, 0.0);
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = warp; i < nv; i += NW) {  // this CTA's part of <V_i, w>, fixed order
      double2 acc = make_double2(0.0, 0.0);
      for (int r = lane; r < R; r += 32) cfma_conj(acc, Vs[(size_t)i * R + r], ws[r]);
      acc = warp_sum2(acc);
      if (lane == 0) part[pass][i] = acc;
    }
    cl.sync();  // every CTA's partials visible cluster-wide
    if (tid < nv) {
      double2 sum = make_double2(0.0, 0.0);
      for (int q = 0; q < ncl; ++q) sum = cadd(sum, cl.map_shared_rank(&part[pass][0], q)[tid]);
      hs[tid] = sum;
      if (c == 0) A.hv[64 * pass + tid] = sum;
    }
    __syncthreads();
    double2 nrm = make_double2(0.0, 0.0);
    for (int r = tid; r < R; r += AC_T) {  // w -= V h (CGS), then ||w||^2 on the second pass
      double2 acc = make_double2(0.0, 0.0);
      for (int i = 0; i < nv; ++i) cfma(acc, Vs[(size_t)i * R + r], hs[i]);
      double2 wi = ws[r];
      wi.x -= acc.x;
      wi.y -= acc.y;
      ws[r] = wi;
      nrm.x = fma(wi.x, wi.x, nrm.x);
      nrm.x = fma(wi.y, wi.y, nrm.x);
    }
    if (pass == 1) {
      nrm = warp_sum2(nrm);
      if (lane == 0) red[warp] = nrm;
      __syncthreads();
      if (tid == 0) {
        double2 t = make_double2(0.0, 0.0);
        for (int q = 0; q < NW; ++q) t = cadd(t, red[q]);
        part[2][0] = t;
      }
    }
    __syncthreads();
  }
  cl.sync();
  if (tid == 0) {
    double2 sum = make_double2(0.0, 0.0);
    for (int q = 0; q < ncl; ++q) sum = cadd(sum, cl.map_shared_rank(&part[2][0], q)[0]);
    s_hn2 = sum.x;
    if (c == 0) A.hv[128] = sum;
  }
  cl.sync();  // every remote read done: no CTA's shared memory is read after this point
  const double hn = sqrt(s_hn2), f = hn == 0.0 ? 0.0 : 1.0 / hn;  // = givens_update's scale
  for (int r = tid; r < rows; r += AC_T) A.w[row0 + r] = make_double2(ws[r].x * f, ws[r].y * f);
  if (c == 0 && tid == 0) givens_update(A.j, A.m, A.hv, A.S);  // reads CTA 0's hv writes
}

// Fused Arnoldi step configuration for (n, m): cluster size and rows per CTA, or cl = 0 (the
// multi-kernel step) when the basis rows of a CTA do not fit its shared memory or no cluster of
// that size can be resident.  H2B_NO_FUSED_ARNOLDI forces the multi-kernel step (A/B timing).
struct FusedArnoldi {
  int cl = 0, R = 0;
};
FusedArnoldi fused_arnoldi_config(int64_t n, int m) {
  FusedArnoldi f;
  if (getenv("H2B_NO_FUSED_ARNOLDI") || n <= 0) return f;
  constexpr int DYN_MAX = 200 * 1024;
  if (cudaFuncSetAttribute(k_arnoldi_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(k_arnoldi_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, DYN_MAX) != cudaSuccess) {
    cudaGetLastError();
    return f;
  }
  for (int cl : {16, 8}) {
    const int64_t R = (n + cl - 1) / cl;
    const int64_t bytes = (int64_t)sizeof(double2) * (m + 1) * R;  // nv <= m basis rows + w
    if (bytes > DYN_MAX) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(AC_T);
    cfg.dynamicSmemBytes = (size_t)bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_arnoldi_cluster, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nclusters >= 1) {
      f.cl = cl;
      f.R = (int)R;
      return f;
    }
  }
  return f;
}

// w *= scale[0] (a device scalar: the normalisation of the new basis vector)
__global__ void __launch_bounds__(RT) k_scale_dev(double2* w, int64_t n, const double2* __restrict__ scale) {
  const double f = scale[0].x;
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) {
    double2 v = w[i];
    w[i] = make_double2(v.x * f, v.y * f);
  }
}

// ---------------------------------------------------------------------------
// Graph-driven BiCGStab: one CUDA graph per iteration, every scalar of the recurrence computed
// and tested on the device (the host's only per-iteration work is reading a record that the
// last kernel stores into mapped pinned memory, one iteration behind the GPU).  A status word
// stops the recurrence: once it is non-zero every later kernel of the iteration — and of a
// speculatively queued next iteration — leaves the vectors alone.
// ---------------------------------------------------------------------------
enum BiStatus : int {
  BI_RUN = 0,
  BI_CONV_S = 1,       // converged on ||s|| (x += alpha p pending)
  BI_CONV_R = 2,       // converged on ||r||
  BI_RHO_BREAK = 3,    // rho breakdown: the host restarts with the noise vector or stops
  BI_DENOM_ZERO = 4,   // <rh, v> = 0 (one matvec done)
  BI_CONV_S_DONE = 5,  // BI_CONV_S with its x update applied
  BI_NONFINITE = 6,    // ||r|| not finite (its history entry is recorded)
  BI_OMEGA_ZERO = 7,   // <t, t> = 0 or omega = 0 (two matvecs done)
};
struct BiSc {
  double2 rho, alpha, omega, rho_new;
  double2 cp[3], cs[2], cx[3], cr[2];
  double hist_s, hist_r;
  int status, p_zero, run, pad;
};

// complex128 scalar arithmetic as numpy evaluates it (the reference's scalars are numpy
// complex128): Smith's division, products without fused multiply-adds
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {  // a / b
  const double abr = fabs(b.x), abi = fabs(b.y);
  if (abr >= abi) {
    if (abr == 0.0 && abi == 0.0) return make_double2(a.x / abr, a.y / abr);
    const double rat = b.y / b.x;
    const double scl = 1.0 / __dadd_rn(b.x, __dmul_rn(b.y, rat));
    return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                        __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  const double rat = b.x / b.y;
  const double scl = 1.0 / __dadd_rn(b.y, __dmul_rn(b.x, rat));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// out = Σ_k coef[k] x_k while the status equals `want` (optional ||out||^2 partials)
__global__ void __launch_bounds__(RT) k_lincomb_dev(const BiSc* __restrict__ sc, int want,
                                                    const double2* coef, int nx, const double2* x0,
                                                    const double2* x1, const double2* x2, double2* out,
                                                    int64_t n, double2* nrm_partial) {
  __shared__ double2 sm[RT / 32];
  if (sc->status != want) return;  // uniform over the grid
  const double2 c0 = coef[0], c1 = nx > 1 ? coef[1] : make_double2(0.0, 0.0),
                c2 = nx > 2 ? coef[2] : make_double2(0.0, 0.0);
  double2 nrm = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) {
    double2 acc = make_double2(0.0, 0.0);
    cfma(acc, c0, x0[i]);
    if (nx > 1) cfma(acc, c1, x1[i]);
    if (nx > 2) cfma(acc, c2, x2[i]);
    out[i] = acc;
    nrm.x = fma(acc.x, acc.x, nrm.x);
    nrm.x = fma(acc.y, acc.y, nrm.x);
  }
  if (nrm_partial) {
    double2 t = block_sum2(nrm, sm);
    if (threadIdx.x == 0) nrm_partial[blockIdx.x] = t;
  }
}

// rho_new = <rh, r>: breakdown test, then the coefficients of p = r + beta (p - omega v)
__global__ void k_bi_rho(BiSc* sc, const double2* vals, double thr) {
  ++sc->run;
  if (sc->status) return;
  const double2 rn = vals[0];
  if (hypot(rn.x, rn.y) < thr) {
    sc->status = BI_RHO_BREAK;
    return;
  }
  if (sc->p_zero) {
    sc->cp[0] = make_double2(1.0, 0.0);
    sc->cp[1] = sc->cp[2] = make_double2(0.0, 0.0);
    sc->p_zero = 0;
  } else {
    const double2 beta = cmul(cdiv(rn, sc->rho), cdiv(sc->alpha, sc->omega));
    const double2 bo = cmul(beta, sc->omega);
    sc->cp[0] = make_double2(1.0, 0.0);
    sc->cp[1] = beta;
    sc->cp[2] = make_double2(-bo.x, -bo.y);
  }
  sc->rho_new = rn;
}

// alpha = rho_new / <rh, v>; s = r - alpha v
__global__ void k_bi_alpha(BiSc* sc, const double2* vals) {
  if (sc->status) return;
  const double2 d = vals[0];
  if (d.x == 0.0 && d.y == 0.0) {
    sc->status = BI_DENOM_ZERO;
    return;
  }
  sc->alpha = cdiv(sc->rho_new, d);
  sc->cs[0] = make_double2(1.0, 0.0);
  sc->cs[1] = make_double2(-sc->alpha.x, -sc->alpha.y);
}

// ||s|| test: converged -> x += alpha p (by the BI_CONV_S-gated combination that follows)
__global__ void k_bi_snorm(BiSc* sc, const double2* vals, double bnrm, double tol) {
  if (sc->status) return;
  const double rel = sqrt(vals[0].x) / bnrm;
  sc->hist_s = rel;
  if (rel <= tol) {
    sc->cx[0] = make_double2(1.0, 0.0);
    sc->cx[1] = sc->alpha;
    sc->status = BI_CONV_S;
  }
}

__global__ void k_bi_mark(BiSc* sc, int from, int to) {
  if (sc->status == from) sc->status = to;
}

// omega = <t, s> / <t, t>; x += alpha p + omega s; r = s - omega t
__global__ void k_bi_omega(BiSc* sc, const double2* vals) {
  if (sc->status) return;
  const double tt = vals[0].x;
  if (tt == 0.0) {
    sc->status = BI_OMEGA_ZERO;
    return;
  }
  const double2 om = cdiv(vals[1], make_double2(tt, 0.0));  // numpy: vdot(t, s) / vdot(t, t)
  if (om.x == 0.0 && om.y == 0.0) {
    sc->status = BI_OMEGA_ZERO;
    return;
  }
  sc->omega = om;
  sc->cx[0] = make_double2(1.0, 0.0);
  sc->cx[1] = sc->alpha;
  sc->cx[2] = om;
  sc->cr[0] = make_double2(1.0, 0.0);
  sc->cr[1] = make_double2(-om.x, -om.y);
}

// ---------------------------------------------------------------------------
// Small n: each of the three vector segments of a BiCGStab iteration (dots -> scalar tests ->
// vector updates -> norm -> tests) as ONE launch of a 16-CTA thread-block cluster instead of
// five to seven launches.  Every CTA computes the same scalars from the same cluster sums
// (CTA-order summation over distributed shared memory: deterministic), CTA 0 alone writes the
// state back.  Segment 0: rho / p.  1: alpha / s / ||s|| test / x on convergence.  2: omega /
// x / r / ||r|| test / record.
// ---------------------------------------------------------------------------
struct BiSegArgs {
  BiSc* sc;
  const double2 *rh;
  double2 *r, *p, *v, *s, *t, *x;
  int64_t n;
  int R;  // rows per CTA
  double thr, bnrm, tol;
  double2* rec;
};

template <int NP>
__device__ __forceinline__ void cl_sums(cooperative_groups::cluster_group& cl, double2 (&v)[NP],
                                        double2* part, double2* red, double2* bcast) {
  // v: this thread's partials -> the cluster totals (valid in every thread of every CTA)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = AC_T / 32;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const double2 w = warp_sum2(v[i]);
    if (lane == 0) red[i * NW + warp] = w;
  }
  __syncthreads();
  if (tid < NP) {
    double2 a = make_double2(0.0, 0.0);
    for (int q = 0; q < NW; ++q) a = cadd(a, red[tid * NW + q]);
    part[tid] = a;
  }
  cl.sync();
  if (tid < NP) {
    double2 a = make_double2(0.0, 0.0);
    for (int q = 0; q < (int)cl.num_blocks(); ++q) a = cadd(a, cl.map_shared_rank(part, q)[tid]);
    bcast[tid] = a;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NP; ++i) v[i] = bcast[i];
}

__global__ void __launch_bounds__(AC_T) k_bicg_segment(BiSegArgs A, int seg) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double2 part0[4], part1[4], red[4 * (AC_T / 32)], bc[4];
  __shared__ BiSc S;  // this CTA's copy of the state
  const int tid = threadIdx.x, c = (int)cl.block_rank();
  const int64_t row0 = (int64_t)c * A.R;
  const int64_t row1 = row0 + A.R < A.n ? row0 + A.R : A.n;
  if (tid == 0) S = *A.sc;
  __syncthreads();
  const int status0 = S.status;
  if (seg == 0) {
    if (tid == 0) ++S.run;
    if (status0 == BI_RUN) {
      double2 d[1] = {make_double2(0.0, 0.0)};
      for (int64_t i = row0 + tid; i < row1; i += AC_T) cfma_conj(d[0], A.rh[i], A.r[i]);
      cl_sums<1>(cl, d, part0, red, bc);
      if (tid == 0) {
        const double2 rn = d[0];
        if (hypot(rn.x, rn.y) < A.thr) {
          S.status = BI_RHO_BREAK;
        } else if (S.p_zero) {
          S.cp[0] = make_double2(1.0, 0.0);
          S.cp[1] = S.cp[2] = make_double2(0.0, 0.0);
          S.p_zero = 0;
          S.rho_new = rn;
        } else {
          const double2 beta = cmul(cdiv(rn, S.rho), cdiv(S.alpha, S.omega));
          const double2 bo = cmul(beta, S.omega);
          S.cp[0] = make_double2(1.0, 0.0);
          S.cp[1] = beta;
          S.cp[2] = make_double2(-bo.x, -bo.y);
          S.rho_new = rn;
        }
      }
      __syncthreads();
      if (S.status == BI_RUN)
        for (int64_t i = row0 + tid; i < row1; i += AC_T) {
          double2 acc = make_double2(0.0, 0.0);
          cfma(acc, S.cp[0], A.r[i]);
          cfma(acc, S.cp[1], A.p[i]);
          cfma(acc, S.cp[2], A.v[i]);
          A.p[i] = acc;
        }
    }
  } else if (seg == 1 && status0 == BI_RUN) {
    double2 d[1] = {make_double2(0.0, 0.0)};
    for (int64_t i = row0 + tid; i < row1; i += AC_T) cfma_conj(d[0], A.rh[i], A.v[i]);
    cl_sums<1>(cl, d, part0, red, bc);
    if (tid == 0) {
      if (d[0].x == 0.0 && d[0].y == 0.0) {
        S.status = BI_DENOM_ZERO;
      } else {
        S.alpha = cdiv(S.rho_new, d[0]);
        S.cs[0] = make_double2(1.0, 0.0);
        S.cs[1] = make_double2(-S.alpha.x, -S.alpha.y);
      }
    }
    __syncthreads();
    if (S.status == BI_RUN) {
      double2 nr[1] = {make_double2(0.0, 0.0)};
      for (int64_t i = row0 + tid; i < row1; i += AC_T) {
        double2 acc = make_double2(0.0, 0.0);
        cfma(acc, S.cs[0], A.r[i]);
        cfma(acc, S.cs[1], A.v[i]);
        A.s[i] = acc;
        nr[0].x = fma(acc.x, acc.x, nr[0].x);
        nr[0].x = fma(acc.y, acc.y, nr[0].x);
      }
      cl_sums<1>(cl, nr, part1, red, bc);
      if (tid == 0) {
        const double rel = sqrt(nr[0].x) / A.bnrm;
        S.hist_s = rel;
        if (rel <= A.tol) {
          S.cx[0] = make_double2(1.0, 0.0);
          S.cx[1] = S.alpha;
          S.status = BI_CONV_S_DONE;  // x updated right below
        }
      }
      __syncthreads();
      if (S.status == BI_CONV_S_DONE)
        for (int64_t i = row0 + tid; i < row1; i += AC_T) {
          double2 acc = make_double2(0.0, 0.0);
          cfma(acc, S.cx[0], A.x[i]);
          cfma(acc, S.cx[1], A.p[i]);
          A.x[i] = acc;
        }
    }
  } else if (seg == 2) {
    if (status0 == BI_RUN) {
      double2 d[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
      for (int64_t i = row0 + tid; i < row1; i += AC_T) {
        cfma_conj(d[0], A.t[i], A.t[i]);
        cfma_conj(d[1], A.t[i], A.s[i]);
      }
      cl_sums<2>(cl, d, part0, red, bc);
      if (tid == 0) {
        const double tt = d[0].x;
        if (tt == 0.0) {
          S.status = BI_OMEGA_ZERO;
        } else {
          const double2 om = cdiv(d[1], make_double2(tt, 0.0));
          if (om.x == 0.0 && om.y == 0.0) {
            S.status = BI_OMEGA_ZERO;
          } else {
            S.omega = om;
            S.cx[0] = make_double2(1.0, 0.0);
            S.cx[1] = S.alpha;
            S.cx[2] = om;
            S.cr[0] = make_double2(1.0, 0.0);
            S.cr[1] = make_double2(-om.x, -om.y);
          }
        }
      }
      __syncthreads();
      if (S.status == BI_RUN) {
        double2 nr[1] = {make_double2(0.0, 0.0)};
        for (int64_t i = row0 + tid; i < row1; i += AC_T) {
          double2 acc = make_double2(0.0, 0.0);
          cfma(acc, S.cx[0], A.x[i]);
          cfma(acc, S.cx[1], A.p[i]);
          cfma(acc, S.cx[2], A.s[i]);
          A.x[i] = acc;
          double2 rr = make_double2(0.0, 0.0);
          cfma(rr, S.cr[0], A.s[i]);
          cfma(rr, S.cr[1], A.t[i]);
          A.r[i] = rr;
          nr[0].x = fma(rr.x, rr.x, nr[0].x);
          nr[0].x = fma(rr.y, rr.y, nr[0].x);
        }
        cl_sums<1>(cl, nr, part1, red, bc);
        if (tid == 0) {
          const double rel = sqrt(nr[0].x) / A.bnrm;
          S.hist_r = rel;
          S.rho = S.rho_new;
          if (rel <= A.tol)
            S.status = BI_CONV_R;
          else if (!isfinite(rel))
            S.status = BI_NONFINITE;
        }
      }
    }
    if (c == 0 && tid == 0) {  // the iteration's record (every iteration, whatever the status)
      double2* slot = A.rec + 2 * (S.run & 1);
      slot[1] = make_double2(S.hist_s, S.hist_r);
      slot[0] = make_double2((double)S.status, (double)S.run);
    }
  }
  if (c == 0 && tid == 0) {
    *A.sc = S;
    __threadfence_system();
  }
  cl.sync();  // no CTA's shared memory is read after its exit
}

// restart with a re-seeded shadow residual: scalars back to 1, p = v = 0 (the run counter stays)
__global__ void k_bi_restart(BiSc* sc) {
  sc->rho = sc->alpha = sc->omega = make_double2(1.0, 0.0);
  sc->p_zero = 1;
  sc->status = BI_RUN;
}

// ||r|| test and the iteration's record {status, run}, {hist_s, hist_r} into mapped pinned memory
__global__ void k_bi_final(BiSc* sc, const double2* vals, double bnrm, double tol, double2* rec) {
  if (sc->status == BI_RUN) {
    const double rel = sqrt(vals[0].x) / bnrm;
    sc->hist_r = rel;
    sc->rho = sc->rho_new;
    if (rel <= tol)
      sc->status = BI_CONV_R;
    else if (!isfinite(rel))
      sc->status = BI_NONFINITE;
  }
  double2* slot = rec + 2 * (sc->run & 1);
  slot[1] = make_double2(sc->hist_s, sc->hist_r);
  slot[0] = make_double2((double)sc->status, (double)sc->run);
  __threadfence_system();
}

}  // namespace

// ===========================================================================
// exported vector kernels
// ===========================================================================
extern "C" int h2b_zdotc_multi(const void* V, int64_t ldv, int nv, const void* w, int64_t n,
                               void* out_dev, void* stream) {
  if (nv < 1 || nv > 64 || n < 0 || !V || !w || !out_dev) {
    h2b_set_error("h2b_zdotc_multi: bad arguments (need 1 <= nv <= 64)");
    return H2B_EINVAL;
  }
  Scratch sc;
  TRY(thread_scratch(&sc));
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = nblocks(n);
  k_basis_dots_partial<<<dim3(nb, nv), RT, 0, st>>>((const double2*)V, ldv, nv, (const double2*)w, n,
                                          sc.partial);
  H2B_CHECK_LAUNCH();
  k_reduce_partials<<<nv, 32, 0, st>>>(sc.partial, nb, nv, (double2*)out_dev);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

extern "C" int h2b_zgemv_sub(const void* V, int64_t ldv, int nv, const void* h_dev, void* w,
                             int64_t n, double* nrm2_out_dev, void* stream) {
  if (nv < 0 || nv > 64 || n < 0 || !w) {
    h2b_set_error("h2b_zgemv_sub: bad arguments (need 0 <= nv <= 64)");
    return H2B_EINVAL;
  }
  Scratch sc;
  TRY(thread_scratch(&sc));
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = nblocks(n);
  k_basis_sub<<<nb, RT, 0, st>>>((const double2*)V, ldv, nv, (const double2*)h_dev, (double2*)w, n,
                                 nrm2_out_dev ? sc.partial : nullptr);
  H2B_CHECK_LAUNCH();
  if (nrm2_out_dev) {
    k_reduce_partials<<<1, 32, 0, st>>>(sc.partial, nb, 1, sc.vals);
    H2B_CHECK_LAUNCH();
    H2B_CUDA_TRY(cudaMemcpyAsync(nrm2_out_dev, sc.vals, sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  return H2B_OK;
}

extern "C" int h2b_zaxpby(int64_t n, double ar, double ai, const void* x, double br, double bi,
                          void* y, void* stream) {
  if (n < 0 || !x || !y) {
    h2b_set_error("h2b_zaxpby: bad arguments");
    return H2B_EINVAL;
  }
  Lin3 L;
  L.nx = 2;
  L.c[0] = make_double2(ar, ai);
  L.x[0] = (const double2*)x;
  L.c[1] = make_double2(br, bi);
  L.x[1] = (const double2*)y;
  k_lincomb<<<nblocks(n), RT, 0, (cudaStream_t)stream>>>(L, (double2*)y, n, nullptr);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

// ===========================================================================
// GMRES(m), CGS2, x0 = 0
// ===========================================================================
extern "C" int h2b_gmres(h2b_handle h, const void* b_perm, void* x_perm, int restart, double tol,
                         int max_iter, double* history, h2b_report* report, void* stream) {
  if (!h || !b_perm || !x_perm || !report) {
    h2b_set_error("h2b_gmres: null argument");
    return H2B_EINVAL;
  }
  if (!(tol > 0.0 && tol < 1.0) || max_iter < 1 || restart < 1 || restart > 63) {
    h2b_set_error("h2b_gmres: need 0 < tol < 1, max_iter >= 1, 1 <= restart <= 63");
    return H2B_EINVAL;
  }
  const double t0 = now_s();
  Scratch g_scratch;
  TRY(handle_scratch(h, &g_scratch));
  cudaStream_t st = (cudaStream_t)stream;
  TRY(h2b_order_begin(h, st));
  struct OrderEnd {  // the solve's last work on `st` orders the handle's next call
    h2b_ctx* h;
    cudaStream_t st;
    ~OrderEnd() { h2b_order_end(h, st); }
  } order_end{h, st};
  const int64_t n = h->n;
  const int m = restart;
  // workspace: V (m+1) x n basis, r, tmp, then the device Givens state
  const size_t gs_elems = (size_t)(m + 1) * m + (m + 1) + 3 * (size_t)m + 2;
  double2* ws = nullptr;
  TRY(krylov_ws(h, sizeof(double2) * ((size_t)n * (m + 3) + gs_elems), &ws));
  double2* V = ws;
  double2* r = ws + (size_t)n * (m + 1);
  double2* tmp = r + n;
  GivensState S;
  S.H = tmp + n;
  S.g = S.H + (size_t)(m + 1) * m;
  S.cs_sn = S.g + (m + 1);
  S.res_hn = S.cs_sn + m;
  S.scale = S.res_hn + m + m;
  S.bnrm = S.scale + 1;
  const double2* b = (const double2*)b_perm;
  double2* x = (double2*)x_perm;
  Ops ops{st, n, nblocks(n), g_scratch.partial, g_scratch.vals, g_scratch.host};
  double2* hvals = g_scratch.vals;        // device scalars (CGS2 coefficients, ||w||^2)
  double2* hres = g_scratch.host + SCR_GMRES;  // pinned: (res_j, hn_j) of step j
  S.host_res = nullptr;
  if (!getenv("H2B_GMRES_COPY_RES") && cudaHostGetDevicePointer((void**)&S.host_res, hres, 0) != cudaSuccess) {
    cudaGetLastError();
    S.host_res = nullptr;
  }

  *report = h2b_report{0, 0, 0, 0, 0.0};
  TRY(ops.dots({{b, b}}, true));
  const double bnrm = sqrt(g_scratch.host[0].x);
  H2B_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
  if (bnrm == 0.0) {
    report->converged = 1;
    report->wall_time = now_s() - t0;
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    return H2B_OK;
  }
  H2B_CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
  // ||b|| lives in device memory: the cached step graphs read it there, so a later solve with
  // another right-hand side on the same handle scales its residuals by its own norm
  k_set_norm<<<1, 1, 0, st>>>(g_scratch.vals, S.bnrm);
  H2B_CHECK_LAUNCH();
  const FusedArnoldi fa = fused_arnoldi_config(n, m);
  // one Arnoldi step j (matvec, CGS2, device Givens, normalisation, (res, hn) -> pinned host)
  // as a CUDA graph, captured once per (basis, j) and replayed
  auto step_graph = [&](int j, cudaGraphExec_t* out) -> int {
    const GmresKey key{V, j, m, n};
    auto it = h->gmres_graphs.find(key);
    if (it != h->gmres_graphs.end()) {
      *out = it->second;
      return H2B_OK;
    }
    cudaStream_t cs = nullptr;
    H2B_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    H2B_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    double2* w = V + (size_t)n * (j + 1);
    int nl = 0;
    int rc = h2b_enqueue_matvec(h, V + (size_t)n * j, w, 1, cs, &nl);
    if (!rc) {
      const int nb = ops.nb;
      if (fa.cl > 0) {  // the whole post-matvec step as one cluster launch
        ArnoldiArgs aa{V, n, j + 1, fa.R, w, hvals, S, j, m};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(fa.cl);
        cfg.blockDim = dim3(AC_T);
        cfg.dynamicSmemBytes = sizeof(double2) * (size_t)(j + 2) * fa.R;
        cfg.stream = cs;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = fa.cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, k_arnoldi_cluster, aa);
        if (le != cudaSuccess) {
          h2b_set_error(std::string("h2b_gmres: fused Arnoldi step: ") + cudaGetErrorString(le));
          rc = H2B_ECUDA;
        }
      } else {
      k_basis_dots_partial<<<dim3(nb, j + 1), RT, 0, cs>>>(V, n, j + 1, w, n, ops.partial);
      k_reduce_partials<<<j + 1, 32, 0, cs>>>(ops.partial, nb, j + 1, hvals);
      k_basis_sub<<<nb, RT, 0, cs>>>(V, n, j + 1, hvals, w, n, nullptr);
      k_basis_dots_partial<<<dim3(nb, j + 1), RT, 0, cs>>>(V, n, j + 1, w, n, ops.partial);
      k_reduce_partials<<<j + 1, 32, 0, cs>>>(ops.partial, nb, j + 1, hvals + 64);
      k_basis_sub<<<nb, RT, 0, cs>>>(V, n, j + 1, hvals + 64, w, n, ops.partial);
      k_reduce_partials<<<1, 32, 0, cs>>>(ops.partial, nb, 1, hvals + 128);
      k_givens_step<<<1, 32, 0, cs>>>(j, m, hvals, S);
      k_scale_dev<<<nb, RT, 0, cs>>>(w, n, S.scale);
      }
      if (!S.host_res)
        cudaMemcpyAsync(hres + 2 * j, S.res_hn + 2 * j, sizeof(double2) * 2, cudaMemcpyDeviceToHost, cs);
    }
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) {
      h2b_set_error(std::string("h2b_gmres: step capture: ") + cudaGetErrorString(e));
      return H2B_ECUDA;
    }
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      h2b_set_error(std::string("h2b_gmres: step instantiate: ") + cudaGetErrorString(e));
      return H2B_ECUDA;
    }
    h->gmres_graphs.emplace(key, ex);
    *out = ex;
    return H2B_OK;
  };
  TRY(h2b_prepare(h));
  TRY(h2b_ensure_workspace(h, 1));
  std::vector<cudaGraphExec_t> gx(m);
  for (int j = 0; j < m; ++j) TRY(step_graph(j, &gx[j]));
  cudaEvent_t ev[2];
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
  } guard{ev};

  int it = 0, matvecs = 0, nh = 0;
  bool converged = false;
  std::vector<double2> Hh((size_t)(m + 1) * m), gh(m + 1);
  std::vector<cplx> y(m);
  double beta = bnrm;
  while (it < max_iter) {
    if (it > 0) {
      TRY(ops.dots({{r, r}}, true));
      beta = sqrt(g_scratch.host[0].x);
    }
    gh.assign(m + 1, make_double2(0.0, 0.0));
    gh[0] = make_double2(beta, 0.0);
    H2B_CUDA_TRY(cudaMemcpyAsync(S.g, gh.data(), sizeof(double2) * (m + 1), cudaMemcpyHostToDevice, st));
    TRY(ops.lincomb(V, {{cplx(1.0 / beta), r}}, -1));
    // steps run one ahead of the host's convergence check: step j+1 is queued before the host
    // waits for step j's residual.  A speculative step only writes V[j+2], H[:, j+1], g[j+1..j+2]
    // and rotation j+1, none of which the back substitution of a cycle ending at j reads.
    const int it0 = it;
    int j_done = 0;
    H2B_CUDA_TRY(cudaGraphLaunch(gx[0], st));
    H2B_CUDA_TRY(cudaEventRecord(ev[0], st));
    for (int j = 0; j < m; ++j) {
      if (j + 1 < m && it0 + j + 1 < max_iter) {
        H2B_CUDA_TRY(cudaGraphLaunch(gx[j + 1], st));
        H2B_CUDA_TRY(cudaEventRecord(ev[(j + 1) & 1], st));
        ++matvecs;
      }
      H2B_CUDA_TRY(cudaEventSynchronize(ev[j & 1]));
      ++it;
      if (j == 0) ++matvecs;
      const double res = hres[2 * j].x, hn = hres[2 * j + 1].x;
      if (history && nh < max_iter) history[nh] = res;
      ++nh;
      j_done = j + 1;
      if (res <= tol || it >= max_iter || hn == 0.0) break;
    }
    // back substitution on the host (j_done <= 63), x += V y
    H2B_CUDA_TRY(cudaMemcpyAsync(Hh.data(), S.H, sizeof(double2) * (size_t)(m + 1) * m, cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaMemcpyAsync(gh.data(), S.g, sizeof(double2) * (m + 1), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    auto Hc = [&](int i, int l) { return cplx(Hh[(size_t)i * m + l].x, Hh[(size_t)i * m + l].y); };
    for (int i = j_done - 1; i >= 0; --i) {
      cplx acc(gh[i].x, gh[i].y);
      for (int l = i + 1; l < j_done; ++l) acc -= Hc(i, l) * y[l];
      y[i] = acc / Hc(i, i);
    }
    for (int i = 0; i < j_done; ++i) g_scratch.host[i] = make_double2(-y[i].real(), -y[i].imag());
    H2B_CUDA_TRY(cudaMemcpyAsync(hvals, g_scratch.host, sizeof(double2) * j_done, cudaMemcpyHostToDevice, st));
    k_basis_sub<<<ops.nb, RT, 0, st>>>(V, n, j_done, hvals, x, n, nullptr);
    H2B_CHECK_LAUNCH();
    // true residual r = b - A x
    TRY(h2b_run_matvec(h, x, tmp, 1, st));
    ++matvecs;
    TRY(ops.lincomb(r, {{cplx(1.0), b}, {cplx(-1.0), tmp}}, 0));
    TRY(ops.fetch_vals(1));
    const double true_res = sqrt(g_scratch.host[0].x) / bnrm;
    if (true_res <= tol) {
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

// ===========================================================================
// BiCGStab (arith.py:605-689)
// ===========================================================================
// Graph-driven loop: one iteration (two matvecs, three dot launches, the vector updates and
// the scalar kernels above) is ONE CUDA graph; the host queues iteration i+1 before it reads
// iteration i's record, so the GPU never waits for the host.  A speculative iteration after a
// terminal status is a no-op on the vectors (the status is sticky).  Same recurrence, tests and
// order of operations as the host-driven loop below; scalars are numpy-style complex128.
// the host side of the graph-driven loop: one launch of the captured iteration per step, the
// record read one iteration behind
int bicgstab_loop(h2b_ctx* h, cudaGraph_t g, double2* r, double2* rh, double2* p, double2* v, BiSc* sc,
                  int64_t n, int max_iter, const double2* noise, double* history, h2b_report* report,
                  cudaStream_t st, double t0, double2* rec_h, const Scratch& g_scratch) {
  (void)h;
  const int nb = nblocks(n);
  double2* partial = g_scratch.partial;
  double2* vals = g_scratch.vals;
  cudaGraphExec_t gx = nullptr;
  cudaError_t e = cudaGraphInstantiate(&gx, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    h2b_set_error(std::string("h2b_bicgstab: instantiate: ") + cudaGetErrorString(e));
    return H2B_ECUDA;
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct Guard {
    cudaGraphExec_t g;
    cudaEvent_t* e;
    ~Guard() {
      cudaGraphExecDestroy(g);
      if (e[0]) cudaEventDestroy(e[0]);
      if (e[1]) cudaEventDestroy(e[1]);
    }
  } guard{gx, ev};
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  // ---- the loop ----
  int launches = 0;
  auto launch = [&]() -> int {
    H2B_CUDA_TRY(cudaGraphLaunch(gx, st));
    H2B_CUDA_TRY(cudaEventRecord(ev[launches & 1], st));
    ++launches;
    return H2B_OK;
  };
  int it = 0, matvecs = 0, nh = 0;
  bool converged = false, restarted = false;
  TRY(launch());
  int obs = 0;  // launch index of the iteration observed next
  while (true) {
    ++it;
    if (it < max_iter) TRY(launch());  // speculative next iteration
    H2B_CUDA_TRY(cudaEventSynchronize(ev[obs & 1]));
    const double2* slot = rec_h + 2 * ((obs + 1) & 1);
    const int status = (int)slot[0].x;
    if ((int)slot[0].y != obs + 1) {
      h2b_set_error("h2b_bicgstab: iteration record out of sequence");
      return H2B_ECUDA;
    }
    const double hs = slot[1].x, hr = slot[1].y;
    auto push = [&](double val) {
      if (history && nh < max_iter) history[nh] = val;
      ++nh;
    };
    bool stop = true;
    if (status == BI_RUN) {
      push(hr);
      matvecs += 2;
      stop = it >= max_iter;
      obs += 1;
    } else if (status == BI_CONV_R) {
      push(hr);
      matvecs += 2;
      converged = true;
    } else if (status == BI_CONV_S || status == BI_CONV_S_DONE) {
      push(hs);
      matvecs += 1;
      converged = true;
    } else if (status == BI_NONFINITE) {
      push(hr);
      matvecs += 2;
    } else if (status == BI_DENOM_ZERO) {
      matvecs += 1;
    } else if (status == BI_OMEGA_ZERO) {
      matvecs += 2;
    } else if (status == BI_RHO_BREAK && !restarted && noise) {
      // restart once (the reference re-seeds the shadow residual) and redo this iteration
      Ops ops{st, n, nb, partial, vals, g_scratch.host};
      TRY(ops.lincomb(rh, {{cplx(1.0), r}, {cplx(1.0), noise}}, -1));
      H2B_CUDA_TRY(cudaMemsetAsync(v, 0, sizeof(double2) * n, st));
      H2B_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double2) * n, st));
      k_bi_restart<<<1, 1, 0, st>>>(sc);
      H2B_CHECK_LAUNCH();
      restarted = true;
      --it;
      TRY(launch());
      obs = launches - 1;
      stop = false;
    }
    if (stop) break;
  }
  H2B_CUDA_TRY(cudaStreamSynchronize(st));
  report->iterations = it;
  report->converged = converged ? 1 : 0;
  report->n_history = nh < max_iter ? nh : max_iter;
  report->matvecs = matvecs;
  report->wall_time = now_s() - t0;
  return H2B_OK;
}

int bicgstab_graph(h2b_ctx* h, const Scratch& g_scratch, const double2* b, double2* x, double2* r, double2* rh, double2* p,
                   double2* v, double2* s, double2* t, BiSc* sc, double bnrm, double tol, int max_iter,
                   const double2* noise, double* history, h2b_report* report, cudaStream_t st,
                   double t0) {
  const int64_t n = h->n;
  const int nb = nblocks(n);
  double2* partial = g_scratch.partial;
  double2* vals = g_scratch.vals;
  double2* rec_h = g_scratch.host + SCR_BICG;  // pinned, mapped: two records of two double2
  double2* rec = nullptr;
  H2B_CUDA_TRY(cudaHostGetDevicePointer((void**)&rec, rec_h, 0));
  {
    BiSc init{};
    init.rho = init.alpha = init.omega = make_double2(1.0, 0.0);
    init.p_zero = 1;
    H2B_CUDA_TRY(cudaMemcpyAsync(sc, &init, sizeof(BiSc), cudaMemcpyHostToDevice, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));  // `init` leaves scope
  }
  const double eps = 2.220446049250313e-16;
  const double thr = eps * eps * std::max(1.0, bnrm * bnrm);
  TRY(h2b_prepare(h));  // streams, events and the matvec workspace exist before the capture
  TRY(h2b_ensure_workspace(h, 1));
  // ---- capture one iteration ----
  cudaStream_t cs = nullptr;
  H2B_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  H2B_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  auto dots = [&](std::initializer_list<std::pair<const double2*, const double2*>> pairs) {
    DotPairs d;
    d.np = 0;
    for (auto& pr : pairs) {
      d.a[d.np] = pr.first;
      d.b[d.np] = pr.second;
      ++d.np;
    }
    k_dots_partial<<<nb, RT, 0, cs>>>(d, n, partial);
    k_reduce_partials<<<d.np, 32, 0, cs>>>(partial, nb, d.np, vals);
  };
  int nl = 0;
  // small n: the three vector segments as single cluster launches (k_bicg_segment)
  int seg_cl = 0;
  if (!getenv("H2B_BICG_UNFUSED") && n <= 16384) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(AC_T);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaFuncSetAttribute(k_bicg_segment, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaOccupancyMaxActiveClusters(&ncl, k_bicg_segment, &cfg) == cudaSuccess && ncl >= 1)
      seg_cl = 16;
    cudaGetLastError();
  }
  if (seg_cl) {
    BiSegArgs sa{sc, rh, r, p, v, s, t, x, n, (int)((n + seg_cl - 1) / seg_cl), thr, bnrm, tol, rec};
    auto seg = [&](int k) -> int {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(seg_cl);
      cfg.blockDim = dim3(AC_T);
      cfg.stream = cs;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = seg_cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, k_bicg_segment, sa, k) != cudaSuccess) {
        h2b_set_error("h2b_bicgstab: fused segment launch failed");
        return H2B_ECUDA;
      }
      return H2B_OK;
    };
    int rc = seg(0);
    if (!rc) rc = h2b_enqueue_matvec(h, p, v, 1, cs, &nl);
    if (!rc) rc = seg(1);
    if (!rc) rc = h2b_enqueue_matvec(h, s, t, 1, cs, &nl);
    if (!rc) rc = seg(2);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) {
      h2b_set_error(std::string("h2b_bicgstab: capture: ") + cudaGetErrorString(e));
      return H2B_ECUDA;
    }
    return bicgstab_loop(h, g, r, rh, p, v, sc, n, max_iter, noise, history, report, st, t0, rec_h, g_scratch);
  }
  dots({{rh, r}});                                                             // rho_new
  k_bi_rho<<<1, 1, 0, cs>>>(sc, vals, thr);
  k_lincomb_dev<<<nb, RT, 0, cs>>>(sc, BI_RUN, sc->cp, 3, r, p, v, p, n, nullptr);  // p
  int rc = h2b_enqueue_matvec(h, p, v, 1, cs, &nl);                            // v = A p
  if (!rc) {
    dots({{rh, v}});
    k_bi_alpha<<<1, 1, 0, cs>>>(sc, vals);
    k_lincomb_dev<<<nb, RT, 0, cs>>>(sc, BI_RUN, sc->cs, 2, r, v, nullptr, s, n, partial);  // s
    k_reduce_partials<<<1, 32, 0, cs>>>(partial, nb, 1, vals);
    k_bi_snorm<<<1, 1, 0, cs>>>(sc, vals, bnrm, tol);
    k_lincomb_dev<<<nb, RT, 0, cs>>>(sc, BI_CONV_S, sc->cx, 2, x, p, nullptr, x, n, nullptr);
    k_bi_mark<<<1, 1, 0, cs>>>(sc, BI_CONV_S, BI_CONV_S_DONE);
    rc = h2b_enqueue_matvec(h, s, t, 1, cs, &nl);                              // t = A s
  }
  if (!rc) {
    dots({{t, t}, {t, s}});
    k_bi_omega<<<1, 1, 0, cs>>>(sc, vals);
    k_lincomb_dev<<<nb, RT, 0, cs>>>(sc, BI_RUN, sc->cx, 3, x, p, s, x, n, nullptr);    // x
    k_lincomb_dev<<<nb, RT, 0, cs>>>(sc, BI_RUN, sc->cr, 2, s, t, nullptr, r, n, partial);  // r
    k_reduce_partials<<<1, 32, 0, cs>>>(partial, nb, 1, vals);
    k_bi_final<<<1, 1, 0, cs>>>(sc, vals, bnrm, tol, rec);
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) {
    h2b_set_error(std::string("h2b_bicgstab: capture: ") + cudaGetErrorString(e));
    return H2B_ECUDA;
  }
  return bicgstab_loop(h, g, r, rh, p, v, sc, n, max_iter, noise, history, report, st, t0, rec_h, g_scratch);
}

extern "C" int h2b_bicgstab(h2b_handle h, const void* b_perm, void* x_perm, double tol, int max_iter,
                            const void* shadow_perm, const void* restart_noise_perm, double* history,
                            h2b_report* report, void* stream) {
  if (!h || !b_perm || !x_perm || !report) {
    h2b_set_error("h2b_bicgstab: null argument");
    return H2B_EINVAL;
  }
  if (!(tol > 0.0 && tol < 1.0)) {
    h2b_set_error("tol must be in (0, 1)");
    return H2B_EINVAL;
  }
  if (max_iter < 1) {
    h2b_set_error("max_iter must be >= 1");
    return H2B_EINVAL;
  }
  const double t0 = now_s();
  Scratch g_scratch;
  TRY(handle_scratch(h, &g_scratch));
  cudaStream_t st = (cudaStream_t)stream;
  TRY(h2b_order_begin(h, st));
  struct OrderEnd {
    h2b_ctx* h;
    cudaStream_t st;
    ~OrderEnd() { h2b_order_end(h, st); }
  } order_end{h, st};
  const int64_t n = h->n;
  double2* ws = nullptr;
  TRY(krylov_ws(h, sizeof(double2) * (size_t)n * 6 + sizeof(BiSc), &ws));
  double2 *r = ws, *rh = ws + n, *p = ws + 2 * n, *v = ws + 3 * n, *s = ws + 4 * n, *t = ws + 5 * n;
  BiSc* sc = reinterpret_cast<BiSc*>(ws + 6 * n);
  const double2* b = (const double2*)b_perm;
  double2* x = (double2*)x_perm;
  Ops ops{st, n, nblocks(n), g_scratch.partial, g_scratch.vals, g_scratch.host};
  auto H = [&](int i) { return cplx(g_scratch.host[i].x, g_scratch.host[i].y); };
  *report = h2b_report{0, 0, 0, 0, 0.0};

  TRY(ops.dots({{b, b}}, true));
  const double bnrm = sqrt(H(0).real());
  H2B_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
  if (bnrm == 0.0) {
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    report->converged = 1;
    report->wall_time = now_s() - t0;
    return H2B_OK;
  }
  H2B_CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
  H2B_CUDA_TRY(cudaMemcpyAsync(rh, shadow_perm ? shadow_perm : b, sizeof(double2) * n,
                               cudaMemcpyDeviceToDevice, st));
  H2B_CUDA_TRY(cudaMemsetAsync(v, 0, sizeof(double2) * n, st));
  H2B_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double2) * n, st));
  if (!getenv("H2B_BICG_HOST"))  // H2B_BICG_HOST: the host-driven loop below (A/B timing)
    return bicgstab_graph(h, g_scratch, b, x, r, rh, p, v, s, t, sc, bnrm, tol, max_iter,
                          (const double2*)restart_noise_perm, history, report, st, t0);
  cplx rho = 1.0, alpha = 1.0, omega = 1.0;
  bool converged = false, restarted = false, p_zero = true;
  int it = 0, matvecs = 0, nh = 0;
  const double eps = 2.220446049250313e-16;
  const double breakdown = eps * eps;
  while (it < max_iter) {
    ++it;
    TRY(ops.dots({{rh, r}}, true));
    cplx rho_new = H(0);
    if (std::abs(rho_new) < breakdown * std::max(1.0, bnrm * bnrm)) {
      if (restarted || !restart_noise_perm) break;
      TRY(ops.lincomb(rh, {{cplx(1.0), r}, {cplx(1.0), (const double2*)restart_noise_perm}}, -1));
      rho = alpha = omega = 1.0;
      H2B_CUDA_TRY(cudaMemsetAsync(v, 0, sizeof(double2) * n, st));
      H2B_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double2) * n, st));
      p_zero = true;
      restarted = true;
      TRY(ops.dots({{rh, r}}, true));
      rho_new = H(0);
      if (std::abs(rho_new) < breakdown * std::max(1.0, bnrm * bnrm)) break;
    }
    if (it == 1 || p_zero) {
      H2B_CUDA_TRY(cudaMemcpyAsync(p, r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
      p_zero = false;
    } else {
      const cplx beta = (rho_new / rho) * (alpha / omega);
      TRY(ops.lincomb(p, {{cplx(1.0), r}, {beta, p}, {-beta * omega, v}}, -1));
    }
    TRY(h2b_run_matvec(h, p, v, 1, st));
    ++matvecs;
    TRY(ops.dots({{rh, v}}, true));
    const cplx denom = H(0);
    if (denom == cplx(0)) break;
    alpha = rho_new / denom;
    TRY(ops.lincomb(s, {{cplx(1.0), r}, {-alpha, v}}, 0));
    TRY(ops.fetch_vals(1));
    const double s_nrm = sqrt(H(0).real());
    if (s_nrm / bnrm <= tol) {
      TRY(ops.lincomb(x, {{cplx(1.0), x}, {alpha, p}}, -1));
      if (history && nh < max_iter) history[nh] = s_nrm / bnrm;
      ++nh;
      converged = true;
      break;
    }
    TRY(h2b_run_matvec(h, s, t, 1, st));
    ++matvecs;
    TRY(ops.dots({{t, t}, {t, s}}, true));
    const double tt = H(0).real();
    if (tt == 0.0) break;
    omega = H(1) / tt;
    if (omega == cplx(0)) break;
    TRY(ops.lincomb(x, {{cplx(1.0), x}, {alpha, p}, {omega, s}}, -1));
    TRY(ops.lincomb(r, {{cplx(1.0), s}, {-omega, t}}, 0));
    TRY(ops.fetch_vals(1));
    rho = rho_new;
    const double rel = sqrt(H(0).real()) / bnrm;
    if (history && nh < max_iter) history[nh] = rel;
    ++nh;
    if (rel <= tol) {
      converged = true;
      break;
    }
    if (!std::isfinite(rel)) break;
  }
  H2B_CUDA_TRY(cudaStreamSynchronize(st));
  report->iterations = it;
  report->converged = converged ? 1 : 0;
  report->n_history = nh < max_iter ? nh : max_iter;
  report->matvecs = matvecs;
  report->wall_time = now_s() - t0;
  return H2B_OK;
}

// ===========================================================================
// building blocks of the row-distributed GMRES (paper_1703_01175_b200/dist.py): the same device
// Givens recurrence as h2b_gmres, on a caller-owned state, plus the normalisation by a device
// scalar — the host never reads a vector element between steps
// ===========================================================================
extern "C" int64_t h2b_gmres_state_elems(int m) {
  return (int64_t)(m + 1) * m + (m + 1) + 3 * (int64_t)m + 2;
}

extern "C" int h2b_gmres_givens(void* state, int m, int j, const void* hvals_dev, double* host_res,
                                void* stream) {
  if (!state || !hvals_dev || m < 1 || m > 63 || j < 0 || j >= m) {
    h2b_set_error("h2b_gmres_givens: bad arguments (need 1 <= m <= 63, 0 <= j < m)");
    return H2B_EINVAL;
  }
  double2* base = (double2*)state;
  GivensState S;
  S.H = base;
  S.g = S.H + (size_t)(m + 1) * m;
  S.cs_sn = S.g + (m + 1);
  S.res_hn = S.cs_sn + m;
  S.scale = S.res_hn + m + m;
  S.bnrm = S.scale + 1;
  S.host_res = nullptr;
  if (host_res) {
    double2* d = nullptr;
    if (cudaHostGetDevicePointer((void**)&d, host_res, 0) != cudaSuccess) {
      cudaGetLastError();
      h2b_set_error("h2b_gmres_givens: host_res is not mapped pinned memory");
      return H2B_EINVAL;
    }
    S.host_res = d;  // records {res_j, 0}, {hn_j, 0} at 2j, 2j + 1
  }
  k_givens_step<<<1, 32, 0, (cudaStream_t)stream>>>(j, m, (const double2*)hvals_dev, S);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

extern "C" int h2b_zscale_dev(void* w, int64_t n, const void* scale_dev, void* stream) {
  if (!w || !scale_dev || n < 0) {
    h2b_set_error("h2b_zscale_dev: bad arguments");
    return H2B_EINVAL;
  }
  k_scale_dev<<<nblocks(n), RT, 0, (cudaStream_t)stream>>>((double2*)w, n, (const double2*)scale_dev);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}
