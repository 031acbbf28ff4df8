// Multi-RHS H² matvec (q >= H2B_MRHS_MIN columns) on the FP64 tensor pipe (DMMA).
//
// Reference: arith.matmat_apply (/root/reference/pkg/src/h2vie/arith.py:120-130),
// i.e. every phase of _apply_perm (arith.py:52-104) applied to an (n, q) block.
// With q columns every block product of the matvec is a small dense complex GEMM
// (arithmetic intensity ~q/2 flop/B: FP64-compute-bound at q = 64), so all
// phases run through ONE kernel, a grouped complex GEMM on `mma.sync.m8n8k4.f64`
// (SASS DMMA.8x8x4; on B200 the DMMA and DFMA pipes both peak at ~37 TFLOP/s,
// tools/micro/dmma_bench.cu, but DMMA needs 8x fewer issue slots and operand
// loads per flop, so it is the one that can be fed from shared memory):
//
//   item:  C[c_row + i, col0 + c] (+)= Σ_seg A_seg[i, :] · B_seg[:, col0 + c],
//          i < m <= 64, c < 64 (one column tile of the q columns)
//   seg:   A (m x k, k <= 32) read from V, Vᵀ, Tᵀ, T, Sᵀ-panels or D (row-major or
//          transposed view), B = k rows of x, x̂ or ŷ (contiguous or gathered)
//
// Phases (one launch each, serialised on the stream; each saturates the GPU):
//   up      x̂_c = V_cᵀ x_c ; x̂_t = [T_lo;T_hi]ᵀ [x̂_lo; x̂_hi]      (arith.py:58-71)
//   couple  ŷ_t = Σ_s S^{t,s} x̂_s                                    (arith.py:72-81)
//   down    [ŷ_lo; ŷ_hi] += [T_lo; T_hi] ŷ_t                          (arith.py:82-97)
//   near    y_t = Σ_s D_{t,s} x_s + V_t ŷ_t   (near-field + leaf back) (arith.py:98-104)
//
// Complex arithmetic as a real GEMM of twice the size: C_r (2m x q) = A_r (2m x 2k) B_r
// (2k x q) with A_r[2i+a][2j+b] = {re, -im; im, re}[a][b] of A[i][j], B_r[2j+b][c] =
// {re, im}[b] of B[j][c], C_r[2i+a][c] = {re, im}[a] of C[i][c].  A and B stay in their
// interleaved complex layout in shared memory; each lane's fragment load picks re/im and
// flips the sign bit (lane-constant), so no real expansion is ever stored.
#include <algorithm>
#include <vector>

#include "h2b_common.cuh"

namespace {

constexpr int MM_THREADS = 256;  // 8 warps: 4 (rows of C_r) x 2 (columns)
constexpr int MM_M = 64;         // complex rows per item
constexpr int MM_N = 64;         // complex columns per tile
constexpr int MM_K = 32;         // complex K per stage
constexpr int MM_AST = 34;       // A row stride (complex): 68 doubles -> conflict-free fragments
constexpr int MM_STAGES = 3;
constexpr int MM_A_ELEMS = MM_M * MM_AST;
constexpr int MM_B_ELEMS = MM_K * MM_N;
constexpr int MM_STAGE_ELEMS = MM_A_ELEMS + MM_B_ELEMS;
constexpr int MM_SMEM = 16 * MM_STAGES * MM_STAGE_ELEMS;  // 202752 bytes

enum : int32_t { A_V = 0, A_T, A_S, A_D, A_VT, A_TT, A_N };
enum : int32_t { B_X = 0, B_XHAT, B_YHAT, B_N };
constexpr int SEG_TRANS = 1 << 8;   // A[i][j] = src[a_off + j*lda + i]
constexpr int SEG_GATHER = 1 << 9;  // B row r = gather[b_row + r]
constexpr int ITEM_ACC = 1 << 8;

struct MmSeg {
  int64_t a_off;   // element offset of A(0,0) in its source
  int64_t b_row;   // first B row (or first gather index)
  int32_t k, lda;  // K extent (<= MM_K), leading dimension of the source
  int32_t flags;   // a_src | b_src << 4 | SEG_TRANS | SEG_GATHER
  int32_t pad;
};
struct MmItem {
  int64_t c_row;     // first output row
  int32_t m;         // rows (<= MM_M)
  int32_t seg0, nseg;
  int32_t flags;     // c_dst (B_* ids) | ITEM_ACC
  int64_t pad;
};
struct MmBufs {
  const double2* a[A_N];
  double2* b[B_N];   // also the destinations (x̂, ŷ; y passed separately)
  double2* y;
  const int32_t* gather;
};

// buffer selection by id without dynamic indexing of the parameter block (which would spill it
// to local memory)
__device__ __forceinline__ const double2* pick_a(const MmBufs& bf, int id) {
  const double2* p = bf.a[0];
#pragma unroll
  for (int i = 1; i < A_N; ++i) p = id == i ? bf.a[i] : p;
  return p;
}
__device__ __forceinline__ double2* pick_b(const MmBufs& bf, int id) {
  double2* p = bf.b[0];
#pragma unroll
  for (int i = 1; i < B_N; ++i) p = id == i ? bf.b[i] : p;
  return id == B_N ? bf.y : p;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// stage one K-chunk (segment) into shared memory: A -> [MM_M][MM_AST], B -> [MM_K][MM_N]
__device__ __forceinline__ void stage_seg(const MmSeg& s, const MmBufs& bf, int m, int q, int col0,
                                          double2* st) {
  const uint32_t sa = smem_u32(st), sb = smem_u32(st + MM_A_ELEMS);
  const double2* A = pick_a(bf, s.flags & 15);
  const double2* B = pick_b(bf, (s.flags >> 4) & 15);
  const bool trans = s.flags & SEG_TRANS;
  // A: 64 x 32 complex
#pragma unroll
  for (int u = 0; u < (MM_M * MM_K) / MM_THREADS; ++u) {
    const int e = threadIdx.x + u * MM_THREADS;
    int i, j;
    if (trans) { i = e & (MM_M - 1); j = e >> 6; }  // consecutive threads: consecutive i (coalesced)
    else { j = e & (MM_K - 1); i = e >> 5; }
    const bool ok = i < m && j < s.k;
    const double2* src = A + s.a_off + (trans ? (int64_t)j * s.lda + i : (int64_t)i * s.lda + j);
    cp_async16(sa + 16 * (i * MM_AST + j), ok ? src : A, ok ? 16 : 0);
  }
  // B: 32 rows x 64 columns
#pragma unroll
  for (int u = 0; u < (MM_K * MM_N) / MM_THREADS; ++u) {
    const int e = threadIdx.x + u * MM_THREADS;
    const int c = e & (MM_N - 1), r = e >> 6;
    const bool ok = r < s.k && col0 + c < q;
    int64_t row = 0;
    if (ok) row = (s.flags & SEG_GATHER) ? (int64_t)__ldg(bf.gather + s.b_row + r) : s.b_row + r;
    const double2* src = B + row * q + col0 + c;
    cp_async16(sb + 16 * (r * MM_N + c), ok ? src : B, ok ? 16 : 0);
  }
}

__global__ void __launch_bounds__(MM_THREADS, 1) k_zgemm_grouped(const MmItem* __restrict__ items,
                                                                 const MmSeg* __restrict__ segs,
                                                                 MmBufs bf, int q) {
  extern __shared__ __align__(16) double2 sm[];
  const MmItem it = items[blockIdx.x];
  const int col0 = blockIdx.y * MM_N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 3, wn = warp >> 2;
  // lane-constant fragment geometry
  const int fr = lane >> 2, kk = lane & 3;
  const int b = kk & 1, jo = kk >> 1;
  // A fragment of m-tile mt: C_r row R = wm*32 + mt*8 + fr -> complex row i = R>>1, part a = R&1
  const int a = fr & 1;
  const int a_pick = a ^ b;                                           // 0: re, 1: im
  const unsigned long long a_neg = (a == 0 && b == 1) ? 0x8000000000000000ull : 0ull;  // -im
  int a_base[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) a_base[mt] = (((wm * 32 + mt * 8 + fr) >> 1) * MM_AST) * 2 + a_pick;
  int b_base[4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) b_base[nt] = (wn * 32 + nt * 8 + fr) * 2 + b;

  double acc[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  const int ns = it.nseg;
  // prologue: stages 0 .. MM_STAGES-2
#pragma unroll
  for (int s = 0; s < MM_STAGES - 1; ++s) {
    if (s < ns) stage_seg(segs[it.seg0 + s], bf, it.m, q, col0, sm + s * MM_STAGE_ELEMS);
    cp_commit();
  }
  for (int s = 0; s < ns; ++s) {
    cp_wait<MM_STAGES - 2>();
    __syncthreads();  // stage s visible to all; stage s-1 no longer read by anyone
    {
      const int sn = s + MM_STAGES - 1;
      if (sn < ns) stage_seg(segs[it.seg0 + sn], bf, it.m, q, col0, sm + (sn % MM_STAGES) * MM_STAGE_ELEMS);
      cp_commit();
    }
    const double* As = reinterpret_cast<const double*>(sm + (s % MM_STAGES) * MM_STAGE_ELEMS);
    const double* Bs = As + 2 * MM_A_ELEMS;
#pragma unroll 4
    for (int ks = 0; ks < (2 * MM_K) / 4; ++ks) {
      const int j = ks * 2 + jo;  // complex K index of this lane
      double af[4], bfr[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        af[mt] = __longlong_as_double(__double_as_longlong(As[a_base[mt] + 2 * j]) ^ a_neg);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bfr[nt] = Bs[j * (2 * MM_N) + b_base[nt]];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bfr[nt]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // epilogue: C_r fragments -> complex tile in shared memory -> global (coalesced)
  double* Cs = reinterpret_cast<double*>(sm);
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int R = wm * 32 + mt * 8 + fr;
    const int i = R >> 1, part = R & 1;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int c = wn * 32 + nt * 8 + 2 * kk;
      Cs[(i * MM_N + c) * 2 + part] = acc[mt][nt][0];
      Cs[(i * MM_N + c + 1) * 2 + part] = acc[mt][nt][1];
    }
  }
  __syncthreads();
  const int dst_id = it.flags & 15;
  double2* C = pick_b(bf, dst_id);
  const bool accum = it.flags & ITEM_ACC;
  const double2* Ct = reinterpret_cast<const double2*>(sm);
  for (int e = threadIdx.x; e < it.m * MM_N; e += MM_THREADS) {
    const int i = e >> 6, c = e & (MM_N - 1);
    if (col0 + c >= q) continue;
    double2* o = C + (it.c_row + i) * q + col0 + c;
    const double2 v = Ct[i * MM_N + c];
    *o = accum ? cadd(*o, v) : v;
  }
}

// q = 1: the same item / segment lists as a grouped complex GEMV on the CUDA cores
// (memory-bound).  Thread (row i, quarter g) accumulates 8 K-entries of each segment; the four
// partial sums of a row are combined in a fixed order (deterministic).
constexpr int MV_THREADS = 256;
__global__ void __launch_bounds__(MV_THREADS) k_zgemv_grouped(const MmItem* __restrict__ items,
                                                              const MmSeg* __restrict__ segs,
                                                              MmBufs bf) {
  __shared__ double2 red[4][MM_M];
  const MmItem it = items[blockIdx.x];
  double2 acc = make_double2(0.0, 0.0);
  for (int sgi = 0; sgi < it.nseg; ++sgi) {
    const MmSeg s = segs[it.seg0 + sgi];
    const double2* A = pick_a(bf, s.flags & 15) + s.a_off;
    const double2* B = pick_b(bf, (s.flags >> 4) & 15);
    const bool gather = s.flags & SEG_GATHER;
    int i, g;
    if (s.flags & SEG_TRANS) { i = threadIdx.x & (MM_M - 1); g = threadIdx.x >> 6; }
    else { i = threadIdx.x >> 2; g = threadIdx.x & 3; }
    if (i < it.m) {
      const int j0 = g * 8, j1 = min(s.k, j0 + 8);
      double2 av[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        if (j < j1) {
          av[u] = (s.flags & SEG_TRANS) ? A[(int64_t)j * s.lda + i] : A[(int64_t)i * s.lda + j];
          const int64_t row = gather ? (int64_t)__ldg(bf.gather + s.b_row + j) : s.b_row + j;
          xv[u] = B[row];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < j1) cfma(acc, av[u], xv[u]);
    }
  }
  // all segments of an item share the A orientation (checked by h2b_plan_set_phase), so the
  // thread's (row, quarter) is the same for every segment
  int i, g;
  if (it.nseg > 0 && (segs[it.seg0].flags & SEG_TRANS)) { i = threadIdx.x & (MM_M - 1); g = threadIdx.x >> 6; }
  else { i = threadIdx.x >> 2; g = threadIdx.x & 3; }
  red[g][i] = acc;
  __syncthreads();
  if (threadIdx.x < it.m) {
    const int r = threadIdx.x;
    const double2 v = cadd(cadd(red[0][r], red[1][r]), cadd(red[2][r], red[3][r]));
    double2* o = pick_b(bf, it.flags & 15) + it.c_row + r;
    *o = (it.flags & ITEM_ACC) ? cadd(*o, v) : v;
  }
}

int run_grouped(const MmItem* items, int n_items, const MmSeg* segs, const MmBufs& bf, int q,
                cudaStream_t st, int* nl) {
  const int nct = (q + MM_N - 1) / MM_N;
  for (int i0 = 0; i0 < n_items; i0 += 65535) {
    const int cnt = std::min(65535, n_items - i0);
    if (q == 1)
      k_zgemv_grouped<<<cnt, MV_THREADS, 0, st>>>(items + i0, segs, bf);
    else
      k_zgemm_grouped<<<dim3(cnt, nct), MM_THREADS, MM_SMEM, st>>>(items + i0, segs, bf, q);
    H2B_CHECK_LAUNCH();
    ++*nl;
  }
  return H2B_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// host: plan (item / segment lists per phase) and launch
// ---------------------------------------------------------------------------
struct MrhsPlan {
  std::vector<int2> launches;  // {item_first, n_items} in execution order
  MmItem* items = nullptr;
  MmSeg* segs = nullptr;
  int64_t flops_q1 = 0;        // useful real flops per column (for reporting)
};

namespace {

struct Builder {
  std::vector<MmItem> items;
  std::vector<MmSeg> segs;
  std::vector<int2> launches;
  int launch_first = 0;
  // one logical segment, split into K-chunks of MM_K
  void seg(int a_src, int64_t a_off, int lda, bool trans, int m0, int k, int b_src, int64_t b_row,
           bool gather) {
    for (int k0 = 0; k0 < k; k0 += MM_K) {
      MmSeg s{};
      s.a_off = a_off + (trans ? (int64_t)k0 * lda + m0 : (int64_t)m0 * lda + k0);
      s.b_row = b_row + k0;
      s.k = std::min(MM_K, k - k0);
      s.lda = lda;
      s.flags = a_src | (b_src << 4) | (trans ? SEG_TRANS : 0) | (gather ? SEG_GATHER : 0);
      segs.push_back(s);
    }
  }
  int begin_item() { return (int)segs.size(); }
  void end_item(int seg0, int64_t c_row, int m, int dst, bool acc) {
    MmItem it{};
    it.c_row = c_row;
    it.m = m;
    it.seg0 = seg0;
    it.nseg = (int)segs.size() - seg0;
    it.flags = dst | (acc ? ITEM_ACC : 0);
    items.push_back(it);
  }
  void end_launch() {
    const int n = (int)items.size() - launch_first;
    if (n > 0) launches.push_back(int2{launch_first, n});
    launch_first = (int)items.size();
  }
};

}  // namespace

int h2b_mrhs_prepare(h2b_ctx* h) {
  if (h->mrhs) return H2B_OK;
  Builder B;
  const int P = h->P;
  // up: deepest level first (h->up_levels), V_cᵀ x_c / [T_lo;T_hi]ᵀ x̂_children via Vᵀ, Tᵀ
  for (int l : h->up_levels) {
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) {
      const int k = h->c_rank[p];
      if (k == 0) continue;
      const int lo = h->c_child_lo[p];
      for (int m0 = 0; m0 < k; m0 += MM_M) {
        const int m = std::min(MM_M, k - m0);
        const int s0 = B.begin_item();
        if (lo < 0) {
          B.seg(A_VT, h->c_voff[p], h->c_size[p], false, m0, h->c_size[p], B_X, h->c_start[p], false);
        } else {
          const int kc = h->c_rank[lo] + h->c_rank[h->c_child_hi[p]];
          if (kc > 0) B.seg(A_TT, h->c_toff[p], kc, false, m0, kc, B_XHAT, h->c_xoff[lo], false);
        }
        B.end_item(s0, h->c_xoff[p] + m0, m, B_XHAT, false);
      }
    }
    B.end_launch();
  }
  // coupling: every target with k > 0 (zero ŷ_t when it has no admissible partner);
  // the device copy of S holds per-target transposed panels (Σ k_s) x k_t
  std::vector<int64_t> prow_h(P + 1, 0);
  {
    int64_t r = 0;
    for (int t = 0; t < P; ++t) {
      prow_h[t] = r;
      if (h->c_rank[t] == 0) continue;
      for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) r += h->c_rank[h->s_col[b]];
    }
    prow_h[P] = r;
  }
  for (int t = 0; t < P; ++t) {
    const int kt = h->c_rank[t];
    if (kt == 0) continue;
    const int64_t b0 = h->s_row_ptr[t], b1 = h->s_row_ptr[t + 1];
    const int R = (int)(prow_h[t + 1] - prow_h[t]);
    for (int m0 = 0; m0 < kt; m0 += MM_M) {
      const int s0 = B.begin_item();
      if (R > 0) B.seg(A_S, h->s_off[b0], kt, true, m0, R, B_XHAT, prow_h[t], true);
      B.end_item(s0, h->c_xoff[t] + m0, std::min(MM_M, kt - m0), B_YHAT, false);
    }
    (void)b1;
  }
  B.end_launch();
  // down: root first, children rows [lo; hi] += T ŷ_t
  for (int l : h->down_levels) {
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) {
      const int k = h->c_rank[p];
      const int lo = h->c_child_lo[p];
      if (k == 0 || lo < 0) continue;
      const int mc = h->c_rank[lo] + h->c_rank[h->c_child_hi[p]];
      for (int m0 = 0; m0 < mc; m0 += MM_M) {
        const int s0 = B.begin_item();
        B.seg(A_T, h->c_toff[p], k, false, m0, k, B_YHAT, h->c_xoff[p], false);
        B.end_item(s0, h->c_xoff[lo] + m0, std::min(MM_M, mc - m0), B_YHAT, true);
      }
    }
    B.end_launch();
  }
  // near-field + leaf back-transform, one item per (leaf, 64-row chunk): y overwritten
  for (int t : h->h_leaves) {
    const int nt = h->c_size[t];
    for (int m0 = 0; m0 < nt; m0 += MM_M) {
      const int s0 = B.begin_item();
      for (int64_t b = h->d_row_ptr[t]; b < h->d_row_ptr[t + 1]; ++b) {
        const int s = h->d_col[b];
        B.seg(A_D, h->d_off[b], h->c_size[s], false, m0, h->c_size[s], B_X, h->c_start[s], false);
      }
      if (h->c_rank[t] > 0)
        B.seg(A_V, h->c_voff[t], h->c_rank[t], false, m0, h->c_rank[t], B_YHAT, h->c_xoff[t], false);
      B.end_item(s0, h->c_start[t] + m0, std::min(MM_M, nt - m0), B_N, false);
    }
  }
  B.end_launch();

  auto* plan = new MrhsPlan();
  plan->launches = B.launches;
  int64_t acc = 0;
  const size_t bi = sizeof(MmItem) * std::max<size_t>(B.items.size(), 1);
  const size_t bs = sizeof(MmSeg) * std::max<size_t>(B.segs.size(), 1);
  cudaError_t e1 = cudaMalloc(&plan->items, bi), e2 = cudaMalloc(&plan->segs, bs);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaFree(plan->items);
    cudaFree(plan->segs);
    delete plan;
    cudaGetLastError();
    h2b_set_error("multi-RHS plan: device allocation failed");
    return H2B_ENOMEM;
  }
  if (!B.items.empty()) H2B_CUDA_TRY(cudaMemcpy(plan->items, B.items.data(), sizeof(MmItem) * B.items.size(), cudaMemcpyHostToDevice));
  if (!B.segs.empty()) H2B_CUDA_TRY(cudaMemcpy(plan->segs, B.segs.data(), sizeof(MmSeg) * B.segs.size(), cudaMemcpyHostToDevice));
  acc += bi + bs;
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_zgemm_grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, MM_SMEM));
  h->mrhs = plan;
  h->device_bytes += acc;
  return H2B_OK;
}

void h2b_mrhs_free(h2b_ctx* h) {
  if (!h->mrhs) return;
  cudaFree(h->mrhs->items);
  cudaFree(h->mrhs->segs);
  delete h->mrhs;
  h->mrhs = nullptr;
}

int h2b_mrhs_launches(const h2b_ctx* h) { return h->mrhs ? (int)h->mrhs->launches.size() : 0; }

int h2b_launch_mrhs(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl) {
  H2B_TRY(h2b_mrhs_prepare(h));
  MmBufs bf{};
  bf.a[A_V] = h->buf[H2B_SEC_V];
  bf.a[A_T] = h->buf[H2B_SEC_T];
  bf.a[A_S] = h->buf[H2B_SEC_S];
  bf.a[A_D] = h->buf[H2B_SEC_D];
  bf.a[A_VT] = h->vT;
  bf.a[A_TT] = h->tT;
  bf.b[B_X] = const_cast<double2*>(xp);
  bf.b[B_XHAT] = h->xhat;
  bf.b[B_YHAT] = h->yhat;
  bf.y = yp;
  bf.gather = h->s_xcol;
  for (const int2& L : h->mrhs->launches)
    H2B_TRY(run_grouped(h->mrhs->items + L.x, L.y, h->mrhs->segs, bf, q, st, nl));
  return H2B_OK;
}

// ---------------------------------------------------------------------------
// generic plan handles (C-ABI h2b_plan_*): payloads + per-phase item/segment lists built by
// the host (paper_1703_01175_b200/shard.py builds one per rank of a subtree partition)
// ---------------------------------------------------------------------------
static_assert(sizeof(MmItem) == sizeof(h2b_mm_item), "item layout");
static_assert(sizeof(MmSeg) == sizeof(h2b_mm_seg), "segment layout");

struct h2b_plan_ctx {
  int device = 0;
  int n_payloads = 0;
  double2* pay[A_N] = {};
  int64_t pay_elems[A_N] = {};
  struct Phase {
    std::vector<int2> launches;
    MmItem* items = nullptr;
    MmSeg* segs = nullptr;
  };
  std::vector<Phase> phases;
  int64_t device_bytes = 0;
};

extern "C" int h2b_plan_create(int device, int n_payloads, const int64_t* payload_elems,
                               h2b_plan_handle* out) {
  if (!out || n_payloads < 0 || n_payloads > A_N || (n_payloads && !payload_elems)) {
    h2b_set_error("h2b_plan_create: bad arguments (at most 6 payloads)");
    return H2B_EINVAL;
  }
  if (!h2b_device_ok(device)) {
    h2b_set_error("h2b_plan_create: no sm_100 device");
    return H2B_ENODEV;
  }
  H2B_CUDA_TRY(cudaSetDevice(device));
  auto* p = new h2b_plan_ctx();
  p->device = device;
  p->n_payloads = n_payloads;
  for (int i = 0; i < n_payloads; ++i) {
    p->pay_elems[i] = payload_elems[i];
    cudaError_t e = cudaMalloc(&p->pay[i], 16 * (size_t)std::max<int64_t>(payload_elems[i], 1));
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (int j = 0; j < i; ++j) cudaFree(p->pay[j]);
      delete p;
      h2b_set_error("h2b_plan_create: payload allocation failed");
      return H2B_ENOMEM;
    }
    p->device_bytes += 16 * std::max<int64_t>(payload_elems[i], 1);
  }
  *out = p;
  return H2B_OK;
}

extern "C" int h2b_plan_upload(h2b_plan_handle p, int payload, const void* src, size_t bytes, size_t offset) {
  if (!p || payload < 0 || payload >= p->n_payloads || (!src && bytes) ||
      offset + bytes > 16 * (size_t)p->pay_elems[payload]) {
    h2b_set_error("h2b_plan_upload: bad arguments");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  if (bytes) H2B_CUDA_TRY(cudaMemcpy((char*)p->pay[payload] + offset, src, bytes, cudaMemcpyHostToDevice));
  return H2B_OK;
}

extern "C" int h2b_plan_set_phase(h2b_plan_handle p, int phase, int n_launches, const int64_t* launch_items,
                                  const h2b_mm_item* items, int64_t n_items, const h2b_mm_seg* segs,
                                  int64_t n_segs) {
  if (!p || phase < 0 || phase > 64 || n_launches < 0 || n_items < 0 || n_segs < 0) {
    h2b_set_error("h2b_plan_set_phase: bad arguments");
    return H2B_EINVAL;
  }
  int64_t tot = 0;
  for (int i = 0; i < n_launches; ++i) tot += launch_items[i];
  if (tot != n_items) {
    h2b_set_error("h2b_plan_set_phase: launch item counts do not add up to n_items");
    return H2B_EINVAL;
  }
  for (int64_t i = 0; i < n_items; ++i) {  // validate references (the kernel trusts them)
    const h2b_mm_item& it = items[i];
    if (it.m < 0 || it.m > MM_M || it.seg0 < 0 || it.nseg < 0 || it.seg0 + (int64_t)it.nseg > n_segs ||
        (it.flags & 15) > B_N) {
      h2b_set_error("h2b_plan_set_phase: item " + std::to_string(i) + " out of range");
      return H2B_EINVAL;
    }
    for (int s = 1; s < it.nseg; ++s)
      if ((segs[it.seg0 + s].flags ^ segs[it.seg0].flags) & SEG_TRANS) {
        h2b_set_error("h2b_plan_set_phase: item " + std::to_string(i) + " mixes A orientations");
        return H2B_EINVAL;
      }
  }
  for (int64_t i = 0; i < n_segs; ++i) {
    const h2b_mm_seg& sg = segs[i];
    if (sg.k < 0 || sg.k > MM_K || (sg.flags & 15) >= p->n_payloads || ((sg.flags >> 4) & 15) >= B_N ||
        (sg.flags & SEG_GATHER)) {
      h2b_set_error("h2b_plan_set_phase: segment " + std::to_string(i) + " out of range");
      return H2B_EINVAL;
    }
  }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  if ((int)p->phases.size() <= phase) p->phases.resize(phase + 1);
  auto& ph = p->phases[phase];
  cudaFree(ph.items);
  cudaFree(ph.segs);
  ph.items = nullptr;
  ph.segs = nullptr;
  ph.launches.clear();
  H2B_CUDA_TRY(cudaMalloc(&ph.items, sizeof(MmItem) * std::max<int64_t>(n_items, 1)));
  H2B_CUDA_TRY(cudaMalloc(&ph.segs, sizeof(MmSeg) * std::max<int64_t>(n_segs, 1)));
  if (n_items) H2B_CUDA_TRY(cudaMemcpy(ph.items, items, sizeof(MmItem) * n_items, cudaMemcpyHostToDevice));
  if (n_segs) H2B_CUDA_TRY(cudaMemcpy(ph.segs, segs, sizeof(MmSeg) * n_segs, cudaMemcpyHostToDevice));
  int64_t first = 0;
  for (int i = 0; i < n_launches; ++i) {
    ph.launches.push_back(int2{(int)first, (int)launch_items[i]});
    first += launch_items[i];
  }
  p->device_bytes += sizeof(MmItem) * n_items + sizeof(MmSeg) * n_segs;
  return H2B_OK;
}

extern "C" int h2b_plan_run(h2b_plan_handle p, int phase, const void* x, const void* xhat, void* yhat,
                            void* y, int q, void* stream) {
  if (!p || phase < 0 || phase >= (int)p->phases.size() || q < 1) {
    h2b_set_error("h2b_plan_run: bad arguments");
    return H2B_EINVAL;
  }
  static bool attr = false;
  if (!attr) {
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_zgemm_grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, MM_SMEM));
    attr = true;
  }
  MmBufs bf{};
  for (int i = 0; i < A_N; ++i) bf.a[i] = p->pay[i];
  bf.b[B_X] = const_cast<double2*>((const double2*)x);
  bf.b[B_XHAT] = const_cast<double2*>((const double2*)xhat);
  bf.b[B_YHAT] = (double2*)yhat;
  bf.y = (double2*)y;
  bf.gather = nullptr;
  const auto& ph = p->phases[phase];
  int nl = 0;
  for (const int2& L : ph.launches)
    H2B_TRY(run_grouped(ph.items + L.x, L.y, ph.segs, bf, q, (cudaStream_t)stream, &nl));
  return H2B_OK;
}

extern "C" int h2b_plan_destroy(h2b_plan_handle p) {
  if (!p) return H2B_OK;
  cudaSetDevice(p->device);
  for (auto& ph : p->phases) {
    cudaFree(ph.items);
    cudaFree(ph.segs);
  }
  for (int i = 0; i < p->n_payloads; ++i) cudaFree(p->pay[i]);
  delete p;
  return H2B_OK;
}

extern "C" int64_t h2b_plan_device_bytes(h2b_plan_handle p) { return p ? p->device_bytes : -1; }
