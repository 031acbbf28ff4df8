// Far field of the single-RHS H² matvec as ONE persistent launch of subtree programs (sm_100a).
//
// Restates the far-field part of the reference `_apply_perm` (/root/reference/pkg/src/h2vie/
// arith.py:58-99): x̂ = Vᵀx at the leaves, x̂_t = T_loᵀx̂_lo + T_hiᵀx̂_hi upward, ŷ_t = Σ S^{t,s}x̂_s
// over the admissible pairs, ŷ_child += T_child ŷ_t downward and y += V ŷ at the leaves.
//
// For complete binary cluster trees (every leaf on the deepest level, leaves of one size, the
// packed children of ordinal i at ordinals 2i and 2i+1 of the next level; all BASELINE configs)
// the tree is cut at a split level ls into
//   * bottom programs: one per level-ls cluster, its whole subtree down to the leaves, and
//   * top programs:    one per cluster of the topmost level lt with any non-zero rank, its
//                      subtree down to level ls-1 (the level-ls clusters are its external
//                      children, computed by the bottom programs).
// Each program is ONE CTA for the whole launch.  It stages its operator payload (x, V, T and the
// transposed coupling panels Sᵀ of its targets, plus its node table and gather list) with TMA
// bulk copies once at launch and keeps it in shared memory: V and T serve both the upward and
// the downward pass, so every payload element is read from HBM exactly once per matvec (the
// minimal-traffic B_alg convention of SURVEY.md §8d).  The critical path is three inter-CTA
// hand-offs (epoch-stamped flags in global memory):
//   bottom up  -> [flag up] -> top up, top couplings (after the other top programs' flags),
//   top down -> [flag down] -> bottom down; bottom couplings wait only for the neighbouring
//   bottom programs' x̂ and run while the top works.
// With the flat top (r02, see FlatAnc below; at most five levels above the split) there are no
// top programs: every bottom program carries the folded operators of its ancestors and the
// levels above the split cost ONE hand-off (the programs' shares of the ancestors' x̂).
// The near field runs concurrently in k_near_stream (h2b_mega.cu); both add into y, which the
// bottom programs zero at their start (ZeroSync, h2b_common.cuh) unless a memset node did.
#include <algorithm>
#include <cstring>
#include <map>
#include <set>
#include <vector>

#include "h2b_panel.cuh"

namespace {

constexpr int TNT = 256;  // threads per program CTA
constexpr int TREE_FLAT_EXTRA = 6 * 1024;  // shared memory a flat-top program may use beyond the budget
constexpr int TREE_MAXLEV = 24;

// node of a program (64 bytes, staged into shared memory; offsets in double2 elements).  Every
// operand offset is precomputed on the host so that a level step is one record load per node.
struct TNode {
  int32_t k, kind;    // rank; kind: 0 leaf, 1 internal, 2 external child (x̂ / ŷ via global)
  int32_t xh;         // x̂ of the node in smem (ŷ at xh + yoff)
  int32_t pay;        // V (leaf, n x k) or T ((k_lo + k_hi) x k, rows lo then hi)
  int32_t R;          // rows of pay (leaf: points n; internal: k_lo + k_hi)
  int32_t in;         // up: input of the rows (leaf: x segment; internal: [x̂_lo; x̂_hi])
  int32_t sh;         // log2 of k rounded up to a power of two
  int32_t s_pay;      // coupling panel Sᵀ (s_rows x k): global element offset in sbuf (high half in pad)
  int32_t s_rows;     // 0: no couplings
  int32_t xg;         // first gathered x̂ row of the panel (x̂g area / gather index list)
  int32_t gx_lo, gx_hi;  // global x̂ / ŷ offset of the node
  int32_t gy_lo, gy_hi;  // leaf: global y offset; internal with external children: their global ŷ
  int32_t ext, pad;      // internal: 1 if the children are external; pad: s_pay >> 32
};
static_assert(sizeof(TNode) == 64, "TNode layout");

struct TCopy {  // global -> smem bulk copy
  int64_t src;  // element offset in the source buffer
  int32_t kind, elems, smem, pad;
};
enum TSrc : int32_t { TS_X = 0, TS_V, TS_T, TS_S, TS_NODES, TS_GIDX, TS_FM, TS_FH, TS_FF, TS_N };
// TS_FM / TS_FH / TS_FF: the flattened top tier of a bottom program (chains M up to its
// ancestors, the panels H = Sᵀ Mᵀ of the ancestors, the chains F from its root down to its
// leaves; see "flat top" below).  M is staged with the transfers; H and F are requested late,
// into the place of the coupling panels.
__host__ __device__ inline bool ts_late(int kind) { return kind >= TS_FH; }

struct TProg {
  int32_t n_nodes, nlev, n_copy, copy_first;
  int32_t stage_bytes, smem_elems, yoff, xg_smem;
  int32_t n_xg, gidx_smem, n_wait_up, wait_up_first;
  int32_t wait_down, n_ext_wait, ext_wait_first, bottom;
  int32_t lev_first[TREE_MAXLEV + 1];
  int32_t pad[3];
  int32_t f_base, f_stride;  // bottom: per-node slots for F_c = T-chain from the root (-1: none)
  // bottom: the far field of the subtree's y rows is assembled in shared memory (the staged x
  // area, dead after the upward pass) and added to y by ONE bulk reduce-add (instead of an
  // atomic per element): y_n rows from smem y_smem to global row y_g
  int32_t y_smem, y_n, y_g_lo, y_g_hi;
  // flat top (bottom programs, no top programs): n_flat pseudo nodes (one per ancestor above the
  // split level) at nodes[flat_first ..]; gather rows of the ancestors' sources: n_frow headers
  // {log2 partials per entry, first entry, valid entries, first x̂g row} at smem element frow_smem,
  // the entries' first partial (index into px) as int32 at smem element ebase_smem
  int32_t n_flat, flat_first, n_frow, frow_smem;
  int32_t ebase_smem, px_stride, fh_bytes, split_mode;  // split_mode: 0 none, 1 F chains formed here, 2 staged
  int32_t n_wait_far, wait_far_first, fpad2, fpad3;  // flat top: the programs whose partials are read
};

struct TreeArgs {
  const TProg* progs;
  const TCopy* copies;
  const int32_t* waits;  // program ids
  const void* src[TS_N];
  double2* xhat;
  double2* yhat;
  double2* y;
  double2* px;  // flat top: partial x̂ of every ancestor level from every bottom program
  uint32_t* flags_up;
  uint32_t* flags_down;
  MegaCtrl* ctrl;
  uint64_t* trace;  // optional (H2B_TREE_TRACE): 16 timestamps per program
  // y zeroed by the bottom programs at their start (ZeroSync in h2b_common.cuh; nullptr: by the
  // caller); zrows[c] = the rows {first, count} of near-field CTA c, c < near_ctas
  ZeroSync* zs;
  const int2* zrows;
  int near_ctas;
  int defer_s;       // request the staged coupling panels after the up-pass operands
  int trace_levels;  // H2B_TREE_TRACE=2: stamps 9-14 per level of the upward pass; 3: of the downward pass
};

// Code size matters here: every phase of k_far_tree runs once per launch, so its instructions
// are fetched cold (measured: the bottom programs' last step 2.8 us on first execution, 1.7 us
// when repeated).  Rare paths are kept out of line and not unrolled.
__device__ __noinline__ void tmark_impl(uint64_t* trace, int i) {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  trace[32 * blockIdx.x + i] = t;
  trace[32 * blockIdx.x + 16 + i] = clock64();
}
__device__ __forceinline__ void tmark(const TreeArgs& A, int i) {
  if (A.trace && threadIdx.x == 0) tmark_impl(A.trace, i);
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// warp 0 waits until flags[ids[i]] == want for every i: the ids are loaded once (up to four per
// lane in registers), then relaxed sweeps, then one acquire fence; the caller follows with
// __syncthreads
__device__ __noinline__ void wait_flags(const uint32_t* flags, const int32_t* ids, int n, uint32_t want,
                                        MegaCtrl* ctrl) {
  if (threadIdx.x >= 32 || n == 0) return;
  const int lane = threadIdx.x;
  int f[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) f[u] = lane + 32 * u < n ? ids[lane + 32 * u] : -1;
  for (long spins = 0;; ++spins) {
    bool ok = true;
#pragma unroll
    for (int u = 0; u < 4; ++u) ok &= f[u] < 0 || ld_relaxed(flags + f[u]) == want;
#pragma unroll 1
    for (int i = lane + 128; i < n; i += 32) ok &= ld_relaxed(flags + ids[i]) == want;
    if (__all_sync(0xffffffffu, ok)) break;
    if (spins > (1l << 24)) {  // never expected: report instead of hanging the GPU
      atomicExch(&ctrl->error, 2u);
      break;
    }
    __nanosleep(20);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// out[c] = Σ_r P[r*w + c] in[r] for c < w (one warp).  Lane (g, c): column c of row group g,
// rows g, g + G, ... ; every chunk issues its loads before its FMAs (the ops are small: latency,
// not throughput, decides), then the G partial sums meet through xor shuffles.
__device__ __forceinline__ double2 colsum_sum(const double2* P, int R, int w, int sh, const double2* in) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << sh, G = 32 >> sh;
  const int g = lane >> sh, c = lane & (wp - 1);
  double2 a = make_double2(0.0, 0.0), b = a;
  if (w <= 32) {
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
  }
  return a;
}

__device__ __forceinline__ void colsum(const double2* P, int R, int w, int sh, const double2* in, double2* out) {
  const int lane = threadIdx.x & 31;
  if (w <= 32) {
    const double2 s = colsum_sum(P, R, w, sh, in);
    if (lane < w) out[lane] = s;
  } else {
    for (int c = lane; c < w; c += 32) {
      double2 a0 = make_double2(0.0, 0.0), a1 = a0;
      int r = 0;
#pragma unroll 1
      for (; r + 1 < R; r += 2) {
        cfma(a0, P[r * w + c], in[r]);
        cfma(a1, P[(r + 1) * w + c], in[r + 1]);
      }
      if (r < R) cfma(a0, P[r * w + c], in[r]);
      out[c] = cadd(a0, a1);
    }
  }
}

// Σ_j P[r*w + j] v[j] for one row r (a lane's dot product), loads before FMAs in chunks of 4
__device__ __forceinline__ double2 rowdot(const double2* P, int r, int w, const double2* v) {
  double2 a = make_double2(0.0, 0.0), b = a;
  const double2* p = P + r * w;
  for (int j0 = 0; j0 < w; j0 += 4) {
    double2 pv[4], vv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = j0 + i < w;
      pv[i] = ok ? p[j0 + i] : make_double2(0.0, 0.0);
      vv[i] = ok ? v[j0 + i] : make_double2(0.0, 0.0);
    }
    cfma(a, pv[0], vv[0]);
    cfma(b, pv[1], vv[1]);
    cfma(a, pv[2], vv[2]);
    cfma(b, pv[3], vv[3]);
  }
  return cadd(a, b);
}

// ---- CTA-wide level operations --------------------------------------------------------------
// A level's nodes are small (ranks 3..30, a few dozen rows): warp-per-node loops left most of a
// warp idle and chained shared-memory loads, shuffles and node after node (measured ~700 cycles
// for a 4 x 3 coupling panel).  Here all nodes of a level are processed at once, each by a
// group of 2^shk x G threads (column c, row group g); a thread's loads are issued together
// (unconditional, from clamped rows) before its FMAs, and G <= 4 row groups meet in log2 G
// shuffle levels.

// Σ over rows r = g, g + G, ... < R of M[r w + c] in[r] (c < w, R >= 1)
__device__ __forceinline__ double2 col_dot(const double2* M, int R, int w, int c, const double2* in, int g, int G) {
  double2 a0 = make_double2(0.0, 0.0), a1 = a0;
  int r = g;
  for (; r + 3 * G < R; r += 4 * G) {
    const double2 p0 = M[r * w + c], p1 = M[(r + G) * w + c], p2 = M[(r + 2 * G) * w + c],
                  p3 = M[(r + 3 * G) * w + c];
    const double2 x0 = in[r], x1 = in[r + G], x2 = in[r + 2 * G], x3 = in[r + 3 * G];
    cfma(a0, p0, x0);
    cfma(a1, p1, x1);
    cfma(a0, p2, x2);
    cfma(a1, p3, x3);
  }
  for (; r < R; r += G) cfma(a0, M[r * w + c], in[r]);
  return cadd(a0, a1);
}

// Σ_j M[r w + j] v[j] for one row (loads of 4 columns before their FMAs)
__device__ __forceinline__ double2 row_dot(const double2* M, int r, int w, const double2* v) {
  double2 a0 = make_double2(0.0, 0.0), a1 = a0;
  const double2* m = M + r * w;
  int j = 0;
  for (; j + 4 <= w; j += 4) {
    const double2 p0 = m[j], p1 = m[j + 1], p2 = m[j + 2], p3 = m[j + 3];
    const double2 x0 = v[j], x1 = v[j + 1], x2 = v[j + 2], x3 = v[j + 3];
    cfma(a0, p0, x0);
    cfma(a1, p1, x1);
    cfma(a0, p2, x2);
    cfma(a1, p3, x3);
  }
  for (; j < w; ++j) cfma(a0, m[j], v[j]);
  return cadd(a0, a1);
}

// out_i[c] = Σ_r M_i[r w_i + c] in_i[r] (c < w_i) for the nodes i in [a, b) that get() accepts;
// get(nd, M, R, w, in, out) -> bool.  shk: log2 of the columns slot per node (w_i <= 2^shk).
// A node accepted with R = 0 gets out = 0.
template <class Get>
__device__ __forceinline__ void cta_colsum(const TNode* nodes, int a, int b, int shk, Get get) {
  const int n = b - a;
  if (n <= 0) return;
  int shg = 0;  // row groups G = 2^shg: as many as the CTA has threads for, at most 4
  while (shg < 2 && shk + shg < 5 && (n << (shk + shg + 1)) <= TNT) ++shg;
  const int sht = shk + shg, G = 1 << shg;
  const int items = n << sht;
  const int bound = (items + 31) & ~31;  // warp-uniform trip count (the shuffles below)
  for (int it = threadIdx.x; it < bound; it += TNT) {
    const int l = it & ((1 << sht) - 1);
    const int c = l & ((1 << shk) - 1), g = l >> shk;
    double2 s = make_double2(0.0, 0.0);
    double2* out = nullptr;
    bool ok = false;
    if (it < items) {
      const TNode nd = nodes[a + (it >> sht)];
      const double2 *M, *in;
      int R, w;
      if (get(nd, M, R, w, in, out) && c < w) {
        ok = true;
        if (g < R) s = col_dot(M, R, w, c, in, g, G);
      }
    }
    for (int m = 1 << shk; m < (1 << sht); m <<= 1) s = cadd(s, shfl_xor2(s, m));
    if (ok && g == 0) out[c] = s;
  }
}

// for the nodes i in [a, b) that get() accepts, each row r < R_i: emit(nd, r, Σ_j M_i[r w_i + j]
// v_i[j]); get(i, nd, M, R, w, v) -> bool.  2^shr threads per node (rows r = l, l + 2^shr, ...).
template <class Get, class Emit>
__device__ __forceinline__ void cta_rowdot(const TNode* nodes, int a, int b, int shr, Get get, Emit emit) {
  const int items = (b - a) << shr;
  for (int it = threadIdx.x; it < items; it += TNT) {
    const int i = a + (it >> shr);
    const TNode nd = nodes[i];
    const double2 *M, *v;
    int R, w;
    if (!get(i, nd, M, R, w, v)) continue;
    for (int r = it & ((1 << shr) - 1); r < R; r += 1 << shr) emit(nd, r, row_dot(M, r, w, v));
  }
}

// at most 128 registers: 2 warps per scheduler (8192 registers) leave the near-field stream's 3
// warps on scheduler 0 their 80 each within the scheduler's 16K (both kernels co-resident)
#define H2B_TREE_KERNEL k_far_tree
#define H2B_TREE_TR 0
#define H2B_TMARK(A, i) ((void)0)
#include "h2b_tree_kernel.inc"
#undef H2B_TREE_KERNEL
#undef H2B_TREE_TR
#undef H2B_TMARK
#define H2B_TREE_KERNEL k_far_tree_traced
#define H2B_TREE_TR 1
#define H2B_TMARK(A, i) tmark(A, i)
#include "h2b_tree_kernel.inc"
#undef H2B_TREE_KERNEL
#undef H2B_TREE_TR
#undef H2B_TMARK

}  // namespace

// ===========================================================================
// host: the plan
// ===========================================================================
struct TreePlan {
  std::vector<TProg> progs;
  std::vector<TCopy> copies;
  std::vector<int32_t> waits;
  std::vector<TNode> nodes_all;   // staged from a device copy (TS_NODES)
  std::vector<int32_t> gidx_all;  // staged from a device copy (TS_GIDX), 4 per 16-byte element
  std::vector<double2> flat_all;  // flat top: transfer chains and H panels (TS_FM / TS_FH)
  int64_t px_elems = 0;           // flat top: partial x̂ area (elements)
  int64_t n_rows_total = 0;       // N (rows of y)
  bool flat = false;
  int smem_max = 0;               // bytes
  int ls = 0, lt = 0, n_bottom = 0, n_top = 0;
};

namespace {

int level_of_p(const h2b_ctx* h, int p) {
  int l = 0;
  while (l + 1 <= h->depth && h->level_ptr[l + 1] <= p) ++l;
  return l;
}

// the tree qualifies when it is complete in packed order with uniform leaves on the last level
// and only same-level couplings
bool tree_shape_ok(const h2b_ctx* h) {
  const int L = h->depth;
  if (L < 2 || h->uniform_leaf <= 0) return false;
  for (int l = 0; l < L; ++l)
    if (h->level_ptr[l + 1] - h->level_ptr[l] != (1 << l)) return false;
  for (int l = 0; l + 1 < L; ++l)
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) {
      const int i = p - h->level_ptr[l];
      if (h->c_child_lo[p] != h->level_ptr[l + 1] + 2 * i || h->c_child_hi[p] != h->level_ptr[l + 1] + 2 * i + 1)
        return false;
    }
  for (int p = h->level_ptr[L - 1]; p < h->P; ++p)
    if (h->c_child_lo[p] >= 0 || h->c_size[p] != h->uniform_leaf) return false;
  for (int l = 0; l < L; ++l)
    for (int t = h->level_ptr[l]; t < h->level_ptr[l + 1]; ++t)
      for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
        const int s = h->s_col[b];
        if (s < h->level_ptr[l] || s >= h->level_ptr[l + 1]) return false;
      }
  return true;
}

// Flat top (r02): instead of top programs walking the levels above the split level ls (five
// dependent level steps up, the couplings, five down and two more flag hand-offs at cfg2, all
// latency), every bottom program c carries, for each ancestor t_d at level ls - d,
//   M_d = T-chain from c up to t_d (k_c x k_t):  x̂_t = Σ_c M_dᵀ x̂_c,  ŷ_c += M_d ŷ_t, and
//   H_d = Sᵀ_panel(t_d) M_dᵀ ((Σ_s k_s) x k_c): ŷ_c += H_dᵀ [x̂_s]_s  (couplings of t_d, then down).
// Up: c writes its partials M_dᵀ x̂_c to px (fixed slots, no atomics), then ONE flag hand-off;
// down: c sums the partials of the programs below each source (fixed order) and applies H_d
// like a coupling panel (a pseudo node of the program).  The products M and H are formed on
// the host from the uploaded T and Sᵀ (double precision; the reference applies the factors one
// after the other, arith.py:68-99, so results agree to rounding, not bitwise).
struct FlatAnc {
  int d = 0, t = 0, kt = 0, rows = 0;
  std::vector<double2> M, H;   // k_c x kt ; rows x k_c
  std::vector<int32_t> ebase;  // per gathered row: px index of its first partial
};

struct Builder {
  const h2b_ctx* h;
  TreePlan& tp;
  // flat top: host copies of T and Sᵀ, the split / top levels, programs and the px row stride
  const double2* hT = nullptr;
  const double2* hS = nullptr;
  int ls = 0, lt = 0, nb = 0, kp = 0;
  bool flat = false;

  std::vector<FlatAnc> flat_ancestors(int root) const {
    std::vector<FlatAnc> out;
    const int i = root - h->level_ptr[ls];
    const int kc = h->c_rank[root];
    if (kc == 0) return out;  // nothing flows through a rank-0 root (its px slots stay zero)
    std::vector<double2> M;  // k_c x kprev
    int kprev = kc;
    for (int d = 1; d <= ls - lt; ++d) {
      const int t = h->level_ptr[ls - d] + (i >> d);
      const int child = h->level_ptr[ls - d + 1] + (i >> (d - 1));
      const int kt = h->c_rank[t], kch = h->c_rank[child];
      const int r0 = ((i >> (d - 1)) & 1) ? h->c_rank[h->c_child_lo[t]] : 0;
      const double2* T = hT + h->c_toff[t];
      std::vector<double2> Mn((size_t)kc * kt, make_double2(0.0, 0.0));
      for (int b = 0; b < kc; ++b)
        for (int a = 0; a < kt; ++a) {
          double2 acc = make_double2(0.0, 0.0);
          if (d == 1) {
            acc = T[(size_t)(r0 + b) * kt + a];
          } else {
            for (int j = 0; j < kch; ++j) {
              const double2 m = M[(size_t)b * kprev + j], tv = T[(size_t)(r0 + j) * kt + a];
              acc.x += m.x * tv.x - m.y * tv.y;
              acc.y += m.x * tv.y + m.y * tv.x;
            }
          }
          Mn[(size_t)b * kt + a] = acc;
        }
      M.swap(Mn);
      kprev = kt;
      if (kt == 0) break;  // the chain ends: nothing flows through a rank-0 ancestor
      FlatAnc fa;
      fa.d = d;
      fa.t = t;
      fa.kt = kt;
      fa.M = M;
      const int64_t b0 = h->s_row_ptr[t], b1 = h->s_row_ptr[t + 1];
      for (int64_t b = b0; b < b1; ++b) {
        const int sc = h->s_col[b], ks = h->c_rank[sc];
        const double2* St = hS + h->s_off[b];  // Sᵀ block: k_s x k_t
        const int64_t si = sc - h->level_ptr[ls - d];
        for (int r = 0; r < ks; ++r) {
          for (int bb = 0; bb < kc; ++bb) {
            double2 acc = make_double2(0.0, 0.0);
            for (int a = 0; a < kt; ++a) {
              const double2 sv = St[(size_t)r * kt + a], m = M[(size_t)bb * kt + a];
              acc.x += sv.x * m.x - sv.y * m.y;
              acc.y += sv.x * m.y + sv.y * m.x;
            }
            fa.H.push_back(acc);
          }
          fa.ebase.push_back((int32_t)((((int64_t)(d - 1) * nb + (si << d)) * kp) + r));
        }
        fa.rows += ks;
      }
      out.push_back(std::move(fa));
    }
    return out;
  }
  // one program: the subtree of cluster `root` over levels [root level, last] (last inclusive);
  // ext: the level below `last` is external (x̂ from / ŷ to global)
  bool build(int root, int last, bool bottom, int budget_elems) {
    const int L = h->depth;
    const int rl = level_of_p(h, root);
    TProg P{};
    P.bottom = bottom ? 1 : 0;
    P.wait_down = -1;
    // nodes by level (packed order inside a level)
    std::vector<int> nd_p;
    std::vector<int> lev_first;
    const int nl = last - rl + 1 + (bottom ? 0 : 1);
    if (nl > TREE_MAXLEV) return false;
    const int i0 = root - h->level_ptr[rl];
    for (int d = 0; d < nl; ++d) {
      lev_first.push_back((int)nd_p.size());
      const int l = rl + d;
      const int a = h->level_ptr[l] + (i0 << d), cnt = 1 << d;
      for (int p = a; p < a + cnt; ++p) nd_p.push_back(p);
    }
    lev_first.push_back((int)nd_p.size());
    (void)L;
    const int nn = (int)nd_p.size();
    std::map<int, int> idx_of;
    for (int i = 0; i < nn; ++i) idx_of[nd_p[i]] = i;
    // flat top: one pseudo node per ancestor above the split level (behind the real nodes)
    std::vector<FlatAnc> fl;
    if (flat && bottom) fl = flat_ancestors(root);
    const int nfl = (int)fl.size();
    // gather rows of the flat ancestors: 32 >> d entries per row of 2^d partials each
    std::vector<int32_t> frow, ebase_all;
    std::vector<int> fl_efirst(nfl, 0);
    for (int f = 0; f < nfl; ++f) {
      fl_efirst[f] = (int)ebase_all.size();
      ebase_all.insert(ebase_all.end(), fl[f].ebase.begin(), fl[f].ebase.end());
    }
    // smem layout (double2 elements): nodes | gather idx | x | V | T | S | x̂ | ŷ | x̂g
    int off = 4 * (nn + nfl);  // 64-byte nodes
    std::vector<TNode> nodes(nn + nfl);
    std::vector<int32_t> gl;  // gather list (global x̂ index, or ~smem offset for own nodes)
    // coupling rows first (their count sizes the gather list)
    std::vector<int> xh_of(nn + nfl, 0);
    int xh_total = 0;
    for (int i = 0; i < nn; ++i) {
      xh_of[i] = xh_total;
      xh_total += h->c_rank[nd_p[i]];
    }
    for (int f = 0; f < nfl; ++f) {  // a ŷ slot per pseudo node (k_root entries)
      xh_of[nn + f] = xh_total;
      xh_total += h->c_rank[root];
    }
    const int own_end = bottom ? nn : lev_first[nl - 1];  // nodes the program computes
    int n_rows = 0;
    for (int i = 0; i < own_end; ++i) {
      const int t = nd_p[i];
      if (h->c_rank[t] == 0) continue;
      for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) n_rows += h->c_rank[h->s_col[b]];
    }
    const int gidx_smem = off;
    off += (n_rows + 3) / 4;
    int n_frow = 0;
    for (int f = 0; f < nfl; ++f) n_frow += (fl[f].rows + (32 >> fl[f].d) - 1) / (32 >> fl[f].d);
    const int frow_smem = off;
    off += n_frow;
    const int ebase_smem = off;
    off += ((int)ebase_all.size() + 3) / 4;
    int x_smem = -1, v_smem = -1;
    auto push_copy = [&](int kind, int64_t src, int elems, int smem) {
      if (elems <= 0) return;
      if (!tp.copies.empty() && (int)tp.copies.size() > P.copy_first) {
        TCopy& c = tp.copies.back();
        if (c.kind == kind && c.src + c.elems == src && c.smem + c.elems == smem && c.elems + elems <= 65536) {
          c.elems += elems;
          return;
        }
      }
      tp.copies.push_back(TCopy{src, kind, elems, smem, 0});
    };
    P.copy_first = (int)tp.copies.size();
    push_copy(TS_NODES, (int64_t)tp.nodes_all.size() * 4, 4 * (nn + nfl), 0);
    if (bottom) {  // x of the subtree's points
      x_smem = off;
      push_copy(TS_X, h->c_start[root], h->c_size[root], off);
      off += h->c_size[root];
      v_smem = off;
    }
    // payloads
    std::vector<int> lo_idx(nn, -1);
    auto shpow = [](int w) { int sh = 0; while ((1 << sh) < w) ++sh; return sh; };
    for (int i = 0; i < own_end; ++i) {
      const int p = nd_p[i];
      TNode& n = nodes[i];
      n.k = h->c_rank[p];
      n.sh = shpow(n.k);
      const bool leaf = h->c_child_lo[p] < 0;
      n.kind = leaf ? 0 : 1;
      if (leaf) {
        n.R = h->c_size[p];
        n.in = x_smem + (int)(h->c_start[p] - h->c_start[root]);
        n.gy_lo = (int32_t)(uint32_t)(int64_t)h->c_start[p];
        n.gy_hi = (int32_t)((int64_t)h->c_start[p] >> 32);
        const int e = n.R * n.k;
        n.pay = off;
        push_copy(TS_V, h->c_voff[p], e, off);
        off += e;
      } else {
        const int lo = h->c_child_lo[p];
        if (!idx_of.count(lo)) return false;
        lo_idx[i] = idx_of[lo];
        n.R = h->c_rank[lo] + h->c_rank[h->c_child_hi[p]];
        n.ext = lo_idx[i] >= own_end ? 1 : 0;
        if (n.ext) {  // the children's global ŷ (written by the down pass)
          n.gy_lo = (int32_t)(uint32_t)h->c_xoff[lo];
          n.gy_hi = (int32_t)(h->c_xoff[lo] >> 32);
        }
        const int e = n.R * n.k;
        n.pay = off;
        push_copy(TS_T, h->c_toff[p], e, off);
        off += e;
      }
    }
    for (int i = own_end; i < nn; ++i) {  // external children (top programs)
      TNode& n = nodes[i];
      n.k = h->c_rank[nd_p[i]];
      n.kind = 2;
    }
    // coupling panels (Sᵀ, stacked per target) and the gather list.  The panels are staged in
    // shared memory when they fit the budget (H2B_TREE_S_L2: never), else read from L2 after a
    // prefetch at launch.
    int64_t s_total = 0;
    for (int i = 0; i < own_end; ++i) {
      const int t = nd_p[i];
      if (h->c_rank[t] == 0) continue;
      for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b)
        s_total += (int64_t)h->c_rank[h->s_col[b]] * h->c_rank[t];
    }
    const bool s_l2 = getenv("H2B_TREE_S_L2") != nullptr;  // experiment: panels from L2 always
    const int s_first = off;  // the staged panels start here
    const bool stage_s = !s_l2 && off + s_total + 2 * xh_total + n_rows <= budget_elems;
    // reading the panels from L2 was measured 3x slower than the task-graph kernel at cfg1
    // (warp-per-target GEMVs on L2 latency): the tree plan is only taken with staged panels
    if (!stage_s && !s_l2) return false;
    int xg_rows = 0;
    for (int i = 0; i < own_end; ++i) {
      const int t = nd_p[i];
      TNode& n = nodes[i];
      n.s_rows = 0;
      if (n.k == 0) continue;
      const int64_t b0 = h->s_row_ptr[t], b1 = h->s_row_ptr[t + 1];
      int rows = 0;
      for (int64_t b = b0; b < b1; ++b) rows += h->c_rank[h->s_col[b]];
      if (rows == 0) continue;
      n.s_rows = rows;
      n.xg = xg_rows;
      const int64_t so = stage_s ? off : h->s_off[b0];  // smem offset (staged) or sbuf offset (L2)
      n.s_pay = (int32_t)(uint32_t)so;
      n.pad = (int32_t)(so >> 32);
      if (stage_s) {
        // consecutive targets' panels are adjacent in sbuf and here: one bulk copy per run (a
        // program's ~30 panel copies become ~5: fewer, larger requests on the SM's copy queue,
        // which the near-field ring shares)
        if ((int)tp.copies.size() > P.copy_first && tp.copies.back().kind == TS_S && tp.copies.back().smem >= 0 &&
            tp.copies.back().src + tp.copies.back().elems == h->s_off[b0] &&
            tp.copies.back().smem + tp.copies.back().elems == off && tp.copies.back().elems + rows * n.k <= 32768)
          tp.copies.back().elems += rows * n.k;
        else
          tp.copies.push_back(TCopy{h->s_off[b0], TS_S, rows * n.k, off, 0});
        off += rows * n.k;
      } else {  // L2 prefetch range (merged with the previous target's when contiguous)
        TCopy pc{h->s_off[b0], TS_S, rows * n.k, -1, 0};
        if ((int)tp.copies.size() > P.copy_first && tp.copies.back().kind == TS_S &&
            tp.copies.back().src + tp.copies.back().elems == pc.src && tp.copies.back().elems + pc.elems <= 65536)
          tp.copies.back().elems += pc.elems;
        else
          tp.copies.push_back(pc);
      }
      for (int64_t b = b0; b < b1; ++b) {
        const int s = h->s_col[b];
        auto it = idx_of.find(s);
        const bool local = it != idx_of.end() && it->second < own_end;
        // own source: placeholder -2 - (node << 8 | j), resolved to ~smem offset below;
        // other program's source: the global x̂ index
        for (int j = 0; j < h->c_rank[s]; ++j)
          gl.push_back(local ? -2 - (int32_t)((it->second << 8) | j) : (int32_t)(h->c_xoff[s] + j));
        xg_rows += h->c_rank[s];
      }
    }
    // flat top: pseudo nodes; their H panels go where the staged coupling panels were (behind the
    // transfer chains F of the split down pass, see below), their chains M into the x̂g area
    // (consumed before the first gather); gather-row headers
    P.n_flat = nfl;
    P.flat_first = nn;
    P.n_frow = n_frow;
    P.frow_smem = frow_smem;
    P.ebase_smem = ebase_smem;
    P.px_stride = kp;
    const int n_xg_real = xg_rows;
    int m_total = 0, flat_f_base = 0, flat_f_stride = 0;
    if (nfl > 0) {
      const int kc = h->c_rank[root];
      int kmax_all = 0;
      for (int i = 0; i < nn; ++i) kmax_all = std::max(kmax_all, h->c_rank[nd_p[i]]);
      const int64_t need_f = 0;  // (the chains F are staged, not formed in the program)
      int64_t h_off = s_first + need_f, h_total = 0;
      for (int f = 0; f < nfl; ++f) h_total += (int64_t)fl[f].rows * kc;
      if (!stage_s || kc == 0 || need_f + h_total > s_total || kmax_all > 32) return false;
      for (int f = 0; f < nfl; ++f) {
        TNode& n = nodes[nn + f];
        const FlatAnc& fa = fl[f];
        n.k = kc;
        n.kind = 3;
        n.R = fa.kt;
        n.sh = shpow(fa.kt);
        n.s_rows = fa.rows;
        n.xg = xg_rows;
        n.s_pay = (int32_t)h_off;
        n.pad = 0;
        if (fa.rows * kc > 0) {
          tp.copies.push_back(TCopy{(int64_t)tp.flat_all.size(), TS_FH, fa.rows * kc, (int32_t)h_off, 0});
          tp.flat_all.insert(tp.flat_all.end(), fa.H.begin(), fa.H.end());
          h_off += fa.rows * kc;
        }
        const int per = 32 >> fa.d;
        for (int e0 = 0; e0 < fa.rows; e0 += per) {
          frow.push_back(fa.d);
          frow.push_back(fl_efirst[f] + e0);
          frow.push_back(std::min(per, fa.rows - e0));
          frow.push_back(xg_rows + e0);
        }
        xg_rows += fa.rows;
        const int64_t px = ((int64_t)(fa.d - 1) * nb + (root - h->level_ptr[ls])) * kp;
        n.gx_lo = (int32_t)(uint32_t)px;
        n.gx_hi = (int32_t)(px >> 32);
        m_total += kc * fa.kt;
      }
      // chains F_leaf = T...T from the root down to every leaf (k_leaf x k_c), behind the H panels
      {
        std::vector<std::vector<double2>> F(nn);
        F[0].assign((size_t)kc * kc, make_double2(0.0, 0.0));
        for (int j = 0; j < kc; ++j) F[0][(size_t)j * kc + j].x = 1.0;
        for (int lv = 1; lv < nl; ++lv)
          for (int i = lev_first[lv]; i < lev_first[lv + 1]; ++i) {
            const int pi = lev_first[lv - 1] + (i - lev_first[lv]) / 2, hi = (i - lev_first[lv]) & 1;
            const int pp = nd_p[pi], kpar = h->c_rank[pp], kch = h->c_rank[nd_p[i]];
            const int r0 = hi ? h->c_rank[h->c_child_lo[pp]] : 0;
            const double2* T = hT + h->c_toff[pp];
            F[i].assign((size_t)kch * kc, make_double2(0.0, 0.0));
            for (int r = 0; r < kch; ++r)
              for (int c = 0; c < kc; ++c) {
                double2 acc = make_double2(0.0, 0.0);
                for (int j = 0; j < kpar; ++j) {
                  const double2 tv = T[(size_t)(r0 + r) * kpar + j], fv = F[pi][(size_t)j * kc + c];
                  acc.x += tv.x * fv.x - tv.y * fv.y;
                  acc.y += tv.x * fv.y + tv.y * fv.x;
                }
                F[i][(size_t)r * kc + c] = acc;
              }
          }
        int kleaf = 0;
        for (int i = lev_first[nl - 1]; i < nn; ++i) kleaf = std::max(kleaf, h->c_rank[nd_p[i]]);
        const int fs = kleaf * kc, a = lev_first[nl - 1];
        if (need_f + h_total + (int64_t)(nn - a) * fs > s_total || fs == 0) return false;
        flat_f_base = (int)h_off - a * fs;
        flat_f_stride = fs;
        for (int i = a; i < nn; ++i) {
          std::vector<double2> blk((size_t)fs, make_double2(0.0, 0.0));
          std::copy(F[i].begin(), F[i].end(), blk.begin());
          if (i > a && tp.copies.back().kind == TS_FF)  // one bulk copy for all leaves
            tp.copies.back().elems += fs;
          else
            tp.copies.push_back(TCopy{(int64_t)tp.flat_all.size(), TS_FF, fs, (int32_t)h_off, 0});
          tp.flat_all.insert(tp.flat_all.end(), blk.begin(), blk.end());
          h_off += fs;
          h_total += fs;
        }
      }
      P.fh_bytes = (int32_t)(16 * h_total);
    }
    // x̂ and ŷ areas, x̂g
    const int xh_base = off;
    for (int i = 0; i < nn + nfl; ++i) nodes[i].xh = xh_base + xh_of[i];
    for (int i = 0; i < own_end; ++i)  // internal nodes read [x̂_lo; x̂_hi] (adjacent)
      if (nodes[i].kind == 1) nodes[i].in = nodes[lo_idx[i]].xh;
    off += xh_total;
    P.yoff = xh_total;
    off += xh_total;
    P.xg_smem = off;
    {  // flat top: the chains M_d are staged into the x̂g area
      int m_off = off;
      for (int f = 0; f < nfl; ++f) {
        const int e = h->c_rank[root] * fl[f].kt;
        nodes[nn + f].pay = m_off;
        if (e > 0) {
          tp.copies.push_back(TCopy{(int64_t)tp.flat_all.size(), TS_FM, e, m_off, 0});
          tp.flat_all.insert(tp.flat_all.end(), fl[f].M.begin(), fl[f].M.end());
          m_off += e;
        }
      }
    }
    off += std::max(xg_rows, m_total);
    P.n_xg = n_xg_real;
    for (int32_t& g : gl)
      if (g <= -2) {
        const int v = -2 - g;
        g = ~(nodes[v >> 8].xh + (v & 255));
      }
    for (int i = 0; i < nn; ++i) {
      const int64_t gx = h->c_xoff[nd_p[i]];
      nodes[i].gx_lo = (int32_t)(uint32_t)gx;
      nodes[i].gx_hi = (int32_t)(gx >> 32);
    }
    if (off > budget_elems) return false;
    // gather list: staged as 16-byte elements (4 indices each)
    P.gidx_smem = gidx_smem;
    if (!gl.empty() || !frow.empty()) {  // [gather list | flat gather-row headers | entry bases]
      while (tp.gidx_all.size() % 4) tp.gidx_all.push_back(0);
      const int64_t first = (int64_t)tp.gidx_all.size() / 4;
      gl.resize((size_t)(n_rows + 3) / 4 * 4, 0);
      tp.gidx_all.insert(tp.gidx_all.end(), gl.begin(), gl.end());
      tp.gidx_all.insert(tp.gidx_all.end(), frow.begin(), frow.end());
      tp.gidx_all.insert(tp.gidx_all.end(), ebase_all.begin(), ebase_all.end());
      while (tp.gidx_all.size() % 4) tp.gidx_all.push_back(0);
      push_copy(TS_GIDX, first, (int)((int64_t)tp.gidx_all.size() / 4 - first), gidx_smem);
    }
    P.n_copy = (int)tp.copies.size() - P.copy_first;
    int64_t bytes = 0, sbytes = 0, tbytes = 0, fhbytes = 0;
    for (int c = P.copy_first; c < (int)tp.copies.size(); ++c)
      if (tp.copies[c].kind != TS_S || tp.copies[c].smem >= 0)
        (tp.copies[c].kind == TS_S ? sbytes
         : ts_late(tp.copies[c].kind) ? fhbytes
         : (tp.copies[c].kind == TS_T || tp.copies[c].kind == TS_FM) ? tbytes : bytes) +=
            16 * (int64_t)tp.copies[c].elems;
    if (sbytes >= (1 << 20) || tbytes >= (1 << 20)) return false;
    P.pad[1] = (int32_t)tbytes;
    if (bytes >= (1 << 20)) return false;  // one mbarrier transaction count
    P.stage_bytes = (int32_t)bytes;
    P.pad[0] = (int32_t)sbytes;
    {  // threads per node of the CTA-wide level operations: 2^shk >= every rank (column ops),
       // 2^shr >= every row count up to 32 (row ops loop over the rest)
      int kmax = 1, rmax = 1;
      for (int i = 0; i < nn + nfl; ++i) kmax = std::max(kmax, nodes[i].k);
      for (int i = 0; i < own_end; ++i) rmax = std::max(rmax, nodes[i].R);
      for (const FlatAnc& fa : fl) kmax = std::max(kmax, fa.kt);
      int shk = 0, shr = 0;
      while ((1 << shk) < kmax) ++shk;
      while ((1 << shr) < rmax && shr < 5) ++shr;
      if (shk > 5) return false;  // ranks above 32: not for this kernel
      P.pad[2] = shk | (shr << 8);
    }
    P.smem_elems = off;
    P.n_nodes = nn + nfl;
    P.nlev = nl;
    // transfer chains of a bottom program (see k_far_tree): in the staged coupling panels' region
    // (dead once the couplings are done) when it is large enough, else none
    P.f_base = -1;
    P.f_stride = 0;
    P.y_smem = 0;
    P.y_n = 0;
    P.y_g_lo = P.y_g_hi = 0;
    if (bottom && x_smem >= 0 && !getenv("H2B_TREE_Y_ATOMIC")) {
      P.y_smem = x_smem;
      P.y_n = h->c_size[root];
      P.y_g_lo = (int32_t)(uint32_t)(int64_t)h->c_start[root];
      P.y_g_hi = (int32_t)((int64_t)h->c_start[root] >> 32);
    }
    if (nfl > 0) {
      P.f_base = flat_f_base;
      P.f_stride = flat_f_stride;
      P.split_mode = 2;
    } else if (bottom && stage_s && s_total > 0 && !getenv("H2B_TREE_NO_SPLIT")) {
      int kmax = 0;
      for (int i = 0; i < nn; ++i) kmax = std::max(kmax, nodes[i].k);
      const int64_t need = (int64_t)nn * kmax * nodes[0].k;
      if (need > 0 && need <= s_total && nodes[0].k > 0 && kmax <= 32) {
        P.f_base = s_first;
        P.f_stride = kmax * nodes[0].k;
        P.split_mode = 1;
      }
    }
    for (int d = 0; d <= nl; ++d) P.lev_first[d] = lev_first[d];
    P.gidx_smem = gidx_smem;
    tp.nodes_all.insert(tp.nodes_all.end(), nodes.begin(), nodes.end());
    tp.smem_max = std::max(tp.smem_max, 16 * off);
    tp.progs.push_back(P);
    return true;
  }
};

}  // namespace

// Plan the tree far field for handle h (q = 1).  Returns false when the tree does not qualify or
// the programs do not fit (the caller keeps the task-graph kernel).
bool h2b_plan_tree(const h2b_ctx* h, int max_ctas, int budget_bytes, int flat_budget_bytes, const double2* hT,
                   const double2* hS, TreePlan& tp) {
  if (getenv("H2B_NO_TREE") || h->K == 0 || !tree_shape_ok(h)) return false;
  const int L = h->depth;
  int lt = -1;
  for (int l = 0; l < L && lt < 0; ++l)
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p)
      if (h->c_rank[p] > 0) {
        lt = l;
        break;
      }
  if (lt < 0) return false;
  const int budget = budget_bytes / 16;
  for (int ls = L - 1; ls >= lt; --ls) {  // the deepest split whose programs fit the grid
    const int nb = 1 << ls;
    int nt = ls > lt ? (1 << lt) : 0;
    if (nb + nt > max_ctas) continue;
    TreePlan cand;
    bool ok = false;
    // flat top first (no top programs): up to 5 levels above the split (2^d partials per gathered
    // entry sit on one warp's lanes), ranks <= 32 there
    if (ls > lt && ls - lt <= 5 && hT && hS && flat_budget_bytes > 0 && !getenv("H2B_TREE_NO_FLAT")) {
      int kp = 0;
      for (int p = h->level_ptr[lt]; p < h->level_ptr[ls]; ++p) kp = std::max(kp, h->c_rank[p]);
      if (kp <= 32 && kp > 0) {
        Builder B{h, cand};
        B.hT = hT;
        B.hS = hS;
        B.ls = ls;
        B.lt = lt;
        B.nb = nb;
        B.kp = kp;
        B.flat = true;
        ok = true;
        for (int i = 0; i < nb && ok; ++i) ok = B.build(h->level_ptr[ls] + i, L - 1, true, flat_budget_bytes / 16);
        if (ok) {
          cand.flat = true;
          cand.px_elems = (int64_t)(ls - lt) * nb * kp;
          nt = 0;
        } else {
          cand = TreePlan();
        }
      }
    }
    if (!ok) {
      Builder B{h, cand};
      ok = true;
      for (int i = 0; i < nb && ok; ++i) ok = B.build(h->level_ptr[ls] + i, L - 1, true, budget);
      for (int i = 0; i < nt && ok; ++i) ok = B.build(h->level_ptr[lt] + i, ls - 1, false, budget);
    }
    if (!ok) continue;
    // dependencies: program of each cluster (bottom: level >= ls; top: lt <= level < ls)
    std::vector<int> prog_of(h->P, -1);
    for (int i = 0; i < nb; ++i) {
      const int r = h->level_ptr[ls] + i;
      for (int d = 0; ls + d < L; ++d)
        for (int j = 0; j < (1 << d); ++j) prog_of[h->level_ptr[ls + d] + (i << d) + j] = i;
    }
    for (int i = 0; i < nt; ++i)
      for (int d = 0; lt + d < ls; ++d)
        for (int j = 0; j < (1 << d); ++j) prog_of[h->level_ptr[lt + d] + (i << d) + j] = nb + i;
    for (int pi = 0; pi < nb + nt; ++pi) {
      TProg& P = cand.progs[pi];
      const bool bottom = pi < nb;
      const int root = bottom ? h->level_ptr[ls] + pi : h->level_ptr[lt] + (pi - nb);
      const int rl = bottom ? ls : lt;
      const int last = bottom ? L - 1 : ls - 1;
      std::set<int> up;
      for (int d = 0; rl + d <= last; ++d)
        for (int j = 0; j < (1 << d); ++j) {
          const int t = h->level_ptr[rl + d] + ((root - h->level_ptr[rl]) << d) + j;
          if (h->c_rank[t] == 0) continue;
          for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
            const int s = h->s_col[b];
            if (h->c_rank[s] > 0 && prog_of[s] != pi) up.insert(prog_of[s]);
          }
        }
      std::set<int> far;
      if (cand.flat)  // the bottom programs below every source of every ancestor (their partials)
        for (int d = 1; d <= ls - lt; ++d) {
          const int t = h->level_ptr[ls - d] + (pi >> d);
          if (h->c_rank[t] == 0) break;
          for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
            const int s = h->s_col[b];
            if (h->c_rank[s] == 0) continue;
            const int si = s - h->level_ptr[ls - d];
            for (int j = 0; j < (1 << d); ++j)
              if ((si << d) + j != pi) far.insert((si << d) + j);
          }
        }
      P.wait_up_first = (int)cand.waits.size();
      P.n_wait_up = (int)up.size();
      cand.waits.insert(cand.waits.end(), up.begin(), up.end());
      P.wait_far_first = (int)cand.waits.size();
      P.n_wait_far = (int)far.size();
      cand.waits.insert(cand.waits.end(), far.begin(), far.end());
      if (!bottom) {  // external children: the bottom programs under this top program
        P.ext_wait_first = (int)cand.waits.size();
        const int d = ls - lt;
        const int first = (root - h->level_ptr[lt]) << d;
        P.n_ext_wait = 1 << d;
        for (int j = 0; j < (1 << d); ++j) cand.waits.push_back(first + j);
      } else if (ls > lt && !cand.flat) {
        const int parent_top = nb + (pi >> (ls - lt));
        // only when the parent carries rank (otherwise the top writes nothing for this root)
        int par = h->level_ptr[ls - 1] + (pi >> 1);
        P.wait_down = h->c_rank[par] > 0 ? parent_top : -1;
      }
    }
    cand.ls = ls;
    cand.lt = lt;
    cand.n_rows_total = h->n;
    cand.n_bottom = nb;
    cand.n_top = nt;
    tp = std::move(cand);
    return true;
  }
  return false;
}

// device state of the tree far field
struct TreeDev {
  TProg* progs = nullptr;
  TCopy* copies = nullptr;
  int32_t* waits = nullptr;
  TNode* nodes = nullptr;
  int32_t* gidx = nullptr;
  double2* flat = nullptr;    // flat top: transfer chains and H panels
  double2* px = nullptr;      // flat top: partial x̂ (zero where a chain ends at a rank-0 ancestor)
  uint32_t* flags = nullptr;  // up [n], down [n]
  MegaCtrl* ctrl = nullptr;
  uint64_t* trace = nullptr;
  int n_progs = 0, smem = 0;
  bool zero_ok = false;
  ZeroSync* zsync = nullptr;  // h2b_tree_prepare_zero
  int2* zrows = nullptr;      // the near-field CTAs' rows of y
  int zrows_n = 0;
  int rows_per_prog = 0;      // rows of y per bottom program (equal for all when zero_ok)
};

namespace {
template <typename T>
int upload_vec(T** dst, const std::vector<T>& v) {
  const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  H2B_CUDA_TRY(cudaMalloc((void**)dst, bytes));
  if (!v.empty()) H2B_CUDA_TRY(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return H2B_OK;
}
}  // namespace

int h2b_tree_upload(const TreePlan& tp, TreeDev** out, int64_t* bytes) {
  TreeDev* d = new TreeDev();
  int rc = upload_vec(&d->progs, tp.progs);
  if (!rc) rc = upload_vec(&d->copies, tp.copies);
  if (!rc) rc = upload_vec(&d->waits, tp.waits);
  if (!rc) rc = upload_vec(&d->nodes, tp.nodes_all);
  if (!rc) rc = upload_vec(&d->gidx, tp.gidx_all);
  if (!rc) rc = upload_vec(&d->flat, tp.flat_all);
  if (!rc) {
    const size_t pb = 16 * (size_t)std::max<int64_t>(tp.px_elems, 1);
    H2B_CUDA_TRY(cudaMalloc((void**)&d->px, pb));
    H2B_CUDA_TRY(cudaMemset(d->px, 0, pb));
  }
  d->n_progs = (int)tp.progs.size();
  if (!rc) {
    const cudaError_t e1 = cudaMalloc(&d->flags, sizeof(uint32_t) * 2 * std::max(d->n_progs, 1));
    const cudaError_t e2 = cudaMalloc(&d->ctrl, sizeof(MegaCtrl));
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      h2b_set_error("h2b_tree_upload: allocation failed");
      rc = H2B_ENOMEM;
    } else {
      cudaMemset(d->flags, 0, sizeof(uint32_t) * 2 * std::max(d->n_progs, 1));
      cudaMemset(d->ctrl, 0, sizeof(MegaCtrl));
    }
  }
  d->smem = tp.smem_max;
  {
    int64_t rows = 0;
    bool all = true;
    for (const TProg& P : tp.progs)
      if (P.bottom) {
        all = all && P.y_n > 0;
        rows += P.y_n;
      }
    // (programs in row order, equal row counts: the near-field CTAs map rows to programs by division)
    int rpp = 0;
    for (size_t i = 0; i < tp.progs.size(); ++i) {
      const TProg& P = tp.progs[i];
      if (!P.bottom) continue;
      if (rpp == 0) rpp = P.y_n;
      const int64_t yg = (int64_t)(uint32_t)P.y_g_lo | ((int64_t)P.y_g_hi << 32);
      all = all && P.y_n == rpp && yg == (int64_t)i * rpp;
    }
    d->zero_ok = all && rows == tp.n_rows_total && rpp > 0;
    d->rows_per_prog = rpp;
  }
  if (!rc && getenv("H2B_TREE_TRACE")) {
    cudaMalloc(&d->trace, sizeof(uint64_t) * 32 * std::max(d->n_progs, 1));
    cudaMemset(d->trace, 0, sizeof(uint64_t) * 32 * std::max(d->n_progs, 1));
  }
  if (!rc) {
    const cudaError_t e = cudaFuncSetAttribute(k_far_tree, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 14000);
    cudaFuncSetAttribute(k_far_tree, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_far_tree_traced, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 14000);
    cudaFuncSetAttribute(k_far_tree_traced, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) {
      h2b_set_error(std::string("k_far_tree attributes: ") + cudaGetErrorString(e));
      rc = H2B_ECUDA;
    }
  }
  *bytes = (int64_t)(sizeof(TProg) * tp.progs.size() + sizeof(TCopy) * tp.copies.size() +
                     sizeof(TNode) * tp.nodes_all.size() + 4 * tp.gidx_all.size() + 16 * tp.flat_all.size() +
                     16 * tp.px_elems);
  *out = d;
  return rc;
}

void h2b_tree_free(TreeDev* d) {
  if (!d) return;
  void* ptrs[] = {d->progs, d->copies, d->waits, d->nodes, d->gidx, d->flat, d->px, d->flags, d->ctrl, d->trace,
                  d->zsync, d->zrows};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete d;
}

int h2b_tree_static_smem() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_far_tree) != cudaSuccess) {
    cudaGetLastError();
    return 1024;
  }
  return (int)fa.sharedSizeBytes;
}

int h2b_tree_regs() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_far_tree) != cudaSuccess) {
    cudaGetLastError();
    return 255;
  }
  return fa.numRegs;
}

int h2b_tree_error(const TreeDev* d, uint32_t* err) {
  MegaCtrl c{};
  H2B_CUDA_TRY(cudaMemcpy(&c, d->ctrl, sizeof(c), cudaMemcpyDeviceToHost));
  *err = c.error;
  return H2B_OK;
}

// plan + upload for handle h; *planned = 0 when the tree does not qualify (k_mega stays)
int h2b_tree_prepare(h2b_ctx* h, int max_ctas, int budget_bytes, int64_t* bytes, int* planned) {
  *planned = 0;
  *bytes = 0;
  TreePlan tp;
  // flat top: host copies of the transfer matrices and the (already transposed) coupling panels
  std::vector<double2> hT, hS;
  const int flat_budget = getenv("H2B_TREE_NO_FLAT") ? 0 : budget_bytes + TREE_FLAT_EXTRA;
  if (flat_budget > 0 && h->sec_elems[1] > 0 && h->sec_elems[2] > 0 &&
      h->sec_elems[1] + h->sec_elems[2] <= (int64_t)(1 << 26)) {
    hT.resize((size_t)h->sec_elems[1]);
    hS.resize((size_t)h->sec_elems[2]);
    H2B_CUDA_TRY(cudaMemcpy(hT.data(), h->buf[H2B_SEC_T], 16 * hT.size(), cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(hS.data(), h->buf[H2B_SEC_S], 16 * hS.size(), cudaMemcpyDeviceToHost));
  }
  if (!h2b_plan_tree(h, max_ctas, budget_bytes, flat_budget, hT.empty() ? nullptr : hT.data(),
                     hS.empty() ? nullptr : hS.data(), tp))
    return H2B_OK;
  H2B_TRY(h2b_tree_upload(tp, &h->tree, bytes));
  h->tree_ls = tp.ls;
  h->tree_lt = tp.lt;
  h->tree_progs = (int)tp.progs.size();
  h->tree_smem = tp.smem_max;
  h->tree_flat = tp.flat ? 1 : 0;
  h->tree_rows_per_prog = h->tree->rows_per_prog;
  *planned = 1;
  return H2B_OK;
}

// one launch of the far field on `st` (cooperative: the programs wait on one another)
// the zeroing protocol's state (ZeroSync, h2b_common.cuh) when every far-field contribution to
// y is a bottom program's bulk add (which checks its rows' ranges first); else nullptr.  Allocated
// here on first use (never inside a capture: h2b_launch_mega is reached through h2b_prepare'd
// handles whose first matvec runs this before capturing — cudaMalloc is legal in thread-local
// capture mode only outside the capturing stream, so it is done in h2b_tree_prepare_zero).
ZeroSync* h2b_tree_zero_sync(h2b_ctx* h, TreeDev* d) {
  (void)h;
  return d && d->zero_ok ? d->zsync : nullptr;
}

int h2b_tree_prepare_zero(h2b_ctx* h, TreeDev* d) {
  if (!d || !d->zero_ok || d->zsync || !h->near_zero_ok || h->near_grid > NEAR_MAXG) return H2B_OK;
  for (const int2& zr : h->near_zero_row)  // a CTA's rows span at most ZS_SLOTS programs
    if (zr.y > 0 && (zr.x + zr.y - 1) / d->rows_per_prog - zr.x / d->rows_per_prog + 1 > ZS_SLOTS) return H2B_OK;
  H2B_CUDA_TRY(cudaMalloc((void**)&d->zsync, sizeof(ZeroSync)));
  H2B_CUDA_TRY(cudaMemset(d->zsync, 0, sizeof(ZeroSync)));
  H2B_CUDA_TRY(cudaMalloc((void**)&d->zrows, sizeof(int2) * std::max<size_t>(h->near_zero_row.size(), 1)));
  H2B_CUDA_TRY(cudaMemcpy(d->zrows, h->near_zero_row.data(), sizeof(int2) * h->near_zero_row.size(),
                          cudaMemcpyHostToDevice));
  d->zrows_n = (int)h->near_zero_row.size();
  return H2B_OK;
}

int h2b_launch_tree(h2b_ctx* h, const TreeDev* d, const double2* xp, double2* yp, cudaStream_t st, int near_ctas) {
  TreeArgs A;
  A.zs = near_ctas > 0 ? d->zsync : nullptr;
  A.zrows = d->zrows;
  A.near_ctas = A.zs ? std::min(near_ctas, d->zrows_n) : 0;
  A.progs = d->progs;
  A.copies = d->copies;
  A.waits = d->waits;
  A.src[TS_X] = xp;
  A.src[TS_V] = h->buf[H2B_SEC_V];
  A.src[TS_T] = h->buf[H2B_SEC_T];
  A.src[TS_S] = h->buf[H2B_SEC_S];
  A.src[TS_NODES] = d->nodes;
  A.src[TS_GIDX] = d->gidx;
  A.src[TS_FM] = d->flat;
  A.src[TS_FH] = d->flat;
  A.src[TS_FF] = d->flat;
  A.px = d->px;
  A.xhat = h->xhat;
  A.yhat = h->yhat;
  A.y = yp;
  A.flags_up = d->flags;
  A.flags_down = d->flags + d->n_progs;
  A.ctrl = d->ctrl;
  A.trace = d->trace;
  {
    const char* e = getenv("H2B_TREE_TRACE");
    A.trace_levels = e ? atoi(e) : 0;
    const char* d = getenv("H2B_TREE_DEFER_S");  // A/B aid
    // bit 0: coupling panels, bit 2: transfers and chains requested once the leaf-level operands
    // have landed (measured at cfg2: panels 40.3 vs 41.0 us; transfers too: mean 33.6 -> 33.0 us)
    A.defer_s = d ? atoi(d) : 5;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(d->n_progs);
  cfg.blockDim = dim3(TNT);
  cfg.dynamicSmemBytes = d->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  static const bool nocoop = getenv("H2B_TREE_NOCOOP") != nullptr;  // A/B aid
  cfg.numAttrs = nocoop ? 0 : 1;
  if (A.trace)
    H2B_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_far_tree_traced, A));
  else
    H2B_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_far_tree, A));
  return H2B_OK;
}

// development aid: the per-program timeline of the last launch (H2B_TREE_TRACE set at prepare):
// out[32 * i + j] = timestamp j of program i (ns, globaltimer; 0 = not reached; SM clock64 at
// out[32 * i + 16 + j]), programs
// [0, n_bottom) bottom, then top
extern "C" int h2b_tree_trace(h2b_handle h, int64_t* out, int64_t max_progs) {
  if (!h || !out || !h->tree || !h->tree->trace) {
    h2b_set_error("h2b_tree_trace: no tree trace (set H2B_TREE_TRACE before the first matvec)");
    return H2B_ESTATE;
  }
  const int64_t n = std::min<int64_t>(max_progs, h->tree->n_progs);
  H2B_CUDA_TRY(cudaDeviceSynchronize());
  H2B_CUDA_TRY(cudaMemcpy(out, h->tree->trace, sizeof(uint64_t) * 32 * n, cudaMemcpyDeviceToHost));
  return H2B_OK;
}
