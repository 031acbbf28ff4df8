// Shared device helpers and the handle layout of the h2b C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/h2b.h"

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI entry returns an int status and records a message
// ---------------------------------------------------------------------------
void h2b_set_error(const std::string& msg);

#define H2B_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      cudaGetLastError(); /* do not leave a non-sticky error for the next check */   \
      h2b_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
      return _e == cudaErrorMemoryAllocation ? H2B_ENOMEM : H2B_ECUDA;              \
    }                                                                               \
  } while (0)

#define H2B_STR2(x) #x
#define H2B_STR(x) H2B_STR2(x)
#define H2B_CHECK_LAUNCH()                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      h2b_set_error(std::string("kernel launch at " __FILE__ ":" H2B_STR(__LINE__) ": ") + \
                    cudaGetErrorString(_e));                                        \
      return H2B_ECUDA;                                                             \
    }                                                                               \
  } while (0)

#define H2B_TRY(x)        \
  do {                    \
    int _rc = (x);        \
    if (_rc) return _rc;  \
  } while (0)

// ---------------------------------------------------------------------------
// complex128 arithmetic on interleaved double2 (no fast-math)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  return v;
}

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = cadd(v, shfl_xor2(v, m));
  return v;
}

// 256-bit streaming load (sm_100: LDG.E.ENL2.256), read-only, no L1 allocation.
struct __align__(32) cd2 {
  double2 a, b;
};
__device__ __forceinline__ cd2 ld_stream256(const double2* p) {
  cd2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.a.x), "=d"(r.a.y), "=d"(r.b.x), "=d"(r.b.y)
               : "l"(p));
  return r;
}
// 256-bit load through L1 (operands re-read by neighbouring warps)
__device__ __forceinline__ cd2 ld_cached256(const double2* p) {
  cd2 r;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.a.x), "=d"(r.a.y), "=d"(r.b.x), "=d"(r.b.y)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// span programs: a span is a piece of the cluster tree (a subtree below the
// split level, the levels above it, or a single cluster) processed by ONE CTA
// entirely in shared memory.  The host resolves everything at prepare time
// into three descriptor lists per span: bulk copies global->smem (payload,
// inputs and the op list itself), ops (small panel GEMVs on smem offsets,
// grouped into levels separated by __syncthreads) and copies smem->global.
// ---------------------------------------------------------------------------
enum SpanSrc : int32_t {
  SRC_V = 0, SRC_T, SRC_VT, SRC_TT, SRC_X, SRC_XHAT, SRC_YHAT, SRC_OPS, SRC_OUTS, SRC_N
};
struct SpanCopy {        // global (base[kind] + src) <-> smem[smem], elems double2 (32 bytes)
  int64_t src;
  int32_t kind, elems, smem, pad;
  int64_t pad2;
};
struct SpanOp {          // out[c] (+)= sum_r P[r*w+c] in[r], c < w, r < R
  int32_t pay, in, out, R, w, flags, pad0, pad1;
};
constexpr int OP_ACC = 1;       // accumulate into out
constexpr int OP_OUT_Y = 2;     // out is an element offset into global y, not smem
constexpr int OP_OUT_YD = 4;    // with OP_OUT_Y: into y_deep instead (overwrite), see FlatRec
constexpr int SPAN_MAXLEV = 24;
struct SpanHead {
  int32_t copy_first, n_copy, out_first, n_out;
  int32_t ops_smem, n_ops, smem_elems, nlev;
  int32_t lvl[SPAN_MAXLEV + 1];  // op boundaries of each level, execution order
  int32_t pad[3];
};
struct SpanLaunch {      // one kernel launch of the far-field chain
  int32_t head_first, n_heads, smem_elems, big;  // big: 1024-thread CTA
  int32_t level;         // >= 0: per-level fallback kernel for this level instead
};

// near-field work lists (q = 1 fast path)
struct NearItem {        // one CTA: RB rows of one target leaf
  int64_t y_off;         // first permuted row written by the CTA
  int32_t b_first, nb;   // partner-block range in the NearBlk list (shared by the leaf's items)
  int32_t row0, pad;     // first row of the item within the leaf
};
struct NearBlk {
  int64_t d_off;         // element offset of the partner block D_{t,s}
  int64_t x_off;         // first permuted column of the partner leaf
};
// coupling work list
struct CoupleItem {
  int64_t panel;         // element offset of the target's S^T panel (R x w)
  int64_t xcol;          // offset into s_xcol of the panel's first row
  int64_t out;           // x̂/ŷ offset of the target
  int32_t R, w;
};

// ---------------------------------------------------------------------------
// persistent matvec kernel (q = 1): one launch executes a task graph.  CTAs
// claim tasks in queue order from an atomic counter; a task waits only on
// tasks with smaller ids (claimed by running CTAs), so progress is guaranteed.
// Completion flags are epoch-stamped, so nothing is reset between matvecs.
// ---------------------------------------------------------------------------
enum TaskType : int32_t { T_NEAR = 0, T_SPAN = 1, T_COUPLE = 2, T_FLAT_UP = 3, T_FLAT_DOWN = 4 };
// Flattened bottom tier (see plan_mega): for a cluster c at the split level ls,
// W_c = [V_l T_l T_parent(l) ... ]_{leaves l of c} (n_c x k_c, row-major) maps the points of c
// straight to x̂_c (T_FLAT_UP: x̂_c = W_cᵀ x_c) and ŷ_c straight back (T_FLAT_DOWN:
// y_c += W_c ŷ_c + y_deep_c, y_deep = what the levels below ls add, written by "deep" spans).
struct FlatRec {
  int64_t w_off;    // element offset of W_c in the flattened-basis buffer
  int64_t x_off;    // first point of c (x / y / y_deep offset)
  int64_t hat_off;  // x̂ / ŷ offset of c
  int32_t n, k;     // points and rank of c
};
struct Task {
  int32_t type, arg;        // arg: near task / span head / couple group index
  int32_t dep_first, n_dep; // ranges [dep_first, dep_first + n_dep) of DepRange
  int64_t rec_off;          // self-contained task record: 16-byte slots in the record pool
  int32_t rec_len, pad;     // (bulk-loaded into shared memory one task ahead)
};
// Record layouts (16-byte slots):
//   near:   {n_blocks, n_leaves, row0, 0} | n_leaves x {y_off:i64, nb:i32, 0} |
//           n_blocks x {d_off:i64 (row0 applied), x_off:i64}
//   span:   SpanHead (9 slots) | n_copy x SpanCopy (2 slots each)
//   couple: {n_items, cta_mode, 0, 0} | n_items x CoupleItem (2 slots each)
constexpr int REC_SLOTS = 256;  // 4 KB per record buffer
constexpr int NEAR_NRB = 8;      // near-field stream: record buffers (the task in use + NRB - 1 claimed ahead)
constexpr int NEAR_MAXG = 192;  // CTAs of the near stream with kernel-parameter first copies
constexpr int NEAR_REC_MAXB = 160;
struct DepRange {
  int32_t lo, hi;           // task ids [lo, hi) that must be complete
};
struct NearTask {
  int32_t leaf_first, n_leaves;  // consecutive entries of the leaf work list
  int32_t row0, pad;             // first row (when one leaf is split across tasks)
};
struct CoupleGroup {
  int32_t item_first, n_items, cta_mode, pad;
};
// Zeroing of y without a memset node (q = 1 tree step, r02).  Every row of y gets exactly one
// far-field contribution (the bulk add of the bottom program covering it, at that program's
// end) and one near-field contribution (from the one near-field CTA owning it).  Each bottom
// program zeroes its own rows at its START (no atomics, behind its staging wait) and then sets
// flag[c][j] = 1 (release) for every near-field CTA c whose rows overlap its own (it is the j-th
// program of that CTA's range); CTA c waits for its flags before its consumers start — while
// its producer fills the ring, before the first block can have landed — and clears them for the
// next step (it is their only reader).  Nothing is added to either kernel's critical path and
// nothing inside the near-field consumer loop.  Ordering: the far-field kernel is launched
// first, so it also runs first when launches are serialised (profilers); a near-field CTA whose
// flags never come (bounded wait) reports device error 4 instead of hanging.
// H2B_Y_MEMSET=1 selects the memset node instead.
constexpr int ZS_SLOTS = 4;  // programs a near-field CTA's rows may span
struct ZeroSync {
  uint32_t flag[NEAR_MAXG + 8][ZS_SLOTS];
};

struct MegaCtrl {
  uint32_t next, exited, epoch, error;  // far-field task graph
  uint32_t near_next, near_exited;      // near-field stream: task claim counter, CTAs done
  uint32_t pad[2];
};

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct GraphKey {
  const void* x;
  void* y;
  int q;
  bool operator<(const GraphKey& o) const { return std::tie(x, y, q) < std::tie(o.x, o.y, o.q); }
};

struct MrhsPlan;  // h2b_mrhs.cu
struct TreeDev;   // h2b_tree.cu

struct GmresKey {  // one captured Arnoldi step of h2b_gmres
  const void* V;
  int j, m;
  int64_t n;
  bool operator<(const GmresKey& o) const { return std::tie(V, j, m, n) < std::tie(o.V, o.j, o.m, o.n); }
};

struct h2b_ctx {
  int device = 0;
  int64_t n = 0;
  int depth = 0;
  int P = 0;
  int64_t K = 0;
  int64_t n_coupling = 0, n_near = 0;
  int64_t sec_elems[4] = {0, 0, 0, 0};
  int64_t sec_uploaded[4] = {0, 0, 0, 0};  // elements covered by the uploaded chunks
  std::map<int64_t, int64_t> sec_iv[4];     // merged [begin, end) element ranges uploaded
  bool prepared = false;  // device-side transposes / tables done
  int uniform_leaf = 0;   // leaf size if all leaves share it, else 0

  // host copies of the tables
  std::vector<int32_t> level_ptr, c_rank, c_child_lo, c_child_hi, c_size, c_start;
  std::vector<int64_t> c_xoff, c_voff, c_toff, s_row_ptr, s_off, d_row_ptr;
  std::vector<int32_t> s_col, d_col;
  std::vector<int64_t> d_off;
  std::vector<int32_t> up_levels;    // levels with any k>0 cluster (deepest first)
  std::vector<int32_t> down_levels;  // levels with any non-leaf k>0 cluster (root first)
  std::vector<int32_t> h_leaves;

  // device tables
  int32_t *c_start_d = nullptr, *c_size_d = nullptr, *c_rank_d = nullptr, *c_lo = nullptr,
          *c_hi = nullptr, *c_parent = nullptr;
  int64_t *c_xoff_d = nullptr, *c_voff_d = nullptr, *c_toff_d = nullptr;
  int64_t *s_row_ptr_d = nullptr, *s_off_d = nullptr, *d_row_ptr_d = nullptr, *d_off_d = nullptr;
  int64_t* s_prow = nullptr;  // [P] first coupling-panel row of each target
  int32_t* s_xcol = nullptr;  // [panel rows] x̂ index feeding each panel row
  int32_t *s_col_d = nullptr, *d_col_d = nullptr;
  int64_t* perm = nullptr;
  int32_t* leaves = nullptr;
  int n_leaves = 0;
  int32_t* couple_targets = nullptr;  // clusters with k > 0
  int n_couple_targets = 0;
  // payloads: V, T, Sᵀ (transposed in place), D ; plus transposed copies Vᵀ, Tᵀ
  double2* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  double2 *vT = nullptr, *tT = nullptr;
  // q = 1 far-field programs
  int span_mode = 0;  // 0: per-level kernels only, 1: span programs
  int ls = 0, top_staged = 0;
  std::vector<SpanLaunch> up_prog, down_prog_head, down_prog_tail;
  SpanHead* span_heads = nullptr;
  SpanCopy* span_copies = nullptr;
  SpanCopy* span_outs = nullptr;
  SpanOp* span_ops = nullptr;
  // persistent-kernel task graph (q = 1)
  int mega = 0;                  // 1: q = 1 matvec is one persistent launch
  int mega_ns = 0, mega_r = 1;   // near variant (0 generic, 32, 64) and rows per thread
  int mega_grid = 0, mega_smem = 0, n_tasks = 0;
  Task* tasks = nullptr;
  int4* rec_pool = nullptr;      // task records
  int4* l2_prefetch = nullptr;   // {ptr lo/hi, bytes} ranges warmed into L2 at kernel start
  int n_prefetch = 0;
  DepRange* deps = nullptr;
  NearTask* near_tasks = nullptr;
  NearItem* leaf_items = nullptr;  // per leaf: y offset, partner-block range
  CoupleGroup* couple_groups = nullptr;
  MegaCtrl* ctrl = nullptr;
  uint32_t* flags = nullptr;
  int mega_tiers = 0;
  int mega_debug = 0;                  // H2B_OPT_DEBUG (profiling only: results are wrong)
  int2* cta_lists = nullptr;           // per CTA {first, count} into task_list
  int* task_list = nullptr;            // static per-CTA task runs (global topological order)
  double mega_est_us = 0.0;            // planner's makespan estimate
  int mega_blob_slots = 0;             // largest per-CTA task blob (16-byte slots)
  uint64_t* trace = nullptr;           // optional per-task timeline (H2B_OPT_TRACE)
  std::vector<Task> h_tasks;           // host copy of the task list
  // near-field stream kernel (runs beside the far-field task graph; both add into a zeroed y)
  int4* near_recs = nullptr;           // near task records
  int2* near_idx = nullptr;            // per near task {first slot, slots}
  int64_t* iperm = nullptr;         // inverse of perm (original index -> packed), host path
  uint64_t* near_trace = nullptr;  // H2B_NEAR_TRACE: stamps per near CTA
  int near_early = 0;               // first record / block per CTA known at plan time
  std::vector<int2> near_first_rec;
  std::vector<longlong2> near_first_blk;
  // static split: CTA c's rows of y {first, count} (each row belongs to exactly one CTA) and
  // whether they tile [0, n) — then the near kernel zeroes y itself (no memset node)
  std::vector<int2> near_zero_row;
  int near_zero_ok = 0;
  int n_near_tasks = 0, near_rec_max = 0, near_nst = 0, near_smem = 0, near_grid = 0;
  uint32_t near_delay_ns = 0;  // tuning aid (H2B_DEBUG_NEAR_DELAY_NS)
  int near_static = 0;         // near tasks split statically over the CTAs (H2B_NEAR_STATIC)
  int near_dbg = 0;            // profiling only (H2B_NEAR_DBG): see NearArgs::dbg
  // far field as subtree programs (h2b_tree.cu): replaces k_mega beside k_near_stream when set
  TreeDev* tree = nullptr;
  int use_tree = 1;  // H2B_OPT_TREE
  int tree_ls = 0, tree_lt = 0, tree_progs = 0, tree_smem = 0, tree_flat = 0, tree_rows_per_prog = 0;
  // flattened bottom tier (0 = off): W buffer and the deep spans' y_deep
  int mega_flat = 0;
  double2* wbuf = nullptr;
  double2* ydeep = nullptr;
  // near / coupling work lists
  NearItem* near_items = nullptr;
  NearBlk* near_blks = nullptr;
  int n_near_items = 0, near_rb = 0;
  CoupleItem* couple_items = nullptr;
  int n_couple_items = 0, couple_warp_mode = 0;
  // workspace (grown on demand, per q)
  double2 *xhat = nullptr, *yhat = nullptr;
  int64_t ws_q = 0;
  double2 *hxp = nullptr, *hyp = nullptr;  // host-path staging
  void* hpin = nullptr;                     // pinned host staging of pageable x / y
  size_t hpin_bytes = 0;
  int64_t hws_q = 0;
  // streams / events / graphs
  cudaStream_t far_stream = nullptr;
  cudaStream_t host_stream = nullptr;  // h2b_matvec_host
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GmresKey, cudaGraphExec_t> gmres_graphs;  // per-step graphs of h2b_gmres
  int use_graphs = 1;
  int use_mega = 1;  // plan the persistent single-launch kernel for q = 1
  // krylov workspace
  void* kry = nullptr;
  // per-handle Krylov scratch on this handle's device (h2b_krylov.cu): reduction partials,
  // device scalars and mapped pinned host records (GMRES residuals / BiCGStab records in
  // separate slots)
  double2 *ks_partial = nullptr, *ks_vals = nullptr, *ks_host = nullptr;
  // device-side ordering of this handle's work across caller streams: every matvec / solve
  // waits for the previous one (whatever stream it ran on) and records ev_done after itself,
  // because the captured graphs share x̂/ŷ, control flags and workspaces
  cudaEvent_t ev_done = nullptr;
  size_t kry_bytes = 0;
  int64_t device_bytes = 0;
  int launches_q1 = 0;  // kernels per q=1 matvec (reported to the bench)
  // multi-RHS (q >= 2) grouped complex GEMM plan on the FP64 tensor pipe (h2b_mrhs.cu)
  MrhsPlan* mrhs = nullptr;
  int use_mrhs = 1;
};

// implemented in h2b_matvec.cu
int h2b_prepare(h2b_ctx* h);
int h2b_ensure_workspace(h2b_ctx* h, int q);
int h2b_run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st);
// the launches of one matvec without graph replay (for capture into a larger graph)
int h2b_enqueue_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl);
// the handle's Krylov workspace (h2b_krylov.cu), shared by the solvers of one handle
int h2b_krylov_workspace(h2b_ctx* h, size_t bytes, double2** out);
// cross-stream ordering of the handle's device work (see h2b_ctx::ev_done)
int h2b_order_begin(h2b_ctx* h, cudaStream_t st);
int h2b_order_end(h2b_ctx* h, cudaStream_t st);
int h2b_run_phase(h2b_ctx* h, int phase, const double2* xp, double2* yp, int q, cudaStream_t st);
int h2b_launch_gather(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                      cudaStream_t st);
int h2b_launch_host_in(const double2* xh, const int64_t* iperm, int64_t n, double2* out, int q, cudaStream_t st);
int h2b_launch_host_out(const double2* in, const int64_t* iperm, int64_t n, double2* yh, int q, cudaStream_t st);
int h2b_ensure_iperm(h2b_ctx* h);
int h2b_launch_scatter(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                       cudaStream_t st);
void h2b_release_graphs(h2b_ctx* h);
// implemented in h2b_mrhs.cu
int h2b_mrhs_prepare(h2b_ctx* h);
void h2b_mrhs_free(h2b_ctx* h);
int h2b_mrhs_launches(const h2b_ctx* h);
int h2b_mrhs_workspace(h2b_ctx* h, int q);
int h2b_launch_mrhs(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl);

// ---------------------------------------------------------------------------
// Blackwell async bulk copy (TMA 1-D, cp.async.bulk) + mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  // try_wait without a suspend-time hint: the default (short) timeout keeps the waiting warps
  // responsive to a completing transaction.  A phase that never completes is a bug: trap
  // (the launch fails with an error) instead of hanging the GPU.
  for (uint32_t spins = 0; !mbar_try_wait(bar, phase);)
    if (++spins == (1u << 26)) __trap();
}
// The same on shared-window addresses computed once (smem_u32 before a loop): inside a
// latency-bound loop the generic-to-shared conversion of every call re-reads SR_CgaCtaId
// (S2UR + ULEA + IMAD, ~10 % of the near-field consumer's stall samples)
__device__ __forceinline__ void mbar_arrive_expect_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_a(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t phase) {
  for (uint32_t spins = 0; !mbar_try_wait_a(bar, phase);)
    if (++spins == (1u << 26)) __trap();
}
// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
