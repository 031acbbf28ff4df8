/*
 * h2b.h — C ABI of the B200-native H² matvec + Krylov hot path.
 *
 * The reference (`h2vie`, pure Python) has no C ABI on this path; its
 * operator boundary is Python:
 *   matvec(h2, x)                 /root/reference/pkg/src/h2vie/arith.py:108-117
 *   matmat_apply(h2, X, col_block) arith.py:120-130
 *   bicgstab_solve(apply, rhs, tol, max_iter, seed, shadow)   arith.py:605-689
 * and its only native FFI precedent is
 *   assemble_block_raw(centers, chi, k0, volume, diag, rows, cols, out) -> int
 *                                  /root/reference/pkg/src/h2vie/_kernel_core.pyx:13-47
 * (caller-allocated output, integer status).  This header follows that
 * precedent: plain pointers and sizes, caller-owned I/O, int status
 * (H2B_OK = 0, negative = error, message via h2b_last_error()), no C++
 * exceptions and no torch types across the boundary.  The Python drop-in
 * (`paper_1703_01175_b200`) binds it with ctypes; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Index space: every vector argument named *_perm is in the cluster-permuted
 * order of the reference (`xp = x[tree.perm]`, arith.py:113-114); complex
 * values are interleaved (re, im) doubles (numpy complex128 / cuDoubleComplex).
 * Multi-RHS blocks are (N, q) row-major, i.e. numpy `X[perm]` C-order.
 */
#ifndef H2B_H
#define H2B_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H2B_OK 0
#define H2B_EINVAL (-1)   /* bad argument / shape (reference raises ValueError) */
#define H2B_ECUDA (-2)    /* CUDA runtime error */
#define H2B_ENOMEM (-3)   /* device allocation failed */
#define H2B_ESTATE (-4)   /* handle not fully uploaded */
#define H2B_ENODEV (-5)   /* no sm_100 (B200) device: there is no CPU fallback */

typedef struct h2b_ctx* h2b_handle;

/* Level-packed operator description (host pointers, copied by h2b_create).
 * Mirrors paper_1703_01175_b200/pack.py::PackedH2; each table restates one
 * reference structure:
 *   clusters   clustering.py:24-45 (start/stop/level/child_lo/child_hi/parent)
 *   ranks      build.py:76 (NestedBasis.rank)
 *   couplings  build.py:294-309 (dict (t,s) -> S, sorted admissible order)
 *   near-field build.py:321-324 (dict (t,s) -> D, sorted inadmissible order)
 * P = num_clusters, packed index = level-major ordinal (tree.levels order). */
typedef struct h2b_layout {
  int64_t n;             /* number of unknowns N */
  int32_t depth;         /* tree.depth */
  int32_t num_clusters;  /* P */
  const int32_t* level_ptr;   /* [depth+1] */
  const int32_t* c_start;     /* [P] start in permuted index space */
  const int32_t* c_size;      /* [P] */
  const int32_t* c_rank;      /* [P] k_c (0 allowed) */
  const int32_t* c_child_lo;  /* [P] packed index or -1 */
  const int32_t* c_child_hi;  /* [P] */
  const int32_t* c_parent;    /* [P] packed index or -1 */
  const int64_t* c_xhat_off;  /* [P+1] prefix sum of ranks */
  const int64_t* c_v_off;     /* [P] element offset of V_c in vbuf (-1: non-leaf) */
  const int64_t* c_t_off;     /* [P] element offset of (T_lo,T_hi) in tbuf (-1: leaf) */
  int64_t n_coupling;
  const int64_t* s_row_ptr;   /* [P+1] CSR over packed target */
  const int32_t* s_col;       /* [n_coupling] packed source */
  const int64_t* s_off;       /* [n_coupling] element offset in sbuf */
  int64_t n_near;
  const int64_t* d_row_ptr;   /* [P+1] */
  const int32_t* d_col;       /* [n_near] packed source leaf */
  const int64_t* d_off;       /* [n_near] element offset in dbuf */
  const int64_t* perm;        /* [N] tree.perm */
  int64_t v_elems, t_elems, s_elems, d_elems;  /* payload sizes (complex elements) */
} h2b_layout;

/* payload sections for h2b_upload */
#define H2B_SEC_V 0  /* leaf bases     */
#define H2B_SEC_T 1  /* transfers      */
#define H2B_SEC_S 2  /* couplings      */
#define H2B_SEC_D 3  /* near-field     */

/* Library/ABI version and the device it will run on. */
int h2b_version(void);
const char* h2b_last_error(void);
/* 1 if a device with compute capability 10.x is visible, 0 otherwise. */
int h2b_device_ok(int device);

/* Create a handle and copy the index tables to `device`.  Replaces the
 * construction of the reference H2Matrix object as the matvec's input
 * (build.py:135-145). */
int h2b_create(const h2b_layout* layout, int device, h2b_handle* out);
/* Copy `bytes` of payload (host or device memory) into section `sec` at byte offset
 * `offset` (chunked uploads allowed).  All four sections must be covered before use. */
int h2b_upload(h2b_handle h, int sec, const void* src, size_t bytes, size_t offset);
int h2b_destroy(h2b_handle h);
/* Fill the near-field section on the device from the voxel geometry instead of uploading it
 * (SURVEY.md §8f row f3): restates the reference block sampler assemble_block_raw
 * (_kernel_core.pyx:13-47) for every inadmissible pair.  centers: N x 3 doubles, chi: N
 * complex (interleaved), both HOST arrays in the ORIGINAL point order; diag = k0^2 *
 * self_term(volume, k0) (kernel.py:170-187).  H2B_EINVAL on coincident centres. */
int h2b_assemble_near(h2b_handle h, const double* centers, const double* chi, double k0,
                      double volume, double diag_re, double diag_im);
/* Device bytes held by the handle (payloads + tables + workspace). */
int64_t h2b_device_bytes(h2b_handle h);

/* y_perm = S x_perm for q right-hand sides, DEVICE pointers, (N, q) row-major.
 * Replaces arith._apply_perm (arith.py:52-104).  Stream-ordered on `stream`
 * (a cudaStream_t; NULL = legacy default).  No allocation after the first
 * call with a given q.  x_perm and y_perm must not alias.  y_perm is overwritten
 * (it need not be initialised: at q = 1 on small operators the two persistent
 * kernels of the step zero it themselves, rows by rows, before they accumulate
 * into it; elsewhere a memset node does).  Environment switches for A/B runs:
 * H2B_Y_MEMSET=1 (memset node), H2B_TREE_NO_FLAT=1 (top programs instead of the
 * flattened top tier), H2B_NEAR_NG=1 (one near-field consumer group),
 * H2B_NEAR_GRID=n (near-field CTAs), H2B_NO_TREE=1 (task-graph far field). */
int h2b_matvec_perm(h2b_handle h, const void* x_perm, void* y_perm, int q, void* stream);

/* y = S x with HOST buffers in the ORIGINAL ordering, (N, q) row-major:
 * the drop-in for arith.matvec / arith.matmat_apply (arith.py:108-130).
 * Synchronous; one CUDA graph per call: pinned buffers are read and written
 * over PCIe by the permutation kernels themselves (zero copy), pageable ones
 * (numpy) are staged through the handle's pinned buffers by host threads. */
int h2b_matvec_host(h2b_handle h, const void* x, void* y, int q);

/* Profiling split of h2b_matvec_perm: phase 0 = near-field only (y overwritten,
 * arith.py:100-104), phase 1 = far field only (y accumulated, arith.py:58-99). */
int h2b_matvec_phase(h2b_handle h, int phase, const void* x_perm, void* y_perm, int q,
                     void* stream);

/* Run the one-time device preparation (transposes, panel index, schedule)
 * now instead of at the first matvec. */
int h2b_prepare_handle(h2b_handle h);

#define H2B_OPT_GRAPHS 1      /* 1 (default): replay each matvec as a CUDA graph */
#define H2B_OPT_MEGA 2        /* 1 (default): single persistent launch per q=1 matvec
                                 (set before the first matvec) */
#define H2B_OPT_TRACE 3       /* 1: record a per-task timeline of the persistent kernel */
#define H2B_OPT_DEBUG 4       /* profiling only, results are WRONG: bit 0 skips far-field task
                                 bodies, bit 1 near-field task bodies of the persistent kernel */
#define H2B_OPT_TREE 6        /* 1 (default): the q=1 far field of a complete binary tree runs as
                                 subtree programs (one CTA per subtree, payload staged once);
                                 0: the task-graph kernel.  Set before the first matvec. */
#define H2B_OPT_MRHS 5        /* 1 (default): q >= 2 runs every phase as a grouped complex GEMM on
                                 the FP64 tensor pipe (DMMA); 0: per-phase CUDA-core kernels */
int h2b_set_option(h2b_handle h, int option, int value);

/* Per-task timeline of the last persistent-kernel matvec (tracing on): for task i,
 * out[10i..10i+9] = {type (0 near, 1 span, 2 coupling), arg, t_claim, t_ready,
 * t_staged, t_level0, t_level1, t_computed (spans only; else 0), t_done
 * (ns, %globaltimer), smid | cta << 32}. */
int h2b_get_trace(h2b_handle h, int64_t* out, int64_t max_tasks);
/* development aid: per-program timeline of the q=1 tree far field (env H2B_TREE_TRACE at prepare):
   out[32 i + j] = globaltimer stamp j of program i (SM clock64 at out[32 i + 16 + j]) (start, staged, external x̂ ready, x̂ published,
   coupling inputs ready, before / after the parent wait, down pass done, end). */
int h2b_tree_trace(h2b_handle h, int64_t* out, int64_t max_progs);
/* Development aid: per-CTA timeline of the last near-field launch (H2B_NEAR_TRACE set before
 * the first matvec): out[24 c + j], globaltimer ns: 0 entry, 1 first record in, 2 last block
 * issued, 3 first block landed, 4 last block consumed, 5 producer exit; 6 blocks, 7 SM id;
 * SM cycles: producer waits 8 stage free, 9 record landed, 10 record buffer free, 11 index
 * load; consumer (thread 0) waits 12 block landed, 13 record landed; 14 consumer total;
 * 16 block math to stage release, 17 leaf ends. */
int h2b_near_trace(h2b_handle h, int64_t* out, int64_t max_ctas);

#define H2B_Q_LAUNCHES_Q1 1   /* kernels per single-RHS matvec */
#define H2B_Q_SPAN_MODE 2     /* 1 if the q=1 far field uses staged subtree spans */
#define H2B_Q_SPLIT_LEVEL 3   /* tree level at which spans are rooted */
#define H2B_Q_TOP_STAGED 4    /* 1 if levels above the split run as one staged CTA */
#define H2B_Q_DEVICE_BYTES 5
#define H2B_Q_MEGA 6          /* 1 if q=1 matvecs run as one persistent kernel */
#define H2B_Q_MEGA_TASKS 7    /* tasks in its graph */
#define H2B_Q_MEGA_GRID 8     /* CTAs it launches */
#define H2B_Q_MEGA_TIERS 9    /* tiers of span programs */
#define H2B_Q_DEVICE_ERROR 10 /* nonzero if a dependency wait ever timed out (a bug) */
#define H2B_Q_NEAR_TASKS 11   /* near-field tasks of the q=1 stream kernel */
#define H2B_Q_NEAR_STAGES 12  /* TMA ring stages of the near-field stream kernel */
#define H2B_Q_NEAR_SMEM 13    /* dynamic shared memory of the near-field stream kernel (bytes) */
#define H2B_Q_MEGA_SMEM 14    /* dynamic shared memory of the far-field task-graph kernel (bytes) */
#define H2B_Q_NEAR_VARIANT 15 /* 100 * leaf size + rows per thread of the near kernel (0: generic) */
#define H2B_Q_MRHS_LAUNCHES 16 /* kernel launches of one multi-RHS (q >= 2) matvec */
#define H2B_Q_TREE 17         /* q=1 far field as subtree programs: programs | split level << 16 | top level << 24 (0: off) */
int h2b_query(h2b_handle h, int what, int64_t* out);

/* Permutation helpers on device buffers: out[i,:] = in[perm[i],:] (gather,
 * arith.py:113) and out[perm[i],:] = in[i,:] (scatter, arith.py:116). */
int h2b_gather_perm(h2b_handle h, const void* in, void* out, int q, void* stream);
int h2b_scatter_perm(h2b_handle h, const void* in, void* out, int q, void* stream);

/* ---------------------------------------------------------------------
 * Krylov solvers, fully on device (operator = the handle's matvec).
 * Both work in the permuted space (a permutation preserves inner products,
 * so iteration counts are unchanged).  DEVICE pointers, length N.
 * --------------------------------------------------------------------- */
typedef struct h2b_report {
  int32_t iterations;     /* SolveReport.iterations (arith.py:39-44) */
  int32_t converged;      /* SolveReport.converged */
  int32_t n_history;      /* entries written to `history` */
  int32_t matvecs;        /* operator applications performed */
  double wall_time;       /* seconds, host clock around the solve */
} h2b_report;

/* Restarted GMRES(restart), CGS2 Arnoldi, x0 = 0 — restates
 * oracle/krylov_oracle.py::gmres_solve (new: the reference has no GMRES).
 * history: host array of >= max_iter doubles (may be NULL). */
int h2b_gmres(h2b_handle h, const void* b_perm, void* x_perm, int restart, double tol,
              int max_iter, double* history, h2b_report* report, void* stream);

/* Block GMRES(restart) for q <= 64 right-hand sides (BASELINE config 5), all on device: the q-column
 * matvec, block CGS2 (tall-skinny V^H W / W - V C kernels), CholQR2 of every block, the small
 * least-squares problem orthonormalised incrementally in the (restart+1)q-dimensional space (no
 * host work per step: the residual is read from mapped pinned memory one step behind).  B_perm,
 * X_perm: N x q row-major complex128 device arrays in the permuted order.  Converged when every
 * column's true relative residual is <= tol at the end of a cycle (oracle/krylov_oracle.py::
 * block_gmres_solve); history: max over columns of the least-squares residual per block step. */
int h2b_block_gmres(h2b_handle h, const void* B_perm, void* X_perm, int q, int restart, double tol,
                    int max_iter, double* history, h2b_report* report, void* stream);

/* BiCGStab, a line-by-line restatement of arith.bicgstab_solve
 * (arith.py:605-689) incl. the single rho-breakdown restart; the restart's
 * random perturbation (numpy default_rng(seed)) cannot be drawn on device,
 * so the caller passes it pre-drawn in `restart_noise_perm` (N complex,
 * permuted order, already multiplied by ||b|| 1e-8), or NULL to fail on
 * breakdown.  shadow_perm may be NULL (shadow = r0). */
int h2b_bicgstab(h2b_handle h, const void* b_perm, void* x_perm, double tol, int max_iter,
                 const void* shadow_perm, const void* restart_noise_perm,
                 double* history, h2b_report* report, void* stream);

/* ---------------------------------------------------------------------
 * Fused Krylov vector kernels (device pointers, complex128, length n),
 * exposed for solvers driven from the host language.
 * --------------------------------------------------------------------- */
/* out[j] = sum_i conj(V[j*ldv + i]) * w[i], j < nv  (deterministic order) */
int h2b_zdotc_multi(const void* V, int64_t ldv, int nv, const void* w, int64_t n,
                    void* out_dev, void* stream);
/* w[i] -= sum_j V[j*ldv + i] * h[j]; if nrm2_out != NULL also writes ||w||^2 */
int h2b_zgemv_sub(const void* V, int64_t ldv, int nv, const void* h_dev, void* w, int64_t n,
                  double* nrm2_out_dev, void* stream);
/* y = a*x + b*y with complex scalars given by value (re, im) */
int h2b_zaxpby(int64_t n, double ar, double ai, const void* x, double br, double bi, void* y,
               void* stream);
/* Row-distributed GMRES building blocks (paper_1703_01175_b200/dist.py): the device Givens
 * recurrence of h2b_gmres on a caller-owned state of h2b_gmres_state_elems(m) complex128 values
 * (H (m+1) x m | g (m+1) | cosines (m) | residual records (2m) | 1/hn | {||b||, 0}), reading
 * step j's CGS2 coefficients from hvals_dev ([0, j], [64, 64 + j]: the two passes, [128].x:
 * ||w||^2, all already summed over ranks); host_res (mapped pinned, or NULL) receives
 * {res_j, hn_j}.  h2b_zscale_dev: w *= scale_dev[0].x (the normalisation). */
/* Streaming-read calibration: reads `bytes` of device memory through a TMA bulk-copy ring (the
 * near-field kernel's access pattern, no math) — the attainable cold read of that many bytes. */
int h2b_stream_read(const void* src, size_t bytes, void* sink_dev, void* stream);
/* Keeps `stream` busy for `ns` nanoseconds (one thread polling %globaltimer): enqueued before a
 * timed region's start event so that host-side launch latency does not count as device time. */
int h2b_spin_ns(uint64_t ns, void* stream);
/* Development aid: a one-thread kernel on `stream` writes %globaltimer (ns) to dst_dev[0]. */
int h2b_stamp_ns(uint64_t* dst_dev, void* stream);
/* Stage II of the H² builder on the device: nested bases, transfers and
 * couplings from the Stage-I grouped factors (the reference's build_all_cluster_ab output) of a
 * packed block structure.  Results stay on the device until fetched: h2b_builder_ranks (k per
 * cluster), h2b_builder_fetch (0: leaf bases, 1: transfers, 2: couplings, concatenated in packed
 * / CSR order).  Gram matrices up to 80 x 80 (leaf size, k_lo + k_hi). */
int h2b_builder_create(int P, int depth, const int32_t* level_ptr, const int32_t* c_start,
                       const int32_t* c_size, const int32_t* c_child_lo, const int32_t* c_child_hi,
                       const int32_t* c_parent, const int32_t* s1_rank, const int64_t* s1_a_off,
                       const void* s1_a, const int64_t* s1_m_off, const void* s1_m,
                       const int64_t* s1_b_off, const void* s1_b, const int64_t* s1_part_ptr,
                       const int32_t* s1_partner, const int64_t* s1_prow, const int64_t* s_row_ptr,
                       const int32_t* s_col, double eps_acc, int device, void** builder);
int h2b_builder_ranks(void* builder, int32_t* ranks);
int h2b_builder_fetch(void* builder, int what, const int32_t* c_child_lo, void* dst);
int h2b_builder_destroy(void* builder);
/* Stage I on the device: partially pivoted ACA of every cluster's grouped admissible block row
 * (the reference's aca_factorize, entries sampled from the voxel geometry), one CTA per cluster;
 * outputs the factor offsets and partner lists, h2b_stage1_fetch copies A / B / B^T conj(B). */
int h2b_stage1_run(int P, const int32_t* c_start, const int32_t* c_size, const int64_t* perm, int64_t n,
                   const int64_t* s_row_ptr, const int32_t* s_col, const double* centers, const void* chi,
                   double k0, double volume, double eps_aca, int max_rank, int device, int32_t* rank_out,
                   int64_t* a_off, int64_t* b_off, int64_t* m_off, int64_t* part_ptr, int32_t* partner,
                   int64_t* prow, void** stage1);
int h2b_stage1_fetch(void* stage1, void* a, void* b, void* m);
int h2b_stage1_destroy(void* stage1);
/* device pointers of the Stage-I factors A / B / B^T conj(B) (input of h2b_builder_create, which
 * accepts host or device pointers). */
int h2b_stage1_device_ptrs(void* stage1, void** a, void** b, void** m);
/* out[i] = Σ_j S[rows[i], j] x[j]: exact rows of the system matrix (entries from the geometry, self
 * term diag = k0^2 self_term), summed directly over all N columns (original point order; host
 * arrays) — the reference for device-built operators the reference builder cannot produce. */
int h2b_exact_rows(const int64_t* rows, int nrows, int64_t n, const double* centers, const void* chi, double k0,
                   double volume, double diag_re, double diag_im, const void* x, void* out, int device);
int64_t h2b_gmres_state_elems(int m);
int h2b_gmres_givens(void* state, int m, int j, const void* hvals_dev, double* host_res, void* stream);
int h2b_zscale_dev(void* w, int64_t n, const void* scale_dev, void* stream);

/* ---------------------------------------------------------------------
 * Plan handles: a set of device payloads plus per-phase lists of grouped
 * complex GEMM (q >= 2, FP64 tensor pipe) / GEMV (q = 1) work items, built by
 * the host.  The subtree-partitioned multi-GPU matvec (SURVEY.md §8e,
 * paper_1703_01175_b200/shard.py) runs one per rank: phase UP_OWN before the
 * all-gather of x and x̂, the others after it.  Every vector is (rows, q)
 * row-major complex128 on the device.
 *   item: C[c_row + i, :] (+)= sum over its segments of A_seg[i, :] B_seg[:, :], i < m <= 64
 *   seg:  A = payload[a_src][a_off + i*lda + j] (i < m, j < k <= 32),
 *         B row j = (b_src buffer)[b_row + j]
 * flags: seg  = a_src | b_src << 4 (b_src 0 x, 1 xhat, 2 yhat) | 256 (A transposed:
 *               A[i][j] = payload[a_off + j*lda + i]) | 512 (B rows gathered: row j =
 *               gather[b_row + j], table set by h2b_plan_set_gather)
 *        item = dst (0 x, 1 xhat, 2 yhat, 3 y) | 256 (accumulate) | 512 (broadcast to peers)
 * --------------------------------------------------------------------- */
typedef struct h2b_mm_item {
  int64_t c_row;
  int32_t m, seg0, nseg, flags;
  int64_t pad;
} h2b_mm_item;
typedef struct h2b_mm_seg {
  int64_t a_off, b_row;
  int32_t k, lda, flags, pad;
} h2b_mm_seg;
typedef struct h2b_plan_ctx* h2b_plan_handle;

int h2b_plan_create(int device, int n_payloads, const int64_t* payload_elems, h2b_plan_handle* out);
int h2b_plan_upload(h2b_plan_handle p, int payload, const void* src, size_t bytes, size_t offset);
/* launch_items[i] = items of the i-th launch (launches run in order; items of one launch must
 * write disjoint rows) */
int h2b_plan_set_phase(h2b_plan_handle p, int phase, int n_launches, const int64_t* launch_items,
                       const h2b_mm_item* items, int64_t n_items, const h2b_mm_seg* segs,
                       int64_t n_segs);
int h2b_plan_run(h2b_plan_handle p, int phase, const void* x, const void* xhat, void* yhat, void* y,
                 int q, void* stream);
/* q = 1 near-field of a plan on the streaming near-field kernel: items {int64 y_row; int32
 * b_first, nb; int32 row0, pad} (rows_per_thread * 128 / (ns/2) rows of a ns-point leaf each),
 * blocks {int64 d_off (in payload 4), int64 x_row}.  When set, h2b_plan_run(phase 4, q = 1)
 * overwrites y with the near-field and then runs phase 5 (the leaf back-transform items);
 * h2b_plan_run(H2B_PLAN_PHASE_NEAR_FAST, q = 1) runs the near-field alone (it reads only x, so
 * it may run on a second stream beside phases 1-3, with phase 5 after both). */
#define H2B_PLAN_PHASE_NEAR_FAST 6
int h2b_plan_set_near_fast(h2b_plan_handle p, const void* items, int64_t n_items, const void* blks,
                           int64_t n_blks, int ns, int rows_per_thread);
/* q = 1 coupling of a plan on the panel kernels: payload 3 holds, per target, the stacked Sᵀ
 * panel (Σ k_s) x k_t; items {int64 panel, xcol, out; int32 R, w} (out = x̂/ŷ row of the
 * target), xcol = the gathered x̂ row of every panel row.  When set, h2b_plan_run(phase 2, q = 1)
 * runs them instead of the phase's items. */
int h2b_plan_set_couple_fast(h2b_plan_handle p, const void* items, int64_t n_items, const int32_t* xcol,
                             int64_t n_xcol);
/* Row-index table of gathered segments (set before h2b_plan_set_phase validates them). */
int h2b_plan_set_gather(h2b_plan_handle p, const int32_t* idx, int64_t n);
int h2b_plan_destroy(h2b_plan_handle p);
/* Fused exchange over peer memory (NVLink P2P stores): items flagged 512 (broadcast) store
 * their rows into the local buffer AND into every peer's buffer at the same rows (the all-gather
 * of x̂ fused into the kernel that produces it); h2b_plan_bcast_rows pushes this rank's x rows
 * [row0, row0 + nrows) of `buf` the same way.  Peers are the other ranks' exchange buffers,
 * mapped with h2b_ipc_open (or any device pointers this device can store to).  The caller
 * orders the peers' next phase after these stores (e.g. a barrier collective). */
int h2b_plan_set_peers(h2b_plan_handle p, void* const* peer_bufs, int npeers);
int h2b_plan_bcast_rows(h2b_plan_handle p, const void* buf, int64_t row0, int64_t nrows, int q,
                        void* stream);
/* Element offset added to every peer pointer by subsequent runs / broadcasts (alternating
 * exchange buffers inside one allocation). */
int h2b_plan_set_peer_offset(h2b_plan_handle p, int64_t elems);
/* Plain device allocations (exchange buffers to be shared with CUDA IPC), zero-filled. */
int h2b_device_alloc(int device, size_t bytes, void** out);
int h2b_device_free(void* ptr);
/* Structure-exact operators (benchmarks): seeded synthetic payload values from a counter-based
 * generator value(seed, section, global index) — identical wherever a block is materialised.
 * Raw: dev_ptr[e] = value(section, global_off + e).  Plan: descriptors {plan_off, global_off,
 * rows, cols, transposed, section} (n x 6 int64, host), each writing a rows x cols global block
 * as-is or transposed at plan_off of `payload`. */
int h2b_fill_synthetic_raw(void* dev_ptr, int64_t n, int64_t global_off, int section, uint64_t seed,
                           double scale);
int h2b_plan_fill_synthetic(h2b_plan_handle p, int payload, const int64_t* desc, int64_t n_desc,
                            uint64_t seed, double scale);
/* Near-field blocks of a plan sampled on the device: descriptors {plan_off, t_start, nt,
 * s_start, ns} (permuted index space, host), perm / centers / chi as in h2b_assemble_near. */
int h2b_plan_fill_near(h2b_plan_handle p, int payload, const int64_t* desc, int64_t n_desc,
                       const int64_t* perm, int64_t n, const double* centers, const double* chi,
                       double k0, double volume, double diag_re, double diag_im);
/* CUDA IPC of a device buffer between the ranks' processes (64-byte handle). */
int h2b_ipc_get_handle(const void* dev_ptr, void* handle_out);
int h2b_ipc_open(const void* handle, void** dev_ptr_out);
int h2b_ipc_close(void* dev_ptr);
int64_t h2b_plan_device_bytes(h2b_plan_handle p);

#ifdef __cplusplus
}
#endif
#endif /* H2B_H */
