// Persistent single-launch H² matvec (q = 1) for sm_100a.
//
// One launch executes the whole `_apply_perm` (reference arith.py:52-104) as a
// task graph planned on the host (h2b_plan.cu):
//   * T_SPAN   forward / backward span programs (subtrees or upper tiers of
//              the cluster tree), staged with TMA bulk copies    arith.py:58-71, 82-99
//   * T_COUPLE groups of coupling panels ŷ_t = Σ Sᵀ-panel x̂        arith.py:72-81
//   * T_NEAR   near-field row panels streamed through a TMA ring   arith.py:100-104
// CTAs (2 per SM) claim tasks in queue order from an atomic counter, one task
// AHEAD: while a task runs, the self-contained record of the next one (its
// descriptors: block lists, span copies, coupling items) is already being
// bulk-copied into shared memory, so a task starts issuing its data loads
// without a single dependent global round trip.  A task waits (acquire loads
// on epoch-stamped completion flags) only on tasks with smaller ids; the
// lowest unfinished task is always executing, so the schedule cannot
// deadlock.  Data produced inside the launch is read through L2
// (ld.global.cg / TMA), never through the non-coherent L1.  The near-field
// stream is tagged L2::evict_first and the far-field operands are warmed into
// L2 at launch (cp.async.bulk.prefetch.L2), so the latency-bound tree sweeps
// do not queue behind the bandwidth-bound stream.
#include "h2b_span.cuh"

namespace {

constexpr int MNT = 256;  // threads per CTA
constexpr int NST_MAX = 8;

struct MegaArgs {
  const Task* tasks;
  const DepRange* deps;
  const int4* recs;
  const int4* prefetch;
  int n_prefetch;
  MegaCtrl* ctrl;
  uint32_t* flags;
  int n_tasks;
  const double2* dbuf;
  const double2* x;
  double2* y;
  // generic near (ragged leaves)
  const int32_t *leaves, *c_start, *c_size, *d_col;
  const int64_t *d_row_ptr, *d_off;
  // spans
  const SpanCopy* outs;
  SpanBases B;
  // coupling
  const double2* sbuf;
  const int32_t* xcol;
  double2* xhat;
  double2* yhat;
  uint64_t* trace;  // optional: per task {claim, ready, staged, done, smid} (globaltimer ns)
  int smem_elems;   // dynamic shared memory (double2) of the launch
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// bulk copy with an L2 eviction-priority hint
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// near-field rows of a run of leaves (record in shared memory), TMA ring
// ---------------------------------------------------------------------------
template <int NS, int R>
__device__ __forceinline__ void near_task(const MegaArgs& A, const int4* rec, double2* sm,
                                          uint64_t* fbar, uint32_t& fphase, int nst, uint64_t pol) {
  constexpr int LPR = NS / 2;
  constexpr int RPP = MNT / LPR;
  constexpr int RB = R * RPP;        // rows of the task's slice of each block
  constexpr int STG = RB * NS + NS;  // stage: D slice + x segment (double2)
  const int nb = rec[0].x, nl = rec[0].y, row0 = rec[0].z;
  const int64_t* lv = reinterpret_cast<const int64_t*>(rec + 1);        // {y_off, nb} per leaf
  const int64_t* bl = reinterpret_cast<const int64_t*>(rec + 1 + nl);   // {d_off, x_off} per block
  const int r0 = threadIdx.x / LPR;
  const int col = (threadIdx.x % LPR) * 2;
  const int pre = min(nst, nb);
  if (threadIdx.x == 0)
    for (int i = 0; i < pre; ++i) {
      double2* st = sm + (size_t)i * STG;
      mbar_arrive_expect_tx(&fbar[i], 16u * STG);
      bulk_g2s_hint(st, A.dbuf + bl[2 * i], 16u * RB * NS, &fbar[i], pol);
      bulk_g2s(st + RB * NS, A.x + bl[2 * i + 1], 16u * NS, &fbar[i]);
    }
  int li = 0;
  int leaf_end = (int)lv[1];
  double2 acc[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = make_double2(0.0, 0.0);
  for (int i = 0; i < nb; ++i) {
    const int s = i % nst;
    mbar_wait(&fbar[s], (fphase >> s) & 1u);
    fphase ^= 1u << s;
    const double2* st = sm + (size_t)s * STG;
    const double2 xa = st[RB * NS + col], xb = st[RB * NS + col + 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2* d = st + (r0 + r * RPP) * NS + col;
      cfma(acc[r][0], d[0], xa);
      cfma(acc[r][1], d[1], xb);
    }
    if (i + 1 == leaf_end) {  // last partner of this leaf: reduce and store its rows
      const int64_t y_off = lv[2 * li];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double2 a = cadd(acc[r][0], acc[r][1]);
#pragma unroll
        for (int m = LPR / 2; m > 0; m >>= 1) a = cadd(a, shfl_xor2(a, m));
        if ((threadIdx.x % LPR) == 0) A.y[y_off + row0 + r0 + r * RPP] = a;
        acc[r][0] = acc[r][1] = make_double2(0.0, 0.0);
      }
      if (++li < nl) leaf_end += (int)lv[2 * li + 1];
    }
    __syncthreads();  // stage s fully read: refill it
    if (threadIdx.x == 0 && i + nst < nb) {
      double2* sd = sm + (size_t)s * STG;
      mbar_arrive_expect_tx(&fbar[s], 16u * STG);
      bulk_g2s_hint(sd, A.dbuf + bl[2 * (i + nst)], 16u * RB * NS, &fbar[s], pol);
      bulk_g2s(sd + RB * NS, A.x + bl[2 * (i + nst) + 1], 16u * NS, &fbar[s]);
    }
  }
}

// near-field of one leaf with arbitrary block shapes (warp per row); record: {leaf index}
__device__ __forceinline__ void near_task_generic(const MegaArgs& A, int leaf_idx) {
  const int t = A.leaves[leaf_idx];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = A.c_size[t];
  const int64_t t0 = A.c_start[t];
  const int64_t b0 = A.d_row_ptr[t], b1 = A.d_row_ptr[t + 1];
  for (int i = warp; i < nt; i += MNT / 32) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t b = b0; b < b1; ++b) {
      const int s = A.d_col[b];
      const int ns = A.c_size[s];
      const double2* D = A.dbuf + A.d_off[b] + (int64_t)i * ns;
      const double2* xs = A.x + A.c_start[s];
      for (int j = lane; j < ns; j += 32) cfma(acc, D[j], xs[j]);
    }
    acc = warp_sum2(acc);
    if (lane == 0) A.y[t0 + i] = acc;
  }
}

// ---------------------------------------------------------------------------
// coupling of a group of consecutive targets (record: group header + items).
// The panels are one contiguous range of sbuf (one TMA bulk copy) and the
// gathered x̂ rows one contiguous range of s_xcol; all threads gather x̂ into
// shared memory meanwhile.  A single big panel (cta_mode) streams from HBM.
// ---------------------------------------------------------------------------
// static part (before the dependencies are met): the panels' bulk copy
__device__ __forceinline__ void couple_stage_static(const MegaArgs& A, const int4* rec, double2* sm,
                                                    uint64_t* bar) {
  const int n_items = rec[0].x, cta_mode = rec[0].y;
  const CoupleItem* items = reinterpret_cast<const CoupleItem*>(rec + 1);
  const CoupleItem first = items[0], last = items[n_items - 1];
  const int64_t p0 = first.panel;
  const int64_t pe = cta_mode ? 0 : (last.panel + (int64_t)last.R * last.w - p0);
  if (pe > 0 && threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, 16u * (uint32_t)pe);
    bulk_g2s(sm, A.sbuf + p0, 16u * (uint32_t)pe, bar);
  }
}

__device__ __forceinline__ void couple_task(const MegaArgs& A, const int4* rec, double2* red,
                                            double2* sm, uint64_t* bar, uint32_t& phase) {
  const int n_items = rec[0].x, cta_mode = rec[0].y;
  const CoupleItem* items = reinterpret_cast<const CoupleItem*>(rec + 1);
  const CoupleItem first = items[0], last = items[n_items - 1];
  const int64_t p0 = first.panel, x0 = first.xcol;
  const int64_t pe = cta_mode ? 0 : (last.panel + (int64_t)last.R * last.w - p0);
  const int64_t xe = last.xcol + last.R - x0;
  double2* sx = sm + pe;  // gathered x̂ after the staged panels
  for (int64_t e = threadIdx.x; e < xe; e += MNT) sx[e] = __ldcg(A.xhat + A.xcol[x0 + e]);
  if (pe > 0) {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  __syncthreads();
  if (cta_mode) {
    double2* out = A.yhat + first.out;
    if (first.R == 0) {
      for (int c = threadIdx.x; c < first.w; c += MNT) out[c] = make_double2(0.0, 0.0);
      return;
    }
    cta_panel_q<MNT>(A.sbuf + p0, first.R, first.w, [=] __device__(int64_t r, int) { return sx[r]; }, out,
                     false, 1, red);
    return;
  }
  const int warp = threadIdx.x >> 5;
  for (int i = warp; i < n_items; i += MNT / 32) {
    const CoupleItem it = items[i];
    double2* out = A.yhat + it.out;
    if (it.R == 0) {
      for (int c = threadIdx.x & 31; c < it.w; c += 32) out[c] = make_double2(0.0, 0.0);
      continue;
    }
    const double2* in = sx + (it.xcol - x0);
    panel_op(sm + (it.panel - p0), it.R, it.w, panel_shift(it.w), in, out, 0);
  }
}

template <int NS, int R>
__global__ void __launch_bounds__(MNT, 2) k_mega(MegaArgs A) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double2 red[MNT];
  __shared__ __align__(16) int4 recbuf[2][REC_SLOTS];
  __shared__ uint64_t bar, rbar[2];
  __shared__ uint64_t fbar[NST_MAX];
  __shared__ int s_next;
  __shared__ uint32_t s_epoch;
  uint32_t fphase = 0, phase = 0, rphase = 0;
  const int nst = NS > 0 ? max(1, min(NST_MAX, A.smem_elems / (R * (MNT / (NS / 2)) * NS + NS))) : 1;
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST_MAX; ++i) mbar_init(&fbar[i], 1);
    mbar_init(&bar, 1);
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    s_epoch = *(volatile uint32_t*)&A.ctrl->epoch;
  }
  // warm the far-field operands into L2: every CTA's TMA unit takes an equal strided share
  // (a prefetch occupies the issuing SM's TMA unit, so it must not pile up on a few SMs)
  if (threadIdx.x == 0)
  for (int i = blockIdx.x; i < A.n_prefetch; i += gridDim.x) {
    const int4 r = A.prefetch[i];
    const uint64_t p = (uint64_t)(uint32_t)r.x | ((uint64_t)(uint32_t)r.y << 32);
    prefetch_l2(reinterpret_cast<const void*>(p), (uint32_t)r.z);
  }
  __syncthreads();
  const uint32_t done = s_epoch + 1;
  // claim the first task and start loading its record
  if (threadIdx.x == 0) {
    const int t = (int)atomicAdd(&A.ctrl->next, 1u);
    s_next = t;
    if (t < A.n_tasks) {
      const Task tk = A.tasks[t];
      mbar_arrive_expect_tx(&rbar[0], 16u * tk.rec_len);
      bulk_g2s(recbuf[0], A.recs + tk.rec_off, 16u * tk.rec_len, &rbar[0]);
    }
  }
  __syncthreads();
  int t = s_next, buf = 0;
  while (t < A.n_tasks) {
    __syncthreads();  // everyone has read s_next
    if (A.trace && threadIdx.x == 0) {
      A.trace[8 * t] = gtimer();
      A.trace[8 * t + 4] = smid() | ((uint64_t)blockIdx.x << 32);
    }
    const Task tk = A.tasks[t];
    mbar_wait(&rbar[buf], (rphase >> buf) & 1u);  // this task's record is in shared memory
    rphase ^= 1u << buf;
    const int4* rec = recbuf[buf];
    // static operands stream in while the dependencies are still outstanding
    const SpanHead* hd = reinterpret_cast<const SpanHead*>(rec);
    const SpanCopy* cps = reinterpret_cast<const SpanCopy*>(rec + (sizeof(SpanHead) + 15) / 16);
    if (tk.type == T_SPAN)
      span_stage_static<MNT>(hd, cps, A.B, sm, &bar);
    else if (tk.type == T_COUPLE)
      couple_stage_static(A, rec, sm, &bar);
    // dependencies: every thread checks a share of the flags
    for (int i = tk.dep_first; i < tk.dep_first + tk.n_dep; ++i) {
      const DepRange rg = A.deps[i];
      for (int d = rg.lo + threadIdx.x; d < rg.hi; d += MNT) {
        long spins = 0;
        while (ld_acquire(A.flags + d) != done) {
          if (++spins > (1l << 26)) {  // never expected: report instead of hanging the GPU
            atomicExch(&A.ctrl->error, 1u);
            break;
          }
          __nanosleep(32);
        }
      }
    }
    __syncthreads();  // dependencies met
    // only now claim the next task (a claim must not wait behind a blocked task) and prefetch
    // its record behind this task's execution
    if (threadIdx.x == 0) {
      const int tn = (int)atomicAdd(&A.ctrl->next, 1u);
      s_next = tn;
      if (tn < A.n_tasks) {
        const Task tn_k = A.tasks[tn];
        mbar_arrive_expect_tx(&rbar[buf ^ 1], 16u * tn_k.rec_len);
        bulk_g2s(recbuf[buf ^ 1], A.recs + tn_k.rec_off, 16u * tn_k.rec_len, &rbar[buf ^ 1]);
      }
    }
    // order the acquires before the async-proxy (TMA) reads of the produced data
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (A.trace && threadIdx.x == 0) A.trace[8 * t + 1] = gtimer();
    if (tk.type == T_NEAR) {
      if constexpr (NS == 0)
        near_task_generic(A, rec[0].x);
      else
        near_task<NS, R>(A, rec, sm, fbar, fphase, nst, pol);
    } else if (tk.type == T_SPAN) {
      span_finish<MNT>(hd, cps, A.B, sm, &bar, phase, A.trace ? A.trace + 8 * t + 2 : nullptr);
      phase ^= 1u;
    } else {
      couple_task(A, rec, red, sm, &bar, phase);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(A.flags + t, done);
      if (A.trace) A.trace[8 * t + 3] = gtimer();
    }
    t = s_next;
    buf ^= 1;
  }
  if (threadIdx.x == 0) {
    if (atomicAdd(&A.ctrl->exited, 1u) == gridDim.x - 1) {  // last CTA out resets the queue
      A.ctrl->next = 0;
      A.ctrl->exited = 0;
      __threadfence();
      A.ctrl->epoch = s_epoch + 1;
    }
  }
}

template <int NS, int R>
int launch(h2b_ctx* h, const MegaArgs& A, cudaStream_t st) {
  k_mega<NS, R><<<h->mega_grid, MNT, h->mega_smem, st>>>(A);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

}  // namespace

int h2b_mega_occupancy(int ns, int r, int smem_bytes, int* blocks_per_sm) {
  cudaError_t e;
#define OCC(a, b) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_mega<a, b>, MNT, smem_bytes)
  if (ns == 32 && r == 1) OCC(32, 1);
  else if (ns == 32 && r == 2) OCC(32, 2);
  else if (ns == 64 && r == 1) OCC(64, 1);
  else if (ns == 64 && r == 2) OCC(64, 2);
  else if (ns == 64 && r == 4) OCC(64, 4);
  else if (ns == 64 && r == 8) OCC(64, 8);
  else OCC(0, 1);
#undef OCC
  if (e != cudaSuccess) {
    cudaGetLastError();
    h2b_set_error(std::string("occupancy: ") + cudaGetErrorString(e));
    return H2B_ECUDA;
  }
  return H2B_OK;
}

int h2b_mega_set_smem(int ns, int r, int bytes) {
#define ATTR(a, b) H2B_CUDA_TRY(cudaFuncSetAttribute(k_mega<a, b>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))
  if (ns == 32 && r == 1) ATTR(32, 1);
  else if (ns == 32 && r == 2) ATTR(32, 2);
  else if (ns == 64 && r == 1) ATTR(64, 1);
  else if (ns == 64 && r == 2) ATTR(64, 2);
  else if (ns == 64 && r == 4) ATTR(64, 4);
  else if (ns == 64 && r == 8) ATTR(64, 8);
  else ATTR(0, 1);
#undef ATTR
  return H2B_OK;
}

int h2b_launch_mega(h2b_ctx* h, const double2* xp, double2* yp, cudaStream_t st) {
  MegaArgs A;
  A.tasks = h->tasks;
  A.deps = h->deps;
  A.recs = h->rec_pool;
  A.prefetch = h->l2_prefetch;
  A.n_prefetch = h->n_prefetch;
  A.ctrl = h->ctrl;
  A.flags = h->flags;
  A.n_tasks = h->n_tasks;
  A.dbuf = h->buf[H2B_SEC_D];
  A.x = xp;
  A.y = yp;
  A.leaves = h->leaves;
  A.c_start = h->c_start_d;
  A.c_size = h->c_size_d;
  A.d_col = h->d_col_d;
  A.d_row_ptr = h->d_row_ptr_d;
  A.d_off = h->d_off_d;
  A.outs = h->span_outs;
  A.B.src[SRC_V] = h->buf[H2B_SEC_V];
  A.B.src[SRC_T] = h->buf[H2B_SEC_T];
  A.B.src[SRC_VT] = h->vT;
  A.B.src[SRC_TT] = h->tT;
  A.B.src[SRC_X] = xp;
  A.B.src[SRC_XHAT] = h->xhat;
  A.B.src[SRC_YHAT] = h->yhat;
  A.B.src[SRC_OPS] = reinterpret_cast<const double2*>(h->span_ops);
  A.B.src[SRC_OUTS] = reinterpret_cast<const double2*>(h->span_outs);
  A.B.xhat = h->xhat;
  A.B.yhat = h->yhat;
  A.B.y = yp;
  A.sbuf = h->buf[H2B_SEC_S];
  A.xcol = h->s_xcol;
  A.xhat = h->xhat;
  A.yhat = h->yhat;
  A.trace = h->trace;
  A.smem_elems = h->mega_smem / 16;
  const int ns = h->mega_ns, r = h->mega_r;
  if (ns == 32 && r == 1) return launch<32, 1>(h, A, st);
  if (ns == 32 && r == 2) return launch<32, 2>(h, A, st);
  if (ns == 64 && r == 1) return launch<64, 1>(h, A, st);
  if (ns == 64 && r == 2) return launch<64, 2>(h, A, st);
  if (ns == 64 && r == 4) return launch<64, 4>(h, A, st);
  if (ns == 64 && r == 8) return launch<64, 8>(h, A, st);
  return launch<0, 1>(h, A, st);
}
