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
  int debug;        // profiling aid: task bodies to skip (H2B_OPT_DEBUG)
  const int2* cta_lists;  // per CTA: {first, count} into task_list
  const int* task_list;   // task ids, each CTA's run in global topological order
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
// The ring persists across the CTA's consecutive near tasks: once the current
// task's remaining blocks are all in flight, its refills already stream the
// NEXT task's first blocks (its record was prefetched when it was claimed), so
// the HBM stream of a CTA does not drain between tasks.  `ring` is the stage of
// the current task's block 0; `carry` how many of its blocks the previous task
// issued; returns how many of `next`'s blocks this task issued.
template <int NS, int R>
__device__ __forceinline__ void issue_block(const MegaArgs& A, const int64_t* bl, int i, double2* st,
                                            uint64_t* bar, uint64_t pol) {
  constexpr int RB = R * (MNT / (NS / 2));
  mbar_arrive_expect_tx(bar, 16u * (RB * NS));
  bulk_g2s_hint(st, A.dbuf + bl[2 * i], 16u * RB * NS, bar, pol);
}

template <int NS, int R>
__device__ __forceinline__ int near_task(const MegaArgs& A, const int4* rec, const int4* next,
                                         uint64_t* next_bar, uint32_t next_parity, double2* sm,
                                         uint64_t* fbar, uint32_t& fphase, int nst, uint64_t pol,
                                         uint32_t& ring, int carry) {
  constexpr int LPR = NS / 2;
  constexpr int RPP = MNT / LPR;
  constexpr int RB = R * RPP;        // rows of the task's slice of each block
  constexpr int STG = RB * NS + NS;  // stage: D slice + x segment (double2)
  const int nb = rec[0].x, nl = rec[0].y, row0 = rec[0].z;
  const int64_t* lv = reinterpret_cast<const int64_t*>(rec + 1);        // {y_off, nb} per leaf
  const int64_t* bl = reinterpret_cast<const int64_t*>(rec + 1 + nl);   // {d_off, x_off} per block
  // the next task's record is read by thread 0 only, when it first needs it
  int nb_next = -1;
  const int64_t* bl_next = nullptr;
  auto next_ready = [&]() {
    if (nb_next < 0) {
      if (next) {
        if (next_bar) mbar_wait(next_bar, next_parity);
        nb_next = next[0].x;
        bl_next = reinterpret_cast<const int64_t*>(next + 1 + next[0].y);
      } else {
        nb_next = 0;
      }
    }
    return nb_next;
  };
  const int r0 = threadIdx.x / LPR;
  const int col = (threadIdx.x % LPR) * 2;
  int carry_out = 0;
  if (threadIdx.x == 0) {
    // blocks [0, carry) are in flight already; fill the ring up to nst blocks
    for (int i = carry; i < min(nst, nb); ++i) {
      const int s = (ring + i) % nst;
      issue_block<NS, R>(A, bl, i, sm + (size_t)s * STG, &fbar[s], pol);
    }
    for (int q = 0; nb + q < nst && q < next_ready(); ++q) {  // a short task: start the next one too
      const int s = (ring + nb + q) % nst;
      issue_block<NS, R>(A, bl_next, q, sm + (size_t)s * STG, &fbar[s], pol);
      carry_out = q + 1;
    }
  }
  int li = 0;
  int leaf_end = (int)lv[1];
  double2 acc[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = make_double2(0.0, 0.0);
  for (int i = 0; i < nb; ++i) {
    const int s = (ring + i) % nst;
    // the partner's x segment (L1/L2-resident input) is loaded while the stage is in flight
    const cd2 xv = ld_cached256(A.x + bl[2 * i + 1] + col);
    mbar_wait(&fbar[s], (fphase >> s) & 1u);
    fphase ^= 1u << s;
    const double2* st = sm + (size_t)s * STG;
    const double2 xa = xv.a, xb = xv.b;
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
    __syncthreads();  // stage s fully read: refill it (this task's block i + nst, or the next task's)
    if (threadIdx.x == 0) {
      const int j = i + nst;
      if (j < nb) {
        issue_block<NS, R>(A, bl, j, sm + (size_t)s * STG, &fbar[s], pol);
      } else if (j - nb >= carry_out && j - nb < next_ready()) {
        issue_block<NS, R>(A, bl_next, j - nb, sm + (size_t)s * STG, &fbar[s], pol);
        carry_out = j - nb + 1;
      }
    }
  }
  ring = (ring + nb) % nst;
  return carry_out;  // meaningful in thread 0, the only thread that issues copies
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
  // dynamic shared memory: [work area: near ring / span working set / coupling panels][this
  // CTA's blob: its task list, dependency ranges and task records, one bulk copy]
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double2 red[MNT];
  __shared__ uint32_t s_epoch;
  __shared__ __align__(128) uint64_t bar, bbar;
  __shared__ uint64_t fbar[NST_MAX];
  uint32_t fphase = 0, phase = 0;
  uint32_t ring = 0;  // near-field ring position (persists across the CTA's near tasks)
  int carry = 0;      // blocks of the upcoming near task already in flight
  const int nst = NS > 0 ? max(1, min(NST_MAX, A.smem_elems / (R * (MNT / (NS / 2)) * NS + NS))) : 1;
  const uint64_t pol = policy_evict_first();
  int4* blob = reinterpret_cast<int4*>(sm + A.smem_elems);
  const int2 lst = A.cta_lists[blockIdx.x];  // {blob offset, blob length} in 16-byte slots
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST_MAX; ++i) mbar_init(&fbar[i], 1);
    mbar_init(&bar, 1);
    mbar_init(&bbar, 1);
    s_epoch = *(volatile uint32_t*)&A.ctrl->epoch;
    if (lst.y > 0) {
      mbar_arrive_expect_tx(&bbar, 16u * lst.y);
      bulk_g2s(blob, A.recs + lst.x, 16u * lst.y, &bbar);
    }
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
  if (lst.y > 0) mbar_wait(&bbar, 0);
  const uint32_t done = s_epoch + 1;
  // This CTA's static task list (planned on the host, sorted in the global topological order:
  // the lowest unfinished task is always at the head of some CTA's list, so no CTA can wait
  // forever).  Near-field CTAs own a contiguous run of row panels and never wait.
  const int n_my = lst.y > 0 ? blob[0].x : 0;
  for (int k = 0; k < n_my; ++k) {
    const int4 e0 = blob[1 + 2 * k], e1 = blob[2 + 2 * k];
    const int t = e0.x, type = e0.y;
    const int4* rec = blob + e0.z;
    const int2* deps = reinterpret_cast<const int2*>(blob + e1.x);
    const int n_dep = e1.y;
    if (A.trace && threadIdx.x == 0) {
      A.trace[8 * t] = gtimer();
      A.trace[8 * t + 4] = smid() | ((uint64_t)blockIdx.x << 32);
    }
    const SpanHead* hd = reinterpret_cast<const SpanHead*>(rec);
    const SpanCopy* cps = reinterpret_cast<const SpanCopy*>(rec + (sizeof(SpanHead) + 15) / 16);
    // profiling aid (H2B_OPT_DEBUG): bit 0 skips far-field task bodies, bit 1 near-field ones
    const bool skip = ((A.debug & 1) && type != T_NEAR) || ((A.debug & 2) && type == T_NEAR);
    if (type != T_NEAR) {
      // Every far-field task starts from a freshly initialised transaction barrier (parity 0).
      // Carrying one barrier's parity across a CTA's mixed span / coupling tasks was measured
      // to lose phase sync under load (1-3% of launches read a staging area before its bulk
      // copies had landed); the previous task ended with a CTA barrier, so no thread still
      // waits on the old phase and none of its copies is in flight.
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        mbar_init(&bar, 1);
      }
      phase = 0;
      // static operands stream in while the dependencies are still outstanding
      if (!skip && type == T_SPAN)
        span_stage_static<MNT>(hd, cps, A.B, sm, &bar);
      else if (!skip)
        couple_stage_static(A, rec, sm, &bar);
    }
    // dependencies: warp 0 polls (lanes share the flags) with a backoff, so waiting CTAs do not
    // flood L2 with requests next to the near-field stream; the other warps wait at the barrier
    if (threadIdx.x < 32)
      for (int i = 0; i < n_dep; ++i) {
        const int2 rg = deps[i];
        for (int d = rg.x + threadIdx.x; d < rg.y; d += 32) {
          long spins = 0;
          while (ld_acquire(A.flags + d) != done) {
            if (++spins > (1l << 24)) {  // never expected: report instead of hanging the GPU
              atomicExch(&A.ctrl->error, 1u);
              break;
            }
            __nanosleep(256);
          }
        }
      }
    __syncthreads();
    // order the acquires (made visible to every thread by the barrier) before the async-proxy
    // (TMA) reads of the produced data: the fence follows the barrier in the issuing thread
    if (n_dep) asm volatile("fence.proxy.async.global;" ::: "memory");
    if (A.trace && threadIdx.x == 0) A.trace[8 * t + 1] = gtimer();
    if (skip) {
      // profiling aid only (H2B_OPT_DEBUG): this task's body is skipped
    } else if (type == T_NEAR) {
      if constexpr (NS == 0) {
        near_task_generic(A, rec[0].x);
      } else {
        const bool next_near = k + 1 < n_my && blob[1 + 2 * (k + 1)].y == T_NEAR && !(A.debug & 2);
        carry = near_task<NS, R>(A, rec, next_near ? blob + blob[1 + 2 * (k + 1)].z : nullptr, nullptr, 0,
                                 sm, fbar, fphase, nst, pol, ring, carry);
      }
    } else if (type == T_SPAN) {
      span_finish<MNT>(hd, cps, A.B, sm, &bar, phase, A.trace ? A.trace + 8 * t + 2 : nullptr);
    } else {
      couple_task(A, rec, red, sm, &bar, phase);
    }
    if (type != T_NEAR) {
      // x̂ / ŷ written here with generic stores are read by other CTAs' TMA (async proxy), and
      // this task's generic shared-memory writes precede the next task's TMA writes
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // publish completion from a thread that does not feed the near-field ring (thread 0); a
    // release at GPU scope costs ~0.4 us, so a near-field CTA publishes only its last panel
    // (the planner points every dependency on its panels there)
    if (threadIdx.x == 32 && e1.z) {
      __threadfence();
      st_release(A.flags + t, done);
      if (A.trace) A.trace[8 * t + 3] = gtimer();
    }
  }
  if (threadIdx.x == 0) {
    if (atomicAdd(&A.ctrl->exited, 1u) == gridDim.x - 1) {  // last CTA out advances the epoch
      A.ctrl->exited = 0;
      __threadfence();
      A.ctrl->epoch = s_epoch + 1;
    }
  }
}

template <int NS, int R>
int launch(h2b_ctx* h, const MegaArgs& A, cudaStream_t st) {
  // cooperative launch: all CTAs co-resident (far-field CTAs wait on near-field CTAs)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->mega_grid);
  cfg.blockDim = dim3(MNT);
  cfg.dynamicSmemBytes = h->mega_smem + 16 * h->mega_blob_slots;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  H2B_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_mega<NS, R>, A));
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
  A.debug = h->mega_debug;
  A.cta_lists = h->cta_lists;
  A.task_list = h->task_list;
  const int ns = h->mega_ns, r = h->mega_r;
  if (ns == 32 && r == 1) return launch<32, 1>(h, A, st);
  if (ns == 32 && r == 2) return launch<32, 2>(h, A, st);
  if (ns == 64 && r == 1) return launch<64, 1>(h, A, st);
  if (ns == 64 && r == 2) return launch<64, 2>(h, A, st);
  if (ns == 64 && r == 4) return launch<64, 4>(h, A, st);
  if (ns == 64 && r == 8) return launch<64, 8>(h, A, st);
  return launch<0, 1>(h, A, st);
}
