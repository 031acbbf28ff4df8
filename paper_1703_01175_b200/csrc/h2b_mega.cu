// Persistent single-RHS H² matvec for sm_100a: two concurrent persistent kernels.
//
// `_apply_perm` (reference arith.py:52-104) splits into two independent halves whose
// results are both added into y (zeroed first: by a memset node, or — tree far field — by the
// far-field programs themselves, ZeroSync in h2b_common.cuh):
//   * k_near_stream  the near field y += D x (arith.py:100-104), bandwidth-bound: one CTA
//                    per SM (plus one per SM without a far-field program) streams D row
//                    panels through a TMA ring; tasks (row panels of a few leaves) are split
//                    statically over the CTAs (or claimed from an atomic counter); for
//                    32-point leaves two consumer groups take the stream's leaves in turn.
//   * k_mega         the far field (arith.py:58-99), latency-bound: a task graph planned on
//                    the host (h2b_plan.cu) of T_SPAN forward/backward span programs
//                    (subtrees or upper tiers of the cluster tree, staged with TMA bulk
//                    copies) and T_COUPLE groups of coupling panels ŷ_t = Σ Sᵀ-panel x̂.
//                    One CTA per SM runs a static, topologically sorted task list from its
//                    own bulk-loaded "blob"; tasks wait on epoch-stamped completion flags.
// Both kernels run at the same time (one CTA of each per SM: the planner splits the shared
// memory); with the memset node neither waits on the other (without it the near-field CTAs wait
// for the far-field programs' zeroing flags before their consumers start).  Each y element
// receives exactly one near and at most one far contribution, so the sum is deterministic
// (two-term floating-point addition commutes).  For complete binary trees the far field is
// k_far_tree (h2b_tree.cu) in k_mega's place.
#include "h2b_span.cuh"

namespace {

constexpr int MNT = 256;  // threads per CTA
constexpr int NST_MAX = 8;

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
// no memory clobber: a sweep's loads may all be in flight before the first compare (the
// sweep ends with __all_sync and, once complete, an acquire fence)
__device__ __forceinline__ uint32_t ld_relaxed_nc(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
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
__device__ __forceinline__ void atomic_add2(double2* p, double2 v) {
  atomicAdd(&p->x, v.x);
  atomicAdd(&p->y, v.y);
}

// ===========================================================================
// near field: k_near_stream
// ===========================================================================
struct NearArgs {
  const int4* recs;   // near task records (see Task in h2b_common.cuh)
  const int2* idx;    // per task {first slot, slots}
  int n_tasks;
  MegaCtrl* ctrl;
  const double2* dbuf;
  const double2* x;
  double2* y;
  // generic leaves (record {leaf index})
  const int32_t *leaves, *c_start, *c_size, *d_col;
  const int64_t *d_row_ptr, *d_off;
  int nst;        // ring stages
  int rec_slots;  // slots of each of the two record buffers
  uint32_t delay_ns;  // tuning aid: the producer starts this late (0 = at once)
  int static_split;   // 1: CTA c streams tasks [c T / G, (c+1) T / G) in order (no claims)
  int dbg;            // profiling only (results wrong): 1 no consumer math, 2 no x copies
  uint64_t* trace;    // optional (H2B_NEAR_TRACE): 8 stamps per CTA, see h2b_near_trace
  // static split: each CTA's first record {slot, slots} and first block {D, x} offsets, so the
  // kernel's first two copies need no index or record load (one memory round trip to the first
  // block instead of three: at kernel start the far kernel's staging burst makes each ~2 us)
  int early;
  // no memset of y before the step (r02): with the static split every row of y is updated by
  // exactly one CTA; the far-field programs zero y (ZeroSync in h2b_common.cuh)
  ZeroSync* zeroed;  // nullptr: y is zeroed by the caller
  int2 first_rec[NEAR_MAXG];
  int2 zero_n[NEAR_MAXG];  // .x: flags CTA c waits for (programs covering its rows)
  longlong2 first_blk[NEAR_MAXG];
};

// One CTA streams a sequence of near-field tasks as ONE continuous sequence of D blocks:
// thread 0 (producer) keeps the nst-stage TMA ring full, walking ahead through the blocks of
// the tasks whose records sit in NRB record buffers; all threads (consumers) process the
// blocks in the same order.  A record buffer is refilled with a newly claimed task as soon as
// its task is consumed, so the stream never drains at task boundaries however small the
// tasks are.
constexpr int NRB = NEAR_NRB;  // record buffers: the consumer's task and up to NRB - 1 claimed ahead

__device__ __forceinline__ void bulk_g2s_hint_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int NS, int R>
__device__ __forceinline__ void issue_block(const NearArgs& A, const int64_t* bl, int i, double2* st,
                                            uint64_t* bar, uint64_t pol) {
  // one stage = the task's D slice of block i + the partner's x segment behind it
  constexpr int RB = R * (MNT / (NS / 2));
  mbar_arrive_expect_tx(bar, 16u * (RB * NS + NS));
  bulk_g2s_hint(st, A.dbuf + bl[2 * i], 16u * RB * NS, bar, pol);
  bulk_g2s(st + RB * NS, A.x + bl[2 * i + 1], 16u * NS, bar);
}

// near field of one leaf with arbitrary block shapes (warp per row); record: {leaf index}
__device__ __forceinline__ void near_task_generic(const NearArgs& A, int leaf_idx) {
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
    if (lane == 0) atomic_add2(A.y + t0 + i, acc);
  }
}

// Warp-specialised: warps 0-7 consume D blocks (256 threads, as near_task_generic and the
// block layout assume), warp 8 is the producer.  Its lane 0 claims tasks from the global
// counter (one atomic per task), bulk-loads their records and keeps the nst-stage ring full;
// the claim and record latencies stay off the consumers' path as long as the ring holds work.
//   fbar[s] full  (producer arrive + TMA bytes)  ebar[s] empty (one arrive per consumer warp)
//   rbar[b] record loaded (or end-of-stream mark)  rfree[b] record consumed (per consumer warp)
constexpr int NEAR_THREADS = MNT + 32;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}


// at most 80 registers: its 9 warps sit beside the far kernel's 8 (<= 128 registers) within each
// scheduler's 16K-register share (warp i runs on scheduler i % 4: scheduler 0 holds 3 near
// warps).  Over budget, most near CTAs wait for the far kernel to exit (measured: step 82 us)
// TR: the per-CTA timeline (H2B_NEAR_TRACE) and the profiling switches (A.dbg) are compiled into
// a second instantiation only: the stamps' predicated clock reads sat on the consumer's per-block
// chain (~5 % of its stall samples; near field alone 30.7 -> 28.7 us without them)
// NG: consumer groups.  NG = 2 (r02): warps 0-3 and 4-7 take the leaves of the stream in turn
// (a leaf's blocks all go to one group, so every row of y still gets one update); the per-block
// chain of a group is a little longer (each thread two rows), but two blocks are worked on at
// once — the stream of a CTA is bound by that chain, not by the ring or by HBM.
template <int NS, int R, bool TR = false, int NG = 1>
__global__ void __maxnreg__(80) k_near_stream(NearArgs A) {
  // dynamic shared memory: [ring: nst stages][NRB record buffers]
  extern __shared__ __align__(16) double2 sm[];
  __shared__ uint64_t fbar[NG * NST_MAX], ebar[NST_MAX], rbar[NRB], rfree[NRB];  // fbar: per consumer group and stage
  __shared__ int s_task[NRB];
  constexpr int LPR = NS > 0 ? NS / 2 : 1;
  constexpr int RPP = MNT / LPR;
  constexpr int RB = R * RPP;                       // rows of a task's slice of each block
  constexpr int STG = NS > 0 ? RB * NS + NS : 0;    // stage: D slice + x segment (double2)
  const int nst = NS > 0 ? A.nst : 0;
  int4* rbuf0 = reinterpret_cast<int4*>(sm + (size_t)nst * STG);
  auto rbuf = [&](int b) { return rbuf0 + (size_t)b * A.rec_slots; };
  uint64_t* tr = TR && A.trace ? A.trace + 24 * blockIdx.x : nullptr;
  uint64_t cw[4] = {0, 0, 0, 0};  // trace: wait cycles (see h2b_near_trace)
  if (threadIdx.x == 0) {
    if (tr) {
      tr[0] = gtimer();
      tr[7] = smid();
    }
    for (int i = 0; i < NST_MAX; ++i) {
      for (int g = 0; g < NG; ++g) mbar_init(&fbar[g * NST_MAX + i], 1);
      mbar_init(&ebar[i], MNT / 32 / NG);  // the warps of the group that consumes the stage's block
    }
    for (int b = 0; b < NRB; ++b) {
      mbar_init(&rbar[b], 1);
      mbar_init(&rfree[b], MNT / 32);
    }
  }
  __syncthreads();
  // shared-window addresses of the barriers and the ring, computed once (see mbar_wait_a)
  const uint32_t fbar_a = smem_u32(fbar), ebar_a = smem_u32(ebar), sm_a = smem_u32(sm);
  // y is zeroed by the far-field programs at their start (ZeroSync, h2b_common.cuh): the
  // consumers wait here — while the producer fills the ring and before the first block can have
  // landed — for the flags of the programs covering the CTA's rows, and clear them.  (Nothing of
  // this inside the consumer loop: it is latency-bound, every instruction there costs rate.)
  if (A.zeroed && threadIdx.x < MNT) {
    if (threadIdx.x < A.zero_n[blockIdx.x].x) {
      uint32_t* f = &A.zeroed->flag[blockIdx.x][threadIdx.x];
      for (long spins = 0;; ++spins) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v == 1u) break;
        if (spins > (1l << 22)) {
          atomicExch(&A.ctrl->error, 4u);
          break;
        }
        __nanosleep(100);
      }
      *(volatile uint32_t*)f = 0u;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(MNT) : "memory");
  }
  if (threadIdx.x >= MNT) {
    // ---------------- producer (one lane) ----------------
    if (threadIdx.x == MNT) {
      const uint64_t pol = policy_evict_first();
      if (A.delay_ns) {
        const uint64_t t0 = gtimer();
        while (gtimer() - t0 < A.delay_ns) __nanosleep(256);
      }
      int claimed = 0;  // records 0 .. claimed-1 claimed
      bool end = false;
      // static split: the index entries of this CTA's first NRB tasks, loaded together (one
      // round trip, not NRB sequential ones before the ring fills); the first from the params
      const int s_first = (int)((int64_t)blockIdx.x * A.n_tasks / gridDim.x);
      const int s_end = (int)((int64_t)(blockIdx.x + 1) * A.n_tasks / gridDim.x);
      const bool pre_ok = A.static_split != 0;
      int2 pre[NRB];
      if (pre_ok) {
#pragma unroll
        for (int i = 0; i < NRB; ++i)
          pre[i] = (i == 0 && A.early) ? A.first_rec[blockIdx.x]
                   : s_first + i < s_end ? __ldg(A.idx + s_first + i) : make_int2(0, 0);
      }
      // claim record `claimed` into buffer claimed % NRB, given the counter value c (fetched
      // early: the atomic's round trip overlaps the block issues of the record before)
      auto finish_claim = [&](int c) {
        const int b = claimed % NRB;
        uint64_t c0 = tr ? clock64() : 0;
        if (claimed >= NRB) mbar_wait(&rfree[b], ((claimed / NRB) - 1) & 1u);  // consumers done with it
        if (tr) cw[2] += clock64() - c0;
        if (end) c = A.n_tasks;
        s_task[b] = c;
        if (c < A.n_tasks) {
          if (tr) c0 = clock64();
          const int2 ix = claimed < NRB && pre_ok ? pre[claimed] : A.idx[c];
          mbar_arrive_expect_tx(&rbar[b], 16u * ix.y);
          if (tr) cw[3] += clock64() - c0;
          bulk_g2s(rbuf(b), A.recs + ix.x, 16u * ix.y, &rbar[b]);
        } else {
          end = true;
          mbar_arrive(&rbar[b]);  // end of stream (s_task published by the arrive's release)
        }
        ++claimed;
      };
      // claims: the next task from the global counter (dynamic balance), or this CTA's next task
      // of a static contiguous split (no atomics on the producer's path)
      int s_next = s_first;
      auto claim = [&]() -> int {
        if (A.static_split) {
          const int c = s_next < s_end ? s_next : A.n_tasks;
          ++s_next;
          return c;
        }
        return (int)atomicAdd(&A.ctrl->near_next, 1u);
      };
      const int dbg = TR ? A.dbg : 0;  // (profiling switches: instrumented instantiation only)
      int issued = 0;
      int pturn = 0;     // NG = 2: consumer group of the leaf being issued
      int pst = 0;       // ring stage of the next block (no divisions on the issue path)
      uint32_t pph = 0;  // its phase parity
      const bool early = A.early && s_first < s_end && NS > 0;
      if (early) {  // the first block before any record (its offsets are kernel parameters)
        const longlong2 fb = A.first_blk[blockIdx.x];
        // (NG > 1: the consumers read the partner's x segment from global memory themselves — it is
        // L2-resident — one block ahead; the second bulk request per block cost a 2 us timer tick)
        constexpr bool XC = NG == 1;
        mbar_arrive_expect_tx(&fbar[0], 16u * (RB * NS + ((dbg & 2) || !XC ? 0 : NS)));
        bulk_g2s_hint(sm, A.dbuf + fb.x, 16u * RB * NS, &fbar[0], pol);
        if (!(dbg & 2) && XC) bulk_g2s(sm + RB * NS, A.x + fb.y, 16u * NS, &fbar[0]);
        issued = 1;
        pst = nst == 1 ? 0 : 1;
        pph = nst == 1 ? 1u : 0u;
      }
      for (int i = 0; i < NRB - 1; ++i) finish_claim(claim());
      for (int q = 0;; ++q) {
        // keep NRB - 1 records claimed beyond q: fetch the counter now, complete the claim after
        // this record's blocks are issued
        const bool want = claimed < q + NRB && !end;
        const int pending = want ? claim() : 0;
        const int b = q % NRB;
        uint64_t c1 = tr ? clock64() : 0;
        mbar_wait(&rbar[b], (q / NRB) & 1u);
        if (tr) cw[1] += clock64() - c1;
        if (tr && q == 0) tr[1] = gtimer();
        if (s_task[b] >= A.n_tasks) {
          if (want) finish_claim(pending);  // (an unused claim past the end is harmless)
          break;
        }
        if constexpr (NS > 0) {
          const int4* r = rbuf(b);
          const int nb = r[0].x;
          const int64_t* bl = reinterpret_cast<const int64_t*>(r + 1 + r[0].y);
          // NG = 2: a block completes on the full barrier of the group that consumes its leaf
          // (the leaves of the stream go to the groups in turn), so every group sees every phase
          // of the barriers it waits on — a parity wait tells only adjacent phases apart
          const int64_t* plv = reinterpret_cast<const int64_t*>(r + 1);  // {y_off, blocks} per leaf
          int pl = 0, prem = NG > 1 ? (int)plv[1] : 0;
          if (NG > 1 && q > 0) pturn = (pturn + 1) & (NG - 1);
          for (int j = 0; j < nb; ++j) {
            if constexpr (NG > 1) {
              while (prem == 0) {
                ++pl;
                prem = (int)plv[2 * pl + 1];
                pturn = (pturn + 1) & (NG - 1);
              }
              --prem;
            }
            if (j == 0 && q == 0 && early) continue;  // issued above (the first leaf: group 0)
            ++issued;
            uint64_t c2 = tr ? clock64() : 0;
            if (issued > nst) mbar_wait_a(ebar_a + 8u * pst, pph ^ 1u);  // freed by round (issued - 1) / nst - 1
            if (tr) cw[0] += clock64() - c2;
            const uint32_t sp = sm_a + 16u * (uint32_t)(pst * STG),
                           fb_a = fbar_a + 8u * (uint32_t)((NG > 1 ? pturn * NST_MAX : 0) + pst);
            constexpr bool XC = NG == 1;
            mbar_arrive_expect_tx_a(fb_a, 16u * (RB * NS + ((dbg & 2) || !XC ? 0 : NS)));
            bulk_g2s_hint_a(sp, A.dbuf + bl[2 * j], 16u * RB * NS, fb_a, pol);
            if (!(dbg & 2) && XC) bulk_g2s_a(sp + 16u * RB * NS, A.x + bl[2 * j + 1], 16u * NS, fb_a);
            if (++pst == nst) {
              pst = 0;
              pph ^= 1u;
            }
          }
        }
        if (want) finish_claim(pending);
      }
      if (tr) tr[2] = gtimer();
      // every claimed record has been consumed or marked as the end; wait for the consumers to
      // release the last buffers so no bulk copy is in flight at exit
      for (int q = (claimed > NRB ? claimed - NRB : 0); q < claimed; ++q)
        if (s_task[q % NRB] < A.n_tasks) mbar_wait(&rfree[q % NRB], (q / NRB) & 1u);
      if (tr) {
        tr[5] = gtimer();
        for (int i = 0; i < 4; ++i) tr[8 + i] = cw[i];
      }
      if (atomicAdd(&A.ctrl->near_exited, 1u) == gridDim.x - 1) {
        A.ctrl->near_exited = 0;  // last CTA out resets the claim counter for the next launch
        A.ctrl->near_next = 0;
      }
    }
    return;
  }
  // ---------------- consumers: warps 0-7 ----------------
  const int lane = threadIdx.x & 31;
  if constexpr (NS == 0) {
    // ragged leaves: one leaf per task, plain loads (record: {leaf index})
    for (int q = 0;; ++q) {
      const int b = q % NRB;
      mbar_wait(&rbar[b], (q / NRB) & 1u);
      if (s_task[b] >= A.n_tasks) break;
      near_task_generic(A, rbuf(b)[0].x);
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfree[b]);
    }
  } else if constexpr (NG >= 2) {
    constexpr int GT = MNT / NG;                      // threads of a group
    constexpr int EPT = RB * NS / GT;                 // slice elements per thread
    constexpr int CPL = EPT < 4 ? EPT : 4;
    constexpr int LPRC = NS / CPL;
    constexpr int RPPC = GT / LPRC;
    constexpr int RR = EPT / CPL;
    static_assert(RR * RPPC == RB && CPL * LPRC == NS, "near consumer mapping (two groups)");
    const int grp = threadIdx.x / GT, gt = threadIdx.x % GT;
    const int r0 = gt / LPRC, c0 = gt % LPRC;
    int st = 0;         // ring stage of the stream's next block (both groups count all blocks)
    uint32_t phs = 0;   // bit s: parity of this group's next phase of its full barrier of stage s
    const uint32_t gbar_a = fbar_a + 8u * (uint32_t)(grp * NST_MAX);
    int turn = 0;       // group of the stream's next leaf
    int consumed = 0;
    for (int q = 0;; ++q) {
      const int b = q % NRB;
      mbar_wait(&rbar[b], (q / NRB) & 1u);
      if (s_task[b] >= A.n_tasks) break;
      const int4* rec = rbuf(b);
      const int nl = rec[0].y, row0 = rec[0].z;
      const int64_t* lv = reinterpret_cast<const int64_t*>(rec + 1);  // {y_off, nb} per leaf
      const int64_t* blx = lv + 2 * nl + 1;  // block list {D offset, x offset}: the x offsets
      int bofs = 0;                          // first block of the leaf in the record's list
      for (int li = 0; li < nl; ++li) {
        const int nbl = (int)lv[2 * li + 1];
        const bool mine = turn == grp;
        turn = (turn + 1) & (NG - 1);
        if (!mine) {  // the other group's leaf (its blocks complete on that group's barriers)
          st += nbl;
          while (st >= nst) st -= nst;
          bofs += nbl;
          continue;
        }
        constexpr int NACC = CPL < 2 ? 1 : 2;
        double2 acc[RR][NACC];
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int j = 0; j < NACC; ++j) acc[r][j] = make_double2(0.0, 0.0);
        for (int i = 0; i < nbl; ++i, ++consumed) {
          // the partner's x segment straight from global memory (L2), requested before the wait
          // for the block so that its latency hides behind it
          double2 xv[CPL];
          {
            const double2* xs = A.x + blx[2 * (bofs + i)] + c0;
#pragma unroll
            for (int j = 0; j < CPL; ++j) xv[j] = __ldg(xs + j * LPRC);
          }
          mbar_wait_a(gbar_a + 8u * st, (phs >> st) & 1u);
          phs ^= 1u << st;
          if (TR && tr && consumed == 0 && gt == 0 && grp == 0) tr[3] = gtimer();
          const double2* sp = sm + (size_t)st * STG;
#pragma unroll
          for (int r = 0; r < RR; ++r) {
            double2 dv[CPL];
#pragma unroll
            for (int j = 0; j < CPL; ++j) dv[j] = sp[(r0 + r * RPPC) * NS + c0 + j * LPRC];
#pragma unroll
            for (int j = 0; j < CPL; ++j) cfma(acc[r][j % NACC], dv[j], xv[j]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_a(ebar_a + 8u * st);  // this warp is done with the stage
          if (++st == nst) st = 0;
        }
        const int64_t y_off = lv[2 * li];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          double2 a = acc[r][0];
#pragma unroll
          for (int j = 1; j < NACC; ++j) a = cadd(a, acc[r][j]);
#pragma unroll
          for (int m = LPRC / 2; m > 0; m >>= 1) a = cadd(a, shfl_xor2(a, m));
          if (c0 == 0) atomic_add2(A.y + y_off + row0 + r0 + r * RPPC, a);
        }
        bofs += nbl;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfree[b]);  // this warp is done with the record
    }
    if (TR && tr && threadIdx.x == 0) {
      tr[4] = gtimer();
      tr[6] = consumed;
    }
  } else {
    // consumer mapping: each thread owns CPL interleaved columns (c0 + j LPRC: conflict-free
    // 16-byte loads) of RR rows of the block slice; a leaf's row sums then need log2(LPRC)
    // shuffle levels (3 for 32-wide leaves)
    constexpr int EPT = NS > 0 ? RB * NS / MNT : 1;  // slice elements per thread
    constexpr int CPL = EPT < 4 ? EPT : 4;
    constexpr int LPRC = NS > 0 ? NS / CPL : 1;
    constexpr int RPPC = MNT / LPRC;
    constexpr int RR = EPT / CPL;
    static_assert(NS == 0 || (RR * RPPC == RB && CPL * LPRC == NS), "near consumer mapping");
    const int r0 = threadIdx.x / LPRC;
    const int c0 = threadIdx.x % LPRC;
    int consumed = 0;
    int st = 0;       // ring stage of the next block and its phase parity: the per-block path
    uint32_t ph = 0;  // has no divisions (it is latency-bound: 2 consumer warps per scheduler)
    const bool math = TR ? !(A.dbg & 1) : true;
    const uint64_t cstart = tr ? clock64() : 0;
    for (int q = 0;; ++q) {
      const int b = q % NRB;
      uint64_t c4 = tr ? clock64() : 0;
      mbar_wait(&rbar[b], (q / NRB) & 1u);
      if (tr) cw[1] += clock64() - c4;
      if (s_task[b] >= A.n_tasks) break;
      const int4* rec = rbuf(b);
      const int nb = rec[0].x, nl = rec[0].y, row0 = rec[0].z;
      const int64_t* lv = reinterpret_cast<const int64_t*>(rec + 1);  // {y_off, nb} per leaf
      int li = 0;
      int leaf_end = (int)lv[1];
      constexpr int NACC = CPL < 2 ? 1 : 2;  // accumulators per row (even / odd columns)
      double2 acc[RR][NACC];
#pragma unroll
      for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int j = 0; j < NACC; ++j) acc[r][j] = make_double2(0.0, 0.0);
      for (int i = 0; i < nb; ++i, ++consumed) {
        uint64_t c3 = tr ? clock64() : 0;
        mbar_wait_a(fbar_a + 8u * st, ph);
        if (tr) cw[0] += clock64() - c3;
        if (tr && consumed == 0 && threadIdx.x == 0) tr[3] = gtimer();
        const double2* sp = sm + (size_t)st * STG;
        const uint64_t c5 = tr ? clock64() : 0;
        if (math) {
          double2 xv[CPL];  // a row's loads before its FMAs
#pragma unroll
          for (int j = 0; j < CPL; ++j) xv[j] = sp[RB * NS + c0 + j * LPRC];
#pragma unroll
          for (int r = 0; r < RR; ++r) {
            double2 dv[CPL];
#pragma unroll
            for (int j = 0; j < CPL; ++j) dv[j] = sp[(r0 + r * RPPC) * NS + c0 + j * LPRC];
#pragma unroll
            for (int j = 0; j < CPL; ++j) cfma(acc[r][j % NACC], dv[j], xv[j]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(ebar_a + 8u * st);  // this warp is done with the stage
        if (++st == nst) {
          st = 0;
          ph ^= 1u;
        }
        const uint64_t c6 = tr ? clock64() : 0;
        if (tr) cw[2] += c6 - c5;
        if (i + 1 == leaf_end) {  // last partner of this leaf: reduce and add its rows
          const int64_t y_off = lv[2 * li];
#pragma unroll
          for (int r = 0; r < RR; ++r) {
            double2 a = acc[r][0];
#pragma unroll
            for (int j = 1; j < NACC; ++j) a = cadd(a, acc[r][j]);
#pragma unroll
            for (int m = LPRC / 2; m > 0; m >>= 1) a = cadd(a, shfl_xor2(a, m));
            if (c0 == 0) atomic_add2(A.y + y_off + row0 + r0 + r * RPPC, a);
#pragma unroll
            for (int j = 0; j < NACC; ++j) acc[r][j] = make_double2(0.0, 0.0);
          }
          if (++li < nl) leaf_end += (int)lv[2 * li + 1];
        }
        if (tr) cw[3] += clock64() - c6;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfree[b]);  // this warp is done with the record
    }
    if (tr && threadIdx.x == 0) {
      tr[4] = gtimer();
      tr[6] = consumed;
      tr[12] = cw[0];
      tr[13] = cw[1];
      tr[14] = clock64() - cstart;
      tr[16] = cw[2];
      tr[17] = cw[3];
    }
  }
}

// ===========================================================================
// far field: k_mega
// ===========================================================================
struct MegaArgs {
  const int4* recs;
  const int4* prefetch;
  int n_prefetch;
  MegaCtrl* ctrl;
  uint32_t* flags;
  int n_tasks;
  // spans
  SpanBases B;
  // coupling
  const double2* sbuf;
  const int32_t* xcol;
  double2* xhat;
  double2* yhat;
  // flattened bottom tier
  const double2* wbuf;
  const double2* x;
  double2* y;
  const double2* ydeep;
  uint64_t* trace;  // optional: per task {claim, ready, staged, done, smid} (globaltimer ns)
  int smem_elems;   // dynamic shared memory (double2) of the work area
  int debug;        // profiling aid (H2B_OPT_DEBUG)
  const int2* cta_lists;  // per CTA: {blob offset, blob length} in 16-byte slots
};

// ---------------------------------------------------------------------------
// coupling of a group of consecutive targets (record: group header + items).
// The panels are one contiguous range of sbuf (one TMA bulk copy) and the
// gathered x̂ rows one contiguous range of s_xcol; all threads gather x̂ into
// shared memory meanwhile.  A single big panel (cta_mode) streams from HBM.
// ---------------------------------------------------------------------------
// static part (before the dependencies are met): the panels' bulk copy
// The gather indices are static too: each thread loads the (up to XPRE) indices it will
// gather into registers here, so that after the wait only the x̂ loads remain.
constexpr int XPRE = 2;
__device__ __forceinline__ void couple_stage_static(const MegaArgs& A, const int4* rec, double2* sm,
                                                    uint64_t* bar, int (&xi)[XPRE]) {
  const int n_items = rec[0].x, cta_mode = rec[0].y;
  const CoupleItem* items = reinterpret_cast<const CoupleItem*>(rec + 1);
  const CoupleItem first = items[0], last = items[n_items - 1];
  const int64_t p0 = first.panel;
  const int64_t pe = cta_mode ? 0 : (last.panel + (int64_t)last.R * last.w - p0);
  if (pe > 0 && threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, 16u * (uint32_t)pe);
    bulk_g2s(sm, A.sbuf + p0, 16u * (uint32_t)pe, bar);
  }
  const int64_t x0 = first.xcol, xe = last.xcol + last.R - x0;
#pragma unroll
  for (int j = 0; j < XPRE; ++j) {
    const int64_t e = threadIdx.x + (int64_t)j * MNT;
    xi[j] = e < xe ? __ldg(A.xcol + x0 + e) : 0;
  }
}

__device__ __forceinline__ void couple_task(const MegaArgs& A, const int4* rec, double2* red,
                                            double2* sm, uint64_t* bar, uint32_t& phase, const int (&xi)[XPRE]) {
  const int n_items = rec[0].x, cta_mode = rec[0].y;
  const CoupleItem* items = reinterpret_cast<const CoupleItem*>(rec + 1);
  const CoupleItem first = items[0], last = items[n_items - 1];
  const int64_t p0 = first.panel, x0 = first.xcol;
  const int64_t pe = cta_mode ? 0 : (last.panel + (int64_t)last.R * last.w - p0);
  const int64_t xe = last.xcol + last.R - x0;
  double2* sx = sm + pe;  // gathered x̂ after the staged panels
#pragma unroll
  for (int j = 0; j < XPRE; ++j) {
    const int64_t e = threadIdx.x + (int64_t)j * MNT;
    if (e < xe) sx[e] = __ldcg(A.xhat + xi[j]);
  }
  for (int64_t e = threadIdx.x + (int64_t)XPRE * MNT; e < xe; e += MNT) sx[e] = __ldcg(A.xhat + A.xcol[x0 + e]);
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

// ---------------------------------------------------------------------------
// flattened bottom tier (FlatRec): W_c staged with x_c (up) or alone (down) before the
// dependencies are met
// ---------------------------------------------------------------------------
__device__ __forceinline__ void flat_stage_static(const MegaArgs& A, const FlatRec& f, bool up, double2* sm,
                                                  uint64_t* bar) {
  if (threadIdx.x == 0) {
    const uint32_t wb = 16u * (uint32_t)f.n * f.k;
    mbar_arrive_expect_tx(bar, wb + (up ? 16u * f.n : 0u));
    bulk_g2s(sm, A.wbuf + f.w_off, wb, bar);
    if (up) bulk_g2s(sm + (size_t)f.n * f.k, A.x + f.x_off, 16u * f.n, bar);
  }
}

// x̂_c = W_cᵀ x_c (whole CTA, column-major accumulation as in the span ops)
__device__ __forceinline__ void flat_up(const MegaArgs& A, const FlatRec& f, double2* sm, uint64_t* bar,
                                        double2* red) {
  mbar_wait(bar, 0);
  const double2* xs = sm + (size_t)f.n * f.k;
  cta_panel_q<MNT>(sm, f.n, f.k, [=] __device__(int64_t r, int) { return xs[r]; }, A.xhat + f.hat_off, false, 1,
                   red);
}

// y_c += W_c ŷ_c + y_deep_c, one thread per point, one atomic add per element
__device__ __forceinline__ void flat_down(const MegaArgs& A, const FlatRec& f, double2* sm, uint64_t* bar,
                                          double2* red) {
  if (threadIdx.x < f.k) red[threadIdx.x] = __ldcg(A.yhat + f.hat_off + threadIdx.x);
  mbar_wait(bar, 0);
  __syncthreads();
  for (int r = threadIdx.x; r < f.n; r += MNT) {
    double2 a0 = __ldcg(A.ydeep + f.x_off + r), a1 = make_double2(0.0, 0.0);
    const double2* w = sm + (size_t)r * f.k;
    int c = 0;
    for (; c + 1 < f.k; c += 2) {
      cfma(a0, w[c], red[c]);
      cfma(a1, w[c + 1], red[c + 1]);
    }
    if (c < f.k) cfma(a0, w[c], red[c]);
    const double2 v = cadd(a0, a1);
    atomicAdd(&A.y[f.x_off + r].x, v.x);
    atomicAdd(&A.y[f.x_off + r].y, v.y);
  }
}

__global__ void __launch_bounds__(MNT, 2) k_mega(MegaArgs A) {
  // dynamic shared memory: [work area: span working set / coupling panels][this CTA's blob:
  // its task list, dependency ranges and task records, one bulk copy]
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double2 red[MNT];
  __shared__ uint32_t s_epoch;
  __shared__ __align__(128) uint64_t bar, bbar;
  uint32_t phase = 0;
  int4* blob = reinterpret_cast<int4*>(sm + A.smem_elems);
  const int2 lst = A.cta_lists[blockIdx.x];  // {blob offset, blob length} in 16-byte slots
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bbar, 1);
    s_epoch = *(volatile uint32_t*)&A.ctrl->epoch;
    if (lst.y > 0) {
      mbar_arrive_expect_tx(&bbar, 16u * lst.y);
      bulk_g2s(blob, A.recs + lst.x, 16u * lst.y, &bbar);
    }
  }
  // optional (H2B_OPT_DEBUG bit 6, measured slower on B200): warm the far-field operands into L2,
  // every CTA's TMA unit taking an equal strided share
  if (threadIdx.x == 0 && (A.debug & 64))
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
  // forever).
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
    // profiling aid (H2B_OPT_DEBUG bit 0): task bodies skipped, dependency skeleton only
    const bool skip = A.debug & 1;
    // Every task starts from a freshly initialised transaction barrier (parity 0).  Carrying one
    // barrier's parity across a CTA's mixed span / coupling tasks was measured to lose phase
    // sync under load (1-3% of launches read a staging area before its bulk copies had
    // landed); the previous task ended with a CTA barrier, so no thread still waits on the old
    // phase and none of its copies is in flight.
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      mbar_init(&bar, 1);
    }
    phase = 0;
    // static operands stream in while the dependencies are still outstanding
    const FlatRec& fr = *reinterpret_cast<const FlatRec*>(rec);
    int xi[XPRE] = {};
    if (!skip && type == T_SPAN)
      span_stage_static<MNT>(hd, cps, A.B, sm, &bar);
    else if (!skip && type == T_COUPLE)
      couple_stage_static(A, rec, sm, &bar, xi);
    else if (!skip)
      flat_stage_static(A, fr, type == T_FLAT_UP, sm, &bar);
    // dependencies: warp 0 polls (lanes share the flags) with a short backoff; the other warps
    // wait at the barrier.  Each sweep issues relaxed loads of every outstanding flag back to
    // back (one L2 round trip per sweep however many ranges there are: acquire loads would
    // serialise, one round trip per flag), and one acquire fence follows the last sweep.
    if (threadIdx.x < 32 && n_dep) {
      // lane L takes the flattened dependencies L, L+32, ... (up to four in registers; longer
      // lists sweep the ranges)
      const int lane = threadIdx.x;
      int f0 = -1, f1 = -1, f2 = -1, f3 = -1, cnt = 0, base = 0;
      for (int i = 0; i < n_dep; ++i) {
        const int2 rg = deps[i];
        for (int d = rg.x + ((lane - base) & 31); d < rg.y; d += 32, ++cnt) {
          if (cnt == 0) f0 = d;
          else if (cnt == 1) f1 = d;
          else if (cnt == 2) f2 = d;
          else if (cnt == 3) f3 = d;
        }
        base += rg.y - rg.x;
      }
      const bool small = __all_sync(0xffffffffu, cnt <= 4);
      long spins = 0;
      for (;;) {
        bool ok = true;
        if (small) {
          const uint32_t v0 = f0 >= 0 ? ld_relaxed_nc(A.flags + f0) : done;
          const uint32_t v1 = f1 >= 0 ? ld_relaxed_nc(A.flags + f1) : done;
          const uint32_t v2 = f2 >= 0 ? ld_relaxed_nc(A.flags + f2) : done;
          const uint32_t v3 = f3 >= 0 ? ld_relaxed_nc(A.flags + f3) : done;
          ok = v0 == done && v1 == done && v2 == done && v3 == done;
        } else {
          for (int i = 0; i < n_dep; ++i) {
            const int2 rg = deps[i];
            for (int d = rg.x + lane; d < rg.y; d += 32) ok &= ld_relaxed_nc(A.flags + d) == done;
          }
        }
        if (__all_sync(0xffffffffu, ok)) break;
        if (++spins > (1l << 24)) {  // never expected: report instead of hanging the GPU
          atomicExch(&A.ctrl->error, 1u);
          break;
        }
        __nanosleep(32);
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    // order the acquires (made visible to every thread by the barrier) before the async-proxy
    // (TMA) reads of the produced data: the fence follows the barrier in the issuing thread
    if (n_dep) asm volatile("fence.proxy.async.global;" ::: "memory");
    if (A.trace && threadIdx.x == 0) A.trace[8 * t + 1] = gtimer();
    if (skip) {
      // profiling aid only (H2B_OPT_DEBUG): this task's body is skipped
    } else if (type == T_SPAN) {
      span_finish<MNT>(hd, cps, A.B, sm, &bar, phase, A.trace ? A.trace + 8 * t + 2 : nullptr, 3);
    } else if (type == T_COUPLE) {
      couple_task(A, rec, red, sm, &bar, phase, xi);
    } else if (type == T_FLAT_UP) {
      flat_up(A, fr, sm, &bar, red);
    } else {
      flat_down(A, fr, sm, &bar, red);
    }
    // this task's generic shared-memory writes precede the next task's TMA writes into the
    // same work area (the consumers of x̂ / ŷ order their TMA reads after their acquire)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 32) {  // publish completion (thread 32: warp 0 may still be polling)
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

}  // namespace

int h2b_mega_static_smem() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_mega) != cudaSuccess) {
    cudaGetLastError();
    return 8192;
  }
  return (int)fa.sharedSizeBytes;
}

int h2b_mega_regs() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_mega) != cudaSuccess) {
    cudaGetLastError();
    return 255;
  }
  return fa.numRegs;
}

int h2b_mega_occupancy(int, int, int smem_bytes, int* blocks_per_sm) {
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_mega, MNT, smem_bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    h2b_set_error(std::string("occupancy: ") + cudaGetErrorString(e));
    return H2B_ECUDA;
  }
  return H2B_OK;
}

// Both persistent kernels ask for the largest shared-memory carveout: with a smaller one
// chosen for whichever starts first, the other would not fit beside it on the SM.
int h2b_mega_set_smem(int, int, int bytes) {
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_mega, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  H2B_CUDA_TRY(cudaFuncSetAttribute(k_mega, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  return H2B_OK;
}

#define NEAR_VARIANTS(X) X(32, 1) X(32, 2) X(64, 1) X(64, 2) X(64, 4) X(64, 8)

int h2b_near_stream_static_smem(int ns, int r, int* bytes) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaErrorInvalidValue;
  // (the instantiation with the most static shared memory and registers: two consumer groups, instrumented)
#define X(a, b) \
  if (ns == a && r == b) e = cudaFuncGetAttributes(&fa, k_near_stream<a, b, true, (a == 32 ? 2 : 1)>);
  NEAR_VARIANTS(X)
#undef X
  if (ns != 32 && ns != 64) e = cudaFuncGetAttributes(&fa, k_near_stream<0, 1>);
  if (e != cudaSuccess) {
    cudaGetLastError();
    h2b_set_error(std::string("near stream attributes: ") + cudaGetErrorString(e));
    return H2B_ECUDA;
  }
  *bytes = (int)fa.sharedSizeBytes;
  return H2B_OK;
}

int h2b_near_stream_regs(int ns, int r) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaErrorInvalidValue;
#define X(a, b) \
  if (ns == a && r == b) e = cudaFuncGetAttributes(&fa, k_near_stream<a, b, false, (a == 32 ? 2 : 1)>);
  NEAR_VARIANTS(X)
#undef X
  if (ns != 32 && ns != 64) e = cudaFuncGetAttributes(&fa, k_near_stream<0, 1>);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 255;
  }
  return fa.numRegs;
}

int h2b_near_stream_set_smem(int ns, int r, int bytes) {
#define X(a, b)                                                                                           \
  if (ns == a && r == b) {                                                                                \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, false, (a == 32 ? 2 : 1)>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, false, (a == 32 ? 2 : 1)>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, true, (a == 32 ? 2 : 1)>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<a, b, true, (a == 32 ? 2 : 1)>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)); \
  }
  NEAR_VARIANTS(X)
#undef X
  if (ns != 32 && ns != 64) {
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<0, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<0, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_near_stream<0, 1, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  return H2B_OK;
}

int h2b_launch_tree(h2b_ctx* h, const TreeDev* d, const double2* xp, double2* yp, cudaStream_t st, int near_ctas);
ZeroSync* h2b_tree_zero_sync(h2b_ctx* h, TreeDev* d);

// y = 0; then k_near_stream on st and k_mega (or the tree programs) on h->far_stream,
// concurrently (fork / join)
int h2b_launch_mega(h2b_ctx* h, const double2* xp, double2* yp, cudaStream_t st) {
  const bool run_far = h->mega_grid > 0 && !(h->mega_debug & 2);
  const bool run_near = h->n_near_tasks > 0 && !(h->mega_debug & 4);
  // No memset node (r02): when every row of y belongs to exactly one near CTA (static split) and
  // one bottom program, the programs zero their rows at their start (ZeroSync, h2b_common.cuh).
  const bool nozero_off = getenv("H2B_Y_MEMSET") != nullptr;  // A/B aid and tests (read per capture)
  ZeroSync* zeroed = run_far && run_near && h->tree && h->near_zero_ok && !nozero_off ? h2b_tree_zero_sync(h, h->tree) : nullptr;
  if (!zeroed && !(h->mega_debug & 8)) H2B_CUDA_TRY(cudaMemsetAsync(yp, 0, sizeof(double2) * h->n, st));
  if (run_far && h->tree) {  // subtree programs (h2b_tree.cu) in k_mega's place
    H2B_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
    H2B_CUDA_TRY(cudaStreamWaitEvent(h->far_stream, h->ev_fork, 0));
    H2B_TRY(h2b_launch_tree(h, h->tree, xp, yp, h->far_stream, zeroed ? h->near_grid : 0));
  } else if (run_far) {
    H2B_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
    H2B_CUDA_TRY(cudaStreamWaitEvent(h->far_stream, h->ev_fork, 0));
    MegaArgs A;
    A.recs = h->rec_pool;
    A.prefetch = h->l2_prefetch;
    A.n_prefetch = h->n_prefetch;
    A.ctrl = h->ctrl;
    A.flags = h->flags;
    A.n_tasks = h->n_tasks;
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
    A.B.ydeep = h->ydeep;
    A.wbuf = h->wbuf;
    A.x = xp;
    A.y = yp;
    A.ydeep = h->ydeep;
    A.sbuf = h->buf[H2B_SEC_S];
    A.xcol = h->s_xcol;
    A.xhat = h->xhat;
    A.yhat = h->yhat;
    A.trace = h->trace;
    A.smem_elems = h->mega_smem / 16;
    A.debug = h->mega_debug;
    A.cta_lists = h->cta_lists;
    // cooperative launch: all CTAs co-resident (they wait on one another)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->mega_grid);
    cfg.blockDim = dim3(MNT);
    cfg.dynamicSmemBytes = h->mega_smem + 16 * h->mega_blob_slots;
    cfg.stream = h->far_stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    H2B_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_mega, A));
  }
  if (run_near) {
    NearArgs N;
    N.recs = h->near_recs;
    N.idx = h->near_idx;
    N.n_tasks = h->n_near_tasks;
    N.ctrl = h->ctrl;
    N.dbuf = h->buf[H2B_SEC_D];
    N.x = xp;
    N.y = yp;
    N.leaves = h->leaves;
    N.c_start = h->c_start_d;
    N.c_size = h->c_size_d;
    N.d_col = h->d_col_d;
    N.d_row_ptr = h->d_row_ptr_d;
    N.d_off = h->d_off_d;
    N.nst = std::max(1, h->near_nst);
    N.rec_slots = std::max(1, h->near_rec_max);  // NRB buffers of this size follow the ring
    N.delay_ns = h->near_delay_ns;
    N.static_split = h->near_static;
    N.dbg = h->near_dbg;
    N.trace = h->near_trace;
    N.early = h->near_static && h->near_early && h->near_grid <= NEAR_MAXG;
    N.zeroed = zeroed;
    if (zeroed)
      for (int c = 0; c < h->near_grid; ++c) {
        const int2 zr = h->near_zero_row[c];
        const int rpp = std::max(1, h->tree_rows_per_prog);
        N.zero_n[c] = int2{zr.y > 0 ? (zr.x + zr.y - 1) / rpp - zr.x / rpp + 1 : 0, 0};
      }
    if (N.early)
      for (int c = 0; c < h->near_grid; ++c) {
        N.first_rec[c] = h->near_first_rec[c];
        N.first_blk[c] = h->near_first_blk[c];
      }
    const int ns = h->mega_ns, r = h->mega_r;
    bool launched = false;
    // two consumer groups for 32-point leaves (cfg2: near alone 28.8 -> 27.0 us, its last CTA out
    // 30.8 -> 27.9 us in the step); H2B_NEAR_NG=1: one group (A/B aid)
    static const bool ng2 = getenv("H2B_NEAR_NG") ? atoi(getenv("H2B_NEAR_NG")) == 2 : true;  // (four groups: no gain)
#define X(a, b)                                                                            \
  if (!launched && ns == a && r == b) {                                                    \
    if (a == 32 && ng2 && (N.trace || N.dbg))                                              \
      k_near_stream<a, b, true, (a == 32 ? 2 : 1)><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N);  \
    else if (a == 32 && ng2)                                                               \
      k_near_stream<a, b, false, (a == 32 ? 2 : 1)><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N); \
    else if (N.trace || N.dbg)                                                             \
      k_near_stream<a, b, true><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N);               \
    else                                                                                   \
      k_near_stream<a, b><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N);                     \
    launched = true;                                                                       \
  }
    NEAR_VARIANTS(X)
#undef X
    if (!launched) {
      if (N.trace || N.dbg)
        k_near_stream<0, 1, true><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N);
      else
        k_near_stream<0, 1><<<h->near_grid, NEAR_THREADS, h->near_smem, st>>>(N);
    }
    H2B_CHECK_LAUNCH();
  }
  if (run_far) {
    H2B_CUDA_TRY(cudaEventRecord(h->ev_join, h->far_stream));
    H2B_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
  }
  return H2B_OK;
}

// development aid: the per-CTA timeline of the last near-field launch (H2B_NEAR_TRACE set at
// prepare): out[24 * c + j] for CTA c, globaltimer ns: 0 entry, 1 first record in, 2 last block
// issued, 3 first block landed, 4 last block consumed, 5 producer exit; 6 blocks, 7 SM id;
// SM cycles: producer waits 8 stage free, 9 record landed, 10 record buffer free, 11 index
// load; consumer (thread 0) waits 12 block landed, 13 record landed; 14 consumer total; 16 block
// math to stage release, 17 leaf ends
extern "C" int h2b_near_trace(h2b_handle h, int64_t* out, int64_t max_ctas) {
  if (!h || !out || !h->near_trace) {
    h2b_set_error("h2b_near_trace: no near trace (set H2B_NEAR_TRACE before the first matvec)");
    return H2B_ESTATE;
  }
  const int64_t n = std::min<int64_t>(max_ctas, h->near_grid);
  H2B_CUDA_TRY(cudaDeviceSynchronize());
  H2B_CUDA_TRY(cudaMemcpy(out, h->near_trace, sizeof(uint64_t) * 24 * n, cudaMemcpyDeviceToHost));
  return H2B_OK;
}
