// Execution of one span program by one CTA (shared by the stand-alone span
// kernel and the persistent matvec kernel).  See SpanHead in h2b_common.cuh.
#pragma once

#include "h2b_panel.cuh"

struct SpanBases {
  const double2* src[SRC_N];  // V, T, Vᵀ, Tᵀ, x, x̂, ŷ, ops, outs
  double2* xhat;
  double2* yhat;
  double2* y;
  double2* ydeep;  // deep spans of a flattened bottom tier write here (overwrite)
};

// loads that must see data written earlier in the same kernel by other SMs
// bypass L1 (L1 is not coherent): ld.global.cg
__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

// x̂ / ŷ are produced by other tasks of the same launch; everything else is static
__device__ __forceinline__ bool span_src_dynamic(int kind) { return kind == SRC_XHAT || kind == SRC_YHAT; }

// Phase 1 (may run before the span's dependencies are met): arm the barrier for
// the whole working set and stream in the static part (operator payload, op
// list, write-back list, x) with TMA bulk copies, one copy per thread.
template <int NTH>
__device__ __forceinline__ void span_stage_static(const SpanHead* __restrict__ hd,
                                                  const SpanCopy* __restrict__ copies,
                                                  const SpanBases& B, double2* sm, uint64_t* bar) {
  const int n_copy = hd->n_copy, c_first = hd->copy_first;
  if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (uint32_t)hd->pad[0]);  // total staged bytes
  __syncthreads();
  for (int i = threadIdx.x; i < n_copy; i += NTH) {
    const SpanCopy c = copies[c_first + i];
    if (!span_src_dynamic(c.kind)) bulk_g2s(sm + c.smem, B.src[c.kind] + c.src, 16u * (uint32_t)c.elems, bar);
  }
}

// Phase 2 (dependencies met): stream in x̂ / ŷ, wait for everything, walk the
// levels (one __syncthreads per level, warp per cluster), write back.
template <int NTH>
__device__ __forceinline__ void span_finish(const SpanHead* __restrict__ hd, const SpanCopy* __restrict__ copies,
                                            const SpanBases& B, double2* sm, uint64_t* bar, uint32_t phase,
                                            uint64_t* t_staged = nullptr, int y_mode = 2) {
  const int n_copy = hd->n_copy, c_first = hd->copy_first;
  for (int i = threadIdx.x; i < n_copy; i += NTH) {
    const SpanCopy c = copies[c_first + i];
    if (span_src_dynamic(c.kind)) bulk_g2s(sm + c.smem, B.src[c.kind] + c.src, 16u * (uint32_t)c.elems, bar);
  }
  mbar_wait(bar, phase);
  if (t_staged && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    *t_staged = t;
  }
  const SpanOp* ops = reinterpret_cast<const SpanOp*>(sm + hd->ops_smem);
  const int warp = threadIdx.x >> 5;
  constexpr int NW = NTH / 32;
  const int nlev = hd->nlev;
  for (int lv = 0; lv < nlev; ++lv) {
    const int o1 = hd->lvl[lv + 1];
    for (int i = hd->lvl[lv] + warp; i < o1; i += NW) {
      const SpanOp op = ops[i];
      // y: written by the near field before (y_mode 2: accumulate through L2) or concurrently
      // (y_mode 3: atomic add)
      const bool to_y = op.flags & OP_OUT_Y, deep = op.flags & OP_OUT_YD;
      panel_op(sm + op.pay, op.R, op.w, op.pad0, sm + op.in,
               to_y ? (deep ? B.ydeep : B.y) + op.out : sm + op.out,
               to_y ? (deep ? 0 : y_mode) : ((op.flags & OP_ACC) ? 1 : 0));
    }
    __syncthreads();
    if (t_staged && threadIdx.x == 0 && lv < 2) {  // trace: end of the first two levels
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      t_staged[4 + lv] = t;
    }
  }
  if (t_staged && threadIdx.x == 0) {  // trace: compute finished
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    t_staged[3] = t;
  }
  const int n_out = hd->n_out;
  const SpanCopy* souts = reinterpret_cast<const SpanCopy*>(sm + hd->pad[1]);  // staged with the data
  for (int i = 0; i < n_out; ++i) {
    const SpanCopy c = souts[i];
    double2* dst = (c.kind == SRC_XHAT ? B.xhat : B.yhat) + c.src;
    for (int e = threadIdx.x; e < c.elems; e += NTH) dst[e] = sm[c.smem + e];
  }
}

// both phases back to back (stand-alone span kernel)
template <int NTH>
__device__ __forceinline__ void run_span(const SpanHead* __restrict__ hd, const SpanCopy* __restrict__ copies,
                                         const SpanCopy* __restrict__ /*outs*/, const SpanBases& B,
                                         double2* sm, double2* /*red*/, uint64_t* bar, uint32_t phase,
                                         uint64_t* t_staged = nullptr) {
  span_stage_static<NTH>(hd, copies, B, sm, bar);
  span_finish<NTH>(hd, copies, B, sm, bar, phase, t_staged);
}
