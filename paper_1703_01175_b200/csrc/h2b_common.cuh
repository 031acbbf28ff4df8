// Shared device helpers and the handle layout of the h2b C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
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
      h2b_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
      return _e == cudaErrorMemoryAllocation ? H2B_ENOMEM : H2B_ECUDA;              \
    }                                                                               \
  } while (0)

#define H2B_CHECK_LAUNCH() H2B_CUDA_TRY(cudaGetLastError())

// ---------------------------------------------------------------------------
// complex128 arithmetic on interleaved double2 (no fast-math, exact FMA order)
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
// handle
// ---------------------------------------------------------------------------
struct h2b_ctx {
  int device = 0;
  int64_t n = 0;
  int depth = 0;
  int P = 0;
  int64_t K = 0;
  int64_t n_coupling = 0, n_near = 0;
  int64_t sec_elems[4] = {0, 0, 0, 0};
  int64_t sec_uploaded[4] = {0, 0, 0, 0};
  int uniform_leaf = 0;  // leaf size if all leaves share it, else 0

  // host copies of the tables (scheduling decisions)
  std::vector<int32_t> level_ptr, c_rank, c_child_lo, c_size;
  std::vector<int32_t> up_levels;    // levels with any k>0 cluster (deepest first)
  std::vector<int32_t> down_levels;  // levels with any non-leaf k>0 cluster (root first)
  std::vector<int32_t> h_leaves;

  // device tables
  int32_t *c_start = nullptr, *c_size_d = nullptr, *c_rank_d = nullptr, *c_lo = nullptr,
          *c_hi = nullptr, *c_parent = nullptr;
  int64_t *c_xoff = nullptr, *c_voff = nullptr, *c_toff = nullptr;
  int64_t *s_row_ptr = nullptr, *s_off = nullptr, *d_row_ptr = nullptr, *d_off = nullptr;
  int32_t *s_col = nullptr, *d_col = nullptr;
  int64_t* perm = nullptr;
  int32_t* leaves = nullptr;
  int n_leaves = 0;
  // payloads
  double2* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  // workspace (grown on demand, per q)
  double2 *xhat = nullptr, *yhat = nullptr;
  int64_t ws_q = 0;
  double2 *hx = nullptr, *hy = nullptr, *hxp = nullptr, *hyp = nullptr;  // host-path staging
  int64_t hws_q = 0;
  // krylov workspace
  void* kry = nullptr;
  size_t kry_bytes = 0;
  int64_t device_bytes = 0;
};

// implemented in h2b_matvec.cu
int h2b_ensure_workspace(h2b_ctx* h, int q);
int h2b_run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st);
int h2b_launch_gather(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                      cudaStream_t st);
int h2b_launch_scatter(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                       cudaStream_t st);
