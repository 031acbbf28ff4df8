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
#include <cstring>
#include <vector>

#include "h2b_common.cuh"

// h2b_near.cu: the q = 1 near-field streaming kernel on explicit work lists
int h2b_launch_near_list(const NearItem* items, int n_items, const NearBlk* blks, const double2* dbuf,
                         const double2* x, double2* y, int ns, int R, cudaStream_t st);
int h2b_near_rows_per_item(int ns, int r);
// h2b_far.cu: the q = 1 coupling kernels on explicit work lists
int h2b_launch_couple_list(const CoupleItem* items, int n, const double2* sbuf, const int32_t* xcol,
                           const double2* xhat, double2* yhat, int warp_mode, cudaStream_t st);

namespace {

constexpr int MM_WARPS = 16;                  // MMA warps (4 per SM sub-partition)
constexpr int MM_THREADS = 32 * (MM_WARPS + 1);  // + one producer warp (TMA issue, pad zeroing)
constexpr int MM_TPW = 128 / MM_WARPS;  // max 8x8 tiles per warp (8 q-tiles x 16 n-tiles / warps)
constexpr int MM_M = 64;         // complex rows per item
constexpr int MM_N = 64;         // complex columns per tile
constexpr int MM_K = 32;         // complex K per stage
constexpr int MM_AST = 34;       // A row stride (complex): 68 doubles -> conflict-free fragments
constexpr int MM_TST = 68;       // transposed-A row stride: 32 rows x 68 = the same 2176 elements
constexpr int MM_CST = 65;       // epilogue tile row stride (rows 16 bytes apart in the banks)
constexpr int MM_BST = 68;       // B row stride (complex): rows j, j+1 land 16 banks apart, so a
                                 // half-warp's 64-bit fragment loads of two rows never collide
constexpr int MM_STAGES = 3;
constexpr int MM_A_ELEMS = MM_M * MM_AST;
constexpr int MM_B_ELEMS = MM_K * MM_BST;
constexpr int MM_STAGE_ELEMS = MM_A_ELEMS + MM_B_ELEMS;
constexpr int MM_SMEM = 16 * MM_STAGES * MM_STAGE_ELEMS;
static_assert(MM_M * MM_CST <= MM_STAGE_ELEMS, "epilogue tile must fit in stage 0");
static_assert(MM_SMEM <= 227 * 1024, "shared memory budget");  // 202752 bytes

enum : int32_t { A_V = 0, A_T, A_S, A_D, A_VT, A_TT, A_N };
enum : int32_t { B_X = 0, B_XHAT, B_YHAT, B_N };
constexpr int B_SCR = B_N + 1;  // destination id of split-K parts (single-GPU multi-RHS plan)
constexpr int SEG_TRANS = 1 << 8;   // A[i][j] = src[a_off + j*lda + i]
constexpr int SEG_GATHER = 1 << 9;  // B row r = gather[b_row + r]
constexpr int ITEM_ACC = 1 << 8;
constexpr int ITEM_BCAST = 1 << 9;  // also store the result into every peer's buffer (same rows)
constexpr int MAX_PEERS = 8;

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
  double2* peers[MAX_PEERS];  // other ranks' exchange buffers (P2P-mapped), for ITEM_BCAST
  int npeers;
  double2* scratch;           // split-K partial planes (dst id B_SCR)
};

// the epilogue store of one output element: local (overwrite / accumulate) and, for
// ITEM_BCAST items, the same element of every peer's exchange buffer (NVLink P2P stores: the
// all-gather of x̂ fused into the producing kernel)
__device__ __forceinline__ void store_out(const MmBufs& bf, double2* C, int flags, int64_t idx, double2 v) {
  double2* o = C + idx;
  const double2 r = (flags & ITEM_ACC) ? cadd(*o, v) : v;
  *o = r;
  if (flags & ITEM_BCAST) {
#pragma unroll 1
    for (int p = 0; p < bf.npeers; ++p) bf.peers[p][idx] = r;
  }
}

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
  p = id == B_SCR ? bf.scratch : p;
  return id == B_N ? bf.y : p;
}

// y[e] = sum over the split-K planes, in plane order (deterministic)
__global__ void k_sum_parts(const double2* __restrict__ scr, int parts, int64_t plane, double2* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < plane; e += (int64_t)gridDim.x * blockDim.x) {
    double2 a = scr[e];
    for (int p = 1; p < parts; ++p) a = cadd(a, scr[p * plane + e]);
    y[e] = a;
  }
}


__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mm_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Staging of one K-chunk (segment) with TMA bulk copies (cp.async.bulk, one copy per
// contiguous row, completion counted on the stage's mbarrier): a handful of large requests per
// stage instead of thousands of 16-byte ones, so a single CTA per SM keeps enough bytes in flight.
//   A row-major (non-trans): smem [i][j] stride MM_AST, row i = k elements of source row i
//   A transposed (SEG_TRANS): smem [j][i] stride MM_TST, row j = m elements of source row j
//   B: smem [r][c] stride MM_BST, row r = qv elements of x / x̂ / ŷ row (contiguous or gathered)
// Shapes are not multiples of the MMA tiles, so the few pad elements the MMA reads (rows m..m4,
// column / row k when k is odd, columns qv..q8) are zeroed by the consumer after the copies land
// (they are disjoint from the copied bytes).
__device__ __forceinline__ void issue_seg(const MmSeg& s, const MmBufs& bf, int m, int q, int col0, int qv,
                                          double2* st, uint64_t* bar, int64_t brow) {
  const int lane = threadIdx.x & 31;
  const double2* A = pick_a(bf, s.flags & 15) + s.a_off;
  const double2* B = pick_b(bf, (s.flags >> 4) & 15);
  const bool trans = s.flags & SEG_TRANS;
  const int na = trans ? s.k : m;          // A rows to copy
  const int la = trans ? m : s.k;          // elements per A row
  // every producer lane arrives (count 32): each lane's own pad stores are released by its own
  // arrive; lane 0 also announces the transaction bytes
  if (lane == 0) mbar_arrive_expect_tx(bar, 16u * (uint32_t)(na * la + s.k * qv));
  else mm_arrive(bar);
  __syncwarp();
  double2* As = st;
  double2* Bs = st + MM_A_ELEMS;
  for (int r = lane; r < na; r += 32)
    bulk_g2s(As + r * (trans ? MM_TST : MM_AST), A + (int64_t)r * s.lda, 16u * la, bar);
  if (lane < s.k) bulk_g2s(Bs + lane * MM_BST, B + brow * q + col0, 16u * qv, bar);  // k <= 32
}

// B row of this lane for a segment (gather index or contiguous row), loaded by the producer
// before it waits for the stage to drain, so the index latency overlaps the wait
__device__ __forceinline__ int64_t seg_brow(const MmSeg& s, const MmBufs& bf, int lane) {
  if (lane >= s.k) return 0;
  return (s.flags & SEG_GATHER) ? (int64_t)__ldg(bf.gather + s.b_row + lane) : s.b_row + lane;
}

__device__ __forceinline__ void zero_pads(const MmSeg& s, int m, int qv, double2* st, int lane) {
  const double2 z = make_double2(0.0, 0.0);
  const bool trans = s.flags & SEG_TRANS;
  const int m4 = (m + 3) & ~3, k = s.k, k2 = (k + 1) & ~1, q8 = (qv + 7) & ~7;
  double2* As = st;
  double2* Bs = st + MM_A_ELEMS;
  // A: rows (non-trans) / columns (trans) m..m4 for every j < k2; j = k (odd k) for i < m
  for (int e = lane; e < (m4 - m) * k2; e += 32) {
    const int i = m + e / k2, j = e % k2;
    As[trans ? j * MM_TST + i : i * MM_AST + j] = z;
  }
  if (k & 1)
    for (int i = lane; i < m; i += 32) As[trans ? k * MM_TST + i : i * MM_AST + k] = z;
  // B: columns qv..q8 of rows < k2; row k (odd k) for columns < qv
  for (int e = lane; e < (q8 - qv) * k2; e += 32) {
    const int r = e / (q8 - qv), c = qv + e % (q8 - qv);
    Bs[r * MM_BST + c] = z;
  }
  if (k & 1)
    for (int c = lane; c < qv; c += 32) Bs[k * MM_BST + c] = z;
}

// One staged chunk: nks k4-steps of NU 8x8 tiles per warp (A fragment: B_rᵀ, shared by the NU
// tiles; B fragments: A_rᵀ, with the lane's re/im pick and sign bit folded into the address/XOR).
template <int NU>
__device__ __forceinline__ void mma_chunk(double (&acc)[MM_TPW][2], const double* Bs, const double* bq,
                                          int a_off, int si, int sj, int nks, int jo, int G,
                                          unsigned long long neg) {
#pragma unroll 2
  for (int ks = 0; ks < nks; ++ks) {
    const int j = ks * 2 + jo;
    const double af = Bs[j * (2 * MM_BST) + a_off];
    const double* bp = bq + j * sj;
    double bv[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u)
      bv[u] = __longlong_as_double(__double_as_longlong(bp[u * G * 4 * si]) ^ neg);
#pragma unroll
    for (int u = 0; u < NU; ++u) dmma(acc[u][0], acc[u][1], af, bv[u]);
  }
}

// The MMA runs on the TRANSPOSED real product, C_rᵀ (q x 2m) = B_rᵀ (q x 2k) A_rᵀ (2k x 2m):
// its M dimension is the column tile (64 of the q right-hand sides, always full at q >= 64) and
// its N dimension is 2m in steps of 8, so an item with m rows costs ceil(m/4) n-tiles instead of
// a full 64-row tile (ranks k_t ~ 12-84 at cfg3: the coupling/transfer phases would otherwise
// waste ~40 % of the tensor work on padding).  Tiles (8 q-rows x 8 real columns) are dealt to
// the 8 warps so every SM sub-partition gets the same share: warp w owns q-tile mt = w % MTP
// and the n-tiles nt = w / MTP + G u (MTP = q-tiles rounded up to a power of two, G = 8 / MTP).
// Each lane's accumulator pair is then (re, im) of one complex output element.
__global__ void __launch_bounds__(MM_THREADS, 1) k_zgemm_grouped(const MmItem* __restrict__ items,
                                                                 const MmSeg* __restrict__ segs,
                                                                 MmBufs bf, int q) {
  extern __shared__ __align__(16) double2 sm[];
  const MmItem it = items[blockIdx.x];
  const int col0 = blockIdx.y * MM_N;
  // warp 0 is the producer; MMA warps are numbered 0..MM_WARPS-1 from threadIdx 32 on
  const int lane = threadIdx.x & 31;
  const bool producer = threadIdx.x < 32;
  const int warp = producer ? MM_WARPS : (threadIdx.x >> 5) - 1;
  const int qv = min(MM_N, q - col0);          // valid columns of this tile
  const int MT = (qv + 7) >> 3;                // q-tiles of 8
  const int MTP = MT <= 1 ? 1 : MT <= 2 ? 2 : MT <= 4 ? 4 : 8;
  const int G = MM_WARPS / MTP;
  const int mt = warp % MTP, ng = warp / MTP;
  const int NT = (2 * it.m + 7) >> 3;          // real n-tiles of 8 (<= 16)
  const bool active = !producer && mt < MT;   // the producer warp owns no tiles
  const int nu = NT > ng ? (NT - ng + G - 1) / G : 0;  // n-tiles of this warp
  // lane-constant fragment geometry
  const int kk = lane & 3, b = kk & 1, jo = kk >> 1;
  // A operand (B_rᵀ, m8 x k4 row): row c = mt*8 + lane/4, col kr -> complex row j, part b
  const int a_off = (mt * 8 + (lane >> 2)) * 2 + b;
  // B operand (A_rᵀ, k4 x n8 col): col n = nt*8 + lane/4 -> complex row i = nt*4 + lane/8, part
  // a = (lane/4)&1; value {re, -im; im, re}[a][b] of A[i][j]
  const int a = (lane >> 2) & 1;
  const int pick = a ^ b;
  const unsigned long long neg = (a == 0 && b == 1) ? 0x8000000000000000ull : 0ull;

  double acc[MM_TPW][2];
#pragma unroll
  for (int u = 0; u < MM_TPW; ++u) acc[u][0] = acc[u][1] = 0.0;

  __shared__ __align__(8) uint64_t full[MM_STAGES], empty[MM_STAGES];
  if (threadIdx.x == 0)
    for (int i = 0; i < MM_STAGES; ++i) {
      mbar_init(&full[i], 32);
      mbar_init(&empty[i], MM_WARPS);
    }
  __syncthreads();
  const int ns = it.nseg;
  if (producer) {
    // producer: wait until the buffer's previous chunk is consumed, zero its pads, copy
    for (int s = 0; s < ns; ++s) {
      const int buf = s % MM_STAGES;
      const MmSeg sg = segs[it.seg0 + s];
      const int64_t brow = seg_brow(sg, bf, lane);  // in flight while we wait for the stage
      if (s >= MM_STAGES) mbar_wait(&empty[buf], (uint32_t)(s / MM_STAGES - 1) & 1u);
      double2* st = sm + buf * MM_STAGE_ELEMS;
      zero_pads(sg, it.m, qv, st, lane);
      __syncwarp();
      // order the generic-proxy pad stores (this chunk's and the buffer's earlier ones) before
      // the async-proxy TMA writes into the same buffer
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_seg(sg, bf, it.m, q, col0, qv, st, &full[buf], brow);  // lane 0 arrives first
    }
  } else {
    for (int s = 0; s < ns; ++s) {
      const int buf = s % MM_STAGES;
      const int kc = segs[it.seg0 + s].k;
      const bool tr = segs[it.seg0 + s].flags & SEG_TRANS;
      mbar_wait(&full[buf], (uint32_t)(s / MM_STAGES) & 1u);
      if (active) {
        const double* As = reinterpret_cast<const double*>(sm + buf * MM_STAGE_ELEMS);
        const double* Bs = As + 2 * MM_A_ELEMS;
        const int nks = (2 * kc + 3) >> 2;         // k4 steps holding data (the rest is padding)
        // B-operand offsets: row-major A[i][j] -> i*AST + j, transposed -> j*TST + i (x2 doubles)
        const int si = tr ? 2 : 2 * MM_AST;
        const int sj = tr ? 2 * MM_TST : 2;
        const double* bq = As + (lane >> 3) * si + pick + ng * 4 * si;
        switch (nu) {  // compile-time tile counts: no predicated-off DMMA, no early exits
#define MMC(NU) case NU: mma_chunk<NU>(acc, Bs, bq, a_off, si, sj, nks, jo, G, neg); break;
          MMC(1) MMC(2) MMC(3) MMC(4) MMC(5) MMC(6) MMC(7) MMC(8)
#undef MMC
          default: break;
        }
      }
      __syncwarp();
      if (lane == 0) mm_arrive(&empty[buf]);
    }
  }
  __syncthreads();
  // epilogue: lane holds C_rᵀ[c][n..n+1] = (re, im) of C[i][c], i = nt*4 + lane%4
  double2* Cs = sm;
  if (active) {
    const int c = mt * 8 + (lane >> 2);
#pragma unroll
    for (int u = 0; u < MM_TPW; ++u) {
      if (u >= nu) break;
      Cs[((ng + G * u) * 4 + kk) * MM_CST + c] = make_double2(acc[u][0], acc[u][1]);
    }
  }
  __syncthreads();
  const int dst_id = it.flags & 15;
  double2* C = pick_b(bf, dst_id);
  for (int e = threadIdx.x; e < it.m * MM_N; e += MM_THREADS) {
    const int i = e >> 6, c = e & (MM_N - 1);
    if (c >= qv) continue;
    store_out(bf, C, it.flags, (it.c_row + i) * q + col0 + c, Cs[i * MM_CST + c]);
  }
  if (it.flags & ITEM_BCAST) __threadfence_system();
  // the next CTA on this SM fills the same shared memory with TMA: order this CTA's generic
  // stores (epilogue tile, pads) before any async-proxy write
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// q = 1: the same item / segment lists as a grouped complex GEMV on the CUDA cores (memory-
// bound).  512 threads: thread (row i, part g of 8) accumulates 4 K-entries of each segment
// (row-major A: 8 lanes read one 512-byte A row; transposed A: 64 lanes read 64 consecutive
// elements).  The item's segment descriptors are staged in shared memory first, and two
// segments are loaded per step (8 independent 16-byte streaming loads in flight per thread), so
// the loop never waits on a descriptor load.  The 8 partial sums of a row are combined in a
// fixed order (deterministic).
constexpr int MV_THREADS = 512;
constexpr int MV_SEGS = 256;  // descriptors staged per pass (8 KB)

__device__ __forceinline__ double2 ld_na(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <bool GATHER>
__global__ void __launch_bounds__(MV_THREADS, 1) k_zgemv_grouped(const MmItem* __restrict__ items,
                                                                 const MmSeg* __restrict__ segs,
                                                                 MmBufs bf) {
  __shared__ double2 red[8][MM_M];
  __shared__ MmSeg ss[MV_SEGS];
  const MmItem it = items[blockIdx.x];
  // all segments of an item share the A orientation (checked by h2b_plan_set_phase)
  const bool trans = it.nseg > 0 && (segs[it.seg0].flags & SEG_TRANS);
  const int i = trans ? (threadIdx.x & (MM_M - 1)) : (threadIdx.x >> 3);
  const int g = trans ? (threadIdx.x >> 6) : (threadIdx.x & 7);
  const int j0 = g * 4;
  const bool row_ok = i < it.m;
  double2 acc = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < it.nseg; c0 += MV_SEGS) {
    const int n = min(MV_SEGS, it.nseg - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += MV_THREADS) ss[e] = segs[it.seg0 + c0 + e];
    __syncthreads();
    if (!row_ok) continue;
    constexpr int SU = 4;  // segments per step: 16 streaming loads (256 B) in flight per thread
    for (int s0 = 0; s0 < n; s0 += SU) {
      double2 av[SU][4];
#pragma unroll
      for (int h = 0; h < SU; ++h) {
        const bool live = s0 + h < n;
        const MmSeg& sg = ss[live ? s0 + h : s0];
        const double2* A = pick_a(bf, sg.flags & 15) + sg.a_off;
        const int64_t step = trans ? sg.lda : 1;
        const double2* Ap = A + (trans ? (int64_t)i : (int64_t)i * sg.lda) + (int64_t)j0 * step;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          av[h][u] = (live && j0 + u < sg.k) ? ld_na(Ap + u * step) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int h = 0; h < SU; ++h) {  // x / x̂ / ŷ rows: L1/L2 hits, read when the A stream lands
        if (s0 + h >= n) break;
        const MmSeg& sg = ss[s0 + h];
        const double2* B = pick_b(bf, (sg.flags >> 4) & 15);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < sg.k) {
            int64_t row = sg.b_row + j0 + u;
            if constexpr (GATHER)
              if (sg.flags & SEG_GATHER) row = (int64_t)__ldg(bf.gather + row);
            cfma(acc, av[h][u], __ldg(B + row));
          }
      }
    }
  }
  red[g][i] = acc;
  __syncthreads();
  if (threadIdx.x < it.m) {
    const int r = threadIdx.x;
    double2 v = red[0][r];
#pragma unroll
    for (int gg = 1; gg < 8; ++gg) v = cadd(v, red[gg][r]);
    store_out(bf, pick_b(bf, it.flags & 15), it.flags, it.c_row + r, v);
    if (it.flags & ITEM_BCAST) __threadfence_system();
  }
}

int run_grouped(const MmItem* items, int n_items, const MmSeg* segs, const MmBufs& bf, int q,
                cudaStream_t st, int* nl, bool gather = true) {
  const int nct = (q + MM_N - 1) / MM_N;
  for (int i0 = 0; i0 < n_items; i0 += 65535) {
    const int cnt = std::min(65535, n_items - i0);
    if (q == 1 && gather)
      k_zgemv_grouped<true><<<cnt, MV_THREADS, 0, st>>>(items + i0, segs, bf);
    else if (q == 1)
      k_zgemv_grouped<false><<<cnt, MV_THREADS, 0, st>>>(items + i0, segs, bf);
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
  int split = 1;               // split-K parts of the near-field launch (1: none)
  int csplit = 1;              // split-K parts of the coupling launch (1: none)
  int couple_launch = -1;      // index of the coupling launch in `launches`
  int64_t scratch_rows = 0;    // rows of the split planes: max(split x N, csplit x K)
  double2* scratch = nullptr;  // split planes (near: split x N x q; coupling: csplit x K x q)
  int64_t scratch_q = 0;
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
  // small operators (fewer coupling items than two per SM): every item's K-chunks are split into
  // csplit parts writing partial planes (K x q each), summed into ŷ in a fixed order (as the
  // near field below; measured at cfg1 q = 64: the coupling launch was the longest phase)
  int n_couple_items = 0, max_cchunks = 0;
  for (int t = 0; t < P; ++t) {
    const int kt = h->c_rank[t];
    if (kt == 0) continue;
    const int R = (int)(prow_h[t + 1] - prow_h[t]);
    n_couple_items += (kt + MM_M - 1) / MM_M;
    max_cchunks = std::max(max_cchunks, (R + MM_K - 1) / MM_K);
  }
  int csplit = 1;
  if (n_couple_items > 0 && n_couple_items < 2 * 148 && !getenv("H2B_MRHS_NO_CSPLIT"))
    csplit = std::max(1, std::min({8, (2 * 148 + n_couple_items - 1) / n_couple_items, max_cchunks / 4}));
  if (const char* e = getenv("H2B_MRHS_CSPLIT")) csplit = std::max(1, std::min(16, atoi(e)));  // tuning aid
  for (int t = 0; t < P; ++t) {
    const int kt = h->c_rank[t];
    if (kt == 0) continue;
    const int64_t b0 = h->s_row_ptr[t];
    const int R = (int)(prow_h[t + 1] - prow_h[t]);
    const int nch = (R + MM_K - 1) / MM_K;
    for (int m0 = 0; m0 < kt; m0 += MM_M) {
      for (int pt = 0; pt < csplit; ++pt) {
        const int c_lo = nch * pt / csplit, c_hi = nch * (pt + 1) / csplit;
        const int r_lo = c_lo * MM_K, r_hi = std::min(R, c_hi * MM_K);
        const int s0 = B.begin_item();
        if (r_hi > r_lo)
          B.seg(A_S, h->s_off[b0] + (int64_t)r_lo * kt, kt, true, m0, r_hi - r_lo, B_XHAT, prow_h[t] + r_lo, true);
        if (csplit == 1)
          B.end_item(s0, h->c_xoff[t] + m0, std::min(MM_M, kt - m0), B_YHAT, false);
        else
          B.end_item(s0, (int64_t)pt * h->K + h->c_xoff[t] + m0, std::min(MM_M, kt - m0), B_SCR, false);
      }
    }
  }
  const int couple_launch = (int)B.launches.size();
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
  // near-field + leaf back-transform, one item per (leaf, 64-row chunk): y overwritten.  Small
  // operators (fewer items than two per SM) split every item's segment list into `split` parts
  // writing partial planes, summed in a fixed order afterwards (deterministic split-K).
  int n_near_items = 0, max_segs = 0;
  for (int t : h->h_leaves) {
    n_near_items += (h->c_size[t] + MM_M - 1) / MM_M;
    max_segs = std::max<int>(max_segs, (int)(h->d_row_ptr[t + 1] - h->d_row_ptr[t]) + 1);
  }
  int split = 1;
  if (n_near_items > 0 && n_near_items < 2 * 148)
    split = std::max(1, std::min({8, (2 * 148 + n_near_items - 1) / n_near_items, max_segs / 4}));
  if (const char* e = getenv("H2B_MRHS_SPLIT")) split = std::max(1, std::min(16, atoi(e)));  // tuning aid
  for (int t : h->h_leaves) {
    const int nt = h->c_size[t];
    for (int m0 = 0; m0 < nt; m0 += MM_M) {
      std::vector<int> bl;  // logical segments: partner blocks, then the leaf basis (-1)
      for (int64_t b = h->d_row_ptr[t]; b < h->d_row_ptr[t + 1]; ++b) bl.push_back((int)(b - h->d_row_ptr[t]));
      if (h->c_rank[t] > 0) bl.push_back(-1);
      const int parts = split;
      for (int pt = 0; pt < parts; ++pt) {
        const size_t lo = bl.size() * pt / parts, hi = bl.size() * (pt + 1) / parts;
        const int s0 = B.begin_item();
        for (size_t u = lo; u < hi; ++u) {
          if (bl[u] < 0) {
            B.seg(A_V, h->c_voff[t], h->c_rank[t], false, m0, h->c_rank[t], B_YHAT, h->c_xoff[t], false);
          } else {
            const int64_t b = h->d_row_ptr[t] + bl[u];
            const int s = h->d_col[b];
            B.seg(A_D, h->d_off[b], h->c_size[s], false, m0, h->c_size[s], B_X, h->c_start[s], false);
          }
        }
        if (split == 1)
          B.end_item(s0, h->c_start[t] + m0, std::min(MM_M, nt - m0), B_N, false);
        else
          B.end_item(s0, (int64_t)pt * h->n + h->c_start[t] + m0, std::min(MM_M, nt - m0), B_SCR, false);
      }
    }
  }
  B.end_launch();

  auto* plan = new MrhsPlan();
  plan->launches = B.launches;
  plan->split = split;
  plan->csplit = csplit;
  plan->couple_launch = (int)plan->launches.size() > couple_launch ? couple_launch : -1;
  plan->scratch_rows = std::max<int64_t>(split > 1 ? (int64_t)split * h->n : 0, csplit > 1 ? (int64_t)csplit * h->K : 0);
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
  cudaFree(h->mrhs->scratch);
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
  bf.scratch = h->mrhs->scratch;
  for (size_t li = 0; li < h->mrhs->launches.size(); ++li) {
    const int2& L = h->mrhs->launches[li];
    H2B_TRY(run_grouped(h->mrhs->items + L.x, L.y, h->mrhs->segs, bf, q, st, nl));
    if ((int)li == h->mrhs->couple_launch && h->mrhs->csplit > 1) {  // ŷ = Σ coupling parts
      const int64_t plane = h->K * q;
      k_sum_parts<<<(int)std::min<int64_t>((plane + 255) / 256, 148 * 8), 256, 0, st>>>(
          h->mrhs->scratch, h->mrhs->csplit, plane, h->yhat);
      H2B_CHECK_LAUNCH();
      ++*nl;
    }
  }
  if (h->mrhs->split > 1) {
    const int64_t plane = h->n * q;
    k_sum_parts<<<(int)std::min<int64_t>((plane + 255) / 256, 148 * 8), 256, 0, st>>>(h->mrhs->scratch, h->mrhs->split,
                                                                                      plane, yp);
    H2B_CHECK_LAUNCH();
    ++*nl;
  }
  return H2B_OK;
}

// split-K planes for q columns (allocated before any graph capture)
int h2b_mrhs_workspace(h2b_ctx* h, int q) {
  H2B_TRY(h2b_mrhs_prepare(h));
  MrhsPlan* p = h->mrhs;
  if (p->scratch_rows == 0 || p->scratch_q >= q) return H2B_OK;
  h2b_release_graphs(h);  // captured graphs hold the old planes
  cudaFree(p->scratch);
  p->scratch = nullptr;
  p->scratch_q = 0;
  H2B_CUDA_TRY(cudaMalloc(&p->scratch, sizeof(double2) * (size_t)p->scratch_rows * q));
  p->scratch_q = q;
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
    bool gather = false;  // any SEG_GATHER segment (selects the GEMV instantiation)
  };
  std::vector<Phase> phases;
  int64_t device_bytes = 0;
  double2* peers[MAX_PEERS] = {};
  double2** dpeers = nullptr;  // device copy of `peers`
  int32_t* gather = nullptr;   // B-row index table of SEG_GATHER segments
  int64_t n_gather = 0;
  int npeers = 0;
  int64_t peer_off = 0;        // element offset added to every peer pointer (ping-pong buffers)
  // q = 1 near-field on the streaming kernel (h2b_plan_set_near_fast): y overwritten from
  // payload 4 (D) and the exchange buffer, then phase 5 (leaf back, accumulating) instead of 4
  NearItem* nf_items = nullptr;
  NearBlk* nf_blks = nullptr;
  int nf_n = 0, nf_ns = 0, nf_r = 0;
  // q = 1 coupling on the panel kernels (h2b_plan_set_couple_fast): payload 3 holds Sᵀ panels
  CoupleItem* cf_items = nullptr;
  int32_t* cf_xcol = nullptr;
  int cf_n = 0, cf_warp = 0;
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
        (it.flags & 15) > B_N || (it.flags & ~(15 | ITEM_ACC | ITEM_BCAST))) {
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
        ((sg.flags & SEG_GATHER) && (sg.b_row < 0 || sg.b_row + sg.k > p->n_gather))) {
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
  ph.gather = false;
  for (int64_t i = 0; i < n_segs; ++i) ph.gather |= (segs[i].flags & SEG_GATHER) != 0;
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
  if (p && phase == H2B_PLAN_PHASE_NEAR_FAST) {  // the q = 1 streaming near-field alone
    if (q != 1 || p->nf_n == 0) {
      h2b_set_error("h2b_plan_run: the near-field-only phase needs q = 1 and h2b_plan_set_near_fast");
      return H2B_EINVAL;
    }
    return h2b_launch_near_list(p->nf_items, p->nf_n, p->nf_blks, p->pay[4], (const double2*)x, (double2*)y,
                                p->nf_ns, p->nf_r, (cudaStream_t)stream);
  }
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
  bf.gather = p->gather;
  for (int i = 0; i < p->npeers; ++i) bf.peers[i] = p->peers[i] + p->peer_off;
  bf.npeers = p->npeers;
  int nl = 0;
  if (phase == 2 && q == 1 && p->cf_n > 0)
    return h2b_launch_couple_list(p->cf_items, p->cf_n, p->pay[3], p->cf_xcol, bf.b[B_XHAT], bf.b[B_YHAT],
                                  p->cf_warp, (cudaStream_t)stream);
  if (phase == 4 && q == 1 && p->nf_n > 0) {
    H2B_TRY(h2b_launch_near_list(p->nf_items, p->nf_n, p->nf_blks, p->pay[4], bf.b[B_X], bf.y, p->nf_ns,
                                 p->nf_r, (cudaStream_t)stream));
    phase = 5;  // then the leaf back-transform items (accumulate)
    if (phase >= (int)p->phases.size()) return H2B_OK;
  }
  const auto& ph = p->phases[phase];
  for (const int2& L : ph.launches)
    H2B_TRY(run_grouped(ph.items + L.x, L.y, ph.segs, bf, q, (cudaStream_t)stream, &nl, ph.gather));
  return H2B_OK;
}

namespace {
// rows [r0, r0 + nrows) of `src` (q columns) into `dst` at the same rows, for every peer
__global__ void k_bcast_rows(const double2* __restrict__ src, int64_t off, int64_t n,
                             double2* const* __restrict__ peers, int np, int64_t peer_off) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = src[off + e];
    for (int p = 0; p < np; ++p) peers[p][peer_off + off + e] = v;
  }
  __threadfence_system();
}
}  // namespace

extern "C" int h2b_plan_set_peers(h2b_plan_handle p, void* const* peer_bufs, int npeers) {
  if (!p || npeers < 0 || npeers > MAX_PEERS || (npeers && !peer_bufs)) {
    h2b_set_error("h2b_plan_set_peers: bad arguments (at most 8 peers)");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  for (int i = 0; i < npeers; ++i) p->peers[i] = (double2*)peer_bufs[i];
  p->npeers = npeers;
  if (!p->dpeers) H2B_CUDA_TRY(cudaMalloc(&p->dpeers, sizeof(double2*) * MAX_PEERS));
  if (npeers)  // device copy of the table for k_bcast_rows (set once, outside any capture)
    H2B_CUDA_TRY(cudaMemcpy(p->dpeers, p->peers, sizeof(double2*) * npeers, cudaMemcpyHostToDevice));
  return H2B_OK;
}

extern "C" int h2b_plan_bcast_rows(h2b_plan_handle p, const void* buf, int64_t row0, int64_t nrows, int q,
                                   void* stream) {
  if (!p || !buf || row0 < 0 || nrows < 0 || q < 1) {
    h2b_set_error("h2b_plan_bcast_rows: bad arguments");
    return H2B_EINVAL;
  }
  if (p->npeers == 0 || nrows == 0) return H2B_OK;
  const int64_t n = nrows * q;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_bcast_rows<<<grid, 256, 0, (cudaStream_t)stream>>>((const double2*)buf, row0 * q, n, p->dpeers, p->npeers,
                                                        p->peer_off);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

// payload access for the fill kernels (h2b_fill.cu)
double2* h2b_plan_payload(h2b_plan_handle p, int payload, int64_t* elems, int* device) {
  if (!p || payload < 0 || payload >= p->n_payloads) return nullptr;
  *elems = p->pay_elems[payload];
  *device = p->device;
  return p->pay[payload];
}

extern "C" int h2b_plan_set_near_fast(h2b_plan_handle p, const void* items, int64_t n_items, const void* blks,
                                      int64_t n_blks, int ns, int rows_per_thread) {
  if (!p || n_items < 0 || n_blks < 0 || (n_items && (!items || !blks)) || p->n_payloads < 5 ||
      h2b_near_rows_per_item(ns, rows_per_thread) == 0 || n_items > (1 << 30)) {
    h2b_set_error("h2b_plan_set_near_fast: bad arguments (leaf size 32/64, rows per thread 1/2/4, "
                  "payload 4 = near-field)");
    return H2B_EINVAL;
  }
  const NearItem* it = (const NearItem*)items;
  const NearBlk* bl = (const NearBlk*)blks;
  const int64_t rb = h2b_near_rows_per_item(ns, rows_per_thread);
  for (int64_t i = 0; i < n_items; ++i)  // the kernel trusts the lists
    if (it[i].b_first < 0 || it[i].nb < 0 || it[i].b_first + (int64_t)it[i].nb > n_blks || it[i].row0 < 0 ||
        it[i].row0 + rb > ns) {
      h2b_set_error("h2b_plan_set_near_fast: item " + std::to_string(i) + " out of range");
      return H2B_EINVAL;
    }
  for (int64_t b = 0; b < n_blks; ++b)
    if (bl[b].d_off < 0 || bl[b].d_off + (int64_t)ns * ns > p->pay_elems[4]) {
      h2b_set_error("h2b_plan_set_near_fast: block " + std::to_string(b) + " outside the near-field payload");
      return H2B_EINVAL;
    }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  cudaFree(p->nf_items);
  cudaFree(p->nf_blks);
  p->nf_items = nullptr;
  p->nf_blks = nullptr;
  p->nf_n = 0;
  H2B_CUDA_TRY(cudaMalloc(&p->nf_items, sizeof(NearItem) * std::max<int64_t>(n_items, 1)));
  H2B_CUDA_TRY(cudaMalloc(&p->nf_blks, sizeof(NearBlk) * std::max<int64_t>(n_blks, 1)));
  if (n_items) H2B_CUDA_TRY(cudaMemcpy(p->nf_items, items, sizeof(NearItem) * n_items, cudaMemcpyHostToDevice));
  if (n_blks) H2B_CUDA_TRY(cudaMemcpy(p->nf_blks, blks, sizeof(NearBlk) * n_blks, cudaMemcpyHostToDevice));
  p->nf_n = (int)n_items;
  p->nf_ns = ns;
  p->nf_r = rows_per_thread;
  return H2B_OK;
}

extern "C" int h2b_plan_set_couple_fast(h2b_plan_handle p, const void* items, int64_t n_items,
                                        const int32_t* xcol, int64_t n_xcol) {
  if (!p || n_items < 0 || n_xcol < 0 || (n_items && !items) || (n_xcol && !xcol) || p->n_payloads < 4 ||
      n_items > (1 << 30)) {
    h2b_set_error("h2b_plan_set_couple_fast: bad arguments (payload 3 = coupling panels)");
    return H2B_EINVAL;
  }
  const CoupleItem* it = (const CoupleItem*)items;
  int64_t elems = 0;
  for (int64_t i = 0; i < n_items; ++i) {  // the kernels trust the lists
    if (it[i].R < 0 || it[i].w < 0 || it[i].xcol < 0 || it[i].xcol + it[i].R > n_xcol || it[i].panel < 0 ||
        it[i].panel + (int64_t)it[i].R * it[i].w > p->pay_elems[3] || it[i].out < 0) {
      h2b_set_error("h2b_plan_set_couple_fast: item " + std::to_string(i) + " out of range");
      return H2B_EINVAL;
    }
    elems += (int64_t)it[i].R * it[i].w;
  }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  cudaFree(p->cf_items);
  cudaFree(p->cf_xcol);
  p->cf_items = nullptr;
  p->cf_xcol = nullptr;
  p->cf_n = 0;
  H2B_CUDA_TRY(cudaMalloc(&p->cf_items, sizeof(CoupleItem) * std::max<int64_t>(n_items, 1)));
  H2B_CUDA_TRY(cudaMalloc(&p->cf_xcol, sizeof(int32_t) * std::max<int64_t>(n_xcol, 1)));
  if (n_items) H2B_CUDA_TRY(cudaMemcpy(p->cf_items, items, sizeof(CoupleItem) * n_items, cudaMemcpyHostToDevice));
  if (n_xcol) H2B_CUDA_TRY(cudaMemcpy(p->cf_xcol, xcol, sizeof(int32_t) * n_xcol, cudaMemcpyHostToDevice));
  p->cf_n = (int)n_items;
  p->cf_warp = (n_items > 0 && elems / n_items < 4096) ? 1 : 0;  // as the single-GPU planner
  return H2B_OK;
}

extern "C" int h2b_plan_set_gather(h2b_plan_handle p, const int32_t* idx, int64_t n) {
  if (!p || n < 0 || (n && !idx)) {
    h2b_set_error("h2b_plan_set_gather: bad arguments");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(p->device));
  cudaFree(p->gather);
  p->gather = nullptr;
  H2B_CUDA_TRY(cudaMalloc(&p->gather, sizeof(int32_t) * std::max<int64_t>(n, 1)));
  if (n) H2B_CUDA_TRY(cudaMemcpy(p->gather, idx, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  p->n_gather = n;
  p->device_bytes += 4 * n;
  return H2B_OK;
}

extern "C" int h2b_plan_set_peer_offset(h2b_plan_handle p, int64_t elems) {
  if (!p || elems < 0) {
    h2b_set_error("h2b_plan_set_peer_offset: bad arguments");
    return H2B_EINVAL;
  }
  p->peer_off = elems;
  return H2B_OK;
}

// raw device allocations (exchange buffers that are shared with CUDA IPC)
extern "C" int h2b_device_alloc(int device, size_t bytes, void** out) {
  if (!out) {
    h2b_set_error("h2b_device_alloc: null argument");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(device));
  H2B_CUDA_TRY(cudaMalloc(out, std::max<size_t>(bytes, 16)));
  H2B_CUDA_TRY(cudaMemset(*out, 0, std::max<size_t>(bytes, 16)));
  return H2B_OK;
}

extern "C" int h2b_device_free(void* ptr) {
  if (ptr) H2B_CUDA_TRY(cudaFree(ptr));
  return H2B_OK;
}

// CUDA IPC of an exchange buffer between the ranks' processes (one process per GPU)
extern "C" int h2b_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 bytes */) {
  if (!dev_ptr || !handle_out) {
    h2b_set_error("h2b_ipc_get_handle: null argument");
    return H2B_EINVAL;
  }
  cudaIpcMemHandle_t hd;
  H2B_CUDA_TRY(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)));
  memcpy(handle_out, &hd, sizeof(hd));
  return H2B_OK;
}

extern "C" int h2b_ipc_open(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) {
    h2b_set_error("h2b_ipc_open: null argument");
    return H2B_EINVAL;
  }
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  H2B_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr_out, hd, cudaIpcMemLazyEnablePeerAccess));
  return H2B_OK;
}

extern "C" int h2b_ipc_close(void* dev_ptr) {
  if (dev_ptr) H2B_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
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
  if (p->dpeers) cudaFree(p->dpeers);
  if (p->gather) cudaFree(p->gather);
  cudaFree(p->nf_items);
  cudaFree(p->nf_blks);
  cudaFree(p->cf_items);
  cudaFree(p->cf_xcol);
  delete p;
  return H2B_OK;
}

extern "C" int64_t h2b_plan_device_bytes(h2b_plan_handle p) { return p ? p->device_bytes : -1; }
