// Latency of one "level" of small complex panel GEMVs executed by a 256-thread CTA from
// shared memory: (a) warp per op with a shuffle reduction (current panel_op scheme) vs
// (b) thread per output column with S-way row split (slot table), for realistic shapes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
struct Op { int pay, in, out, R, w, sh; };
// (a) warp per op
__device__ __forceinline__ void warp_op(const double2* sm, const Op& op) {
  const int lane = threadIdx.x & 31;
  const int wp = 1 << op.sh, G = 32 >> op.sh;
  const int g = lane >> op.sh, c = lane & (wp - 1);
  const double2* P = sm + op.pay; const double2* in = sm + op.in;
  double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
  if (c < op.w) {
    int r = g;
    for (; r + 3 * G < op.R; r += 4 * G) {
      cfma(a0, P[r * op.w + c], in[r]); cfma(a1, P[(r + G) * op.w + c], in[r + G]);
      cfma(a2, P[(r + 2 * G) * op.w + c], in[r + 2 * G]); cfma(a3, P[(r + 3 * G) * op.w + c], in[r + 3 * G]);
    }
    if (r < op.R) cfma(a0, P[r * op.w + c], in[r]);
    if (r + G < op.R) cfma(a1, P[(r + G) * op.w + c], in[r + G]);
    if (r + 2 * G < op.R) cfma(a2, P[(r + 2 * G) * op.w + c], in[r + 2 * G]);
  }
  a0 = cadd(cadd(a0, a1), cadd(a2, a3));
  for (int m = wp; m < 32; m <<= 1) a0 = cadd(a0, shfl_xor2(a0, m));
  if (lane < op.w) ((double2*)sm)[op.out + lane] = a0;
}
// (b) slot: (op index << 16) | (column << 4) | split log2; threads t = slot * S + part
struct Slot { int pay, in, out, R, w, c; };
template <int S>
__device__ __forceinline__ void slot_exec(double2* sm, const Slot* slots, int nslot) {
  for (int t = threadIdx.x; t < nslot * S; t += 256) {
    const Slot s = slots[t / S];
    const int part = t % S;
    const double2* P = sm + s.pay + s.c;
    const double2* in = sm + s.in;
    double2 a0 = make_double2(0, 0), a1 = a0;
    int r = part;
    for (; r + S < s.R; r += 2 * S) { cfma(a0, P[r * s.w], in[r]); cfma(a1, P[(r + S) * s.w], in[r + S]); }
    if (r < s.R) cfma(a0, P[r * s.w], in[r]);
    a0 = cadd(a0, a1);
#pragma unroll
    for (int m = 1; m < S; m <<= 1) a0 = cadd(a0, shfl_xor2(a0, m));
    if (part == 0) sm[s.out + s.c] = a0;
  }
}
template <int S, int RMAX>
__device__ __forceinline__ void slot_exec_unrolled(double2* sm, const Slot* slots, int nslot) {
  for (int t = threadIdx.x; t < nslot * S; t += 256) {
    const Slot s = slots[t / S];
    const int part = t % S;
    const double2* P = sm + s.pay + s.c;
    const double2* in = sm + s.in;
    constexpr int NR = RMAX / S;
    double2 pv[NR], iv[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int r = part + j * S;
      if (r < s.R) { pv[j] = P[r * s.w]; iv[j] = in[r]; } else { pv[j] = make_double2(0, 0); iv[j] = pv[j]; }
    }
    double2 a[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
#pragma unroll
    for (int j = 0; j < NR; ++j) cfma(a[j & 3], pv[j], iv[j]);
    double2 a0 = cadd(cadd(a[0], a[1]), cadd(a[2], a[3]));
#pragma unroll
    for (int m = 1; m < S; m <<= 1) a0 = cadd(a0, shfl_xor2(a0, m));
    if (part == 0) sm[s.out + s.c] = a0;
  }
}
template <int MODE, int S>
__global__ void k(const Op* gops, int nops, const Slot* gslots, int nslot, int reps, long long* cyc, double* sink) {
  extern __shared__ double2 sm[];
  __shared__ Op ops[256];
  __shared__ Slot slots[1024];
  for (int i = threadIdx.x; i < nops; i += 256) ops[i] = gops[i];
  for (int i = threadIdx.x; i < nslot; i += 256) slots[i] = gslots[i];
  for (int i = threadIdx.x; i < 10000; i += 256) sm[i] = make_double2(1e-3 * i, 1.0);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (MODE == 0) {
      for (int i = threadIdx.x >> 5; i < nops; i += 8) warp_op(sm, ops[i]);
    } else if (MODE == 1) {
      slot_exec<S>(sm, slots, nslot);
    } else if (MODE == 2) {
      slot_exec_unrolled<S, 32>(sm, slots, nslot);
    } else {
      slot_exec_unrolled<S, 64>(sm, slots, nslot);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  if (sm[threadIdx.x].x == 12345.0) sink[0] = 1;
}
int main() {
  struct Case { const char* name; int nops, R, w; };
  Case cases[] = {{"up leaf V^T: 16 x (R=32,w=6)", 16, 32, 6}, {"up T^T: 8 x (R=16,w=8)", 8, 16, 8},
                  {"up T^T: 2 x (R=16,w=8)", 2, 16, 8}, {"down leaf V: 16 x (R=6,w=32)", 16, 6, 32},
                  {"couple: 64 x (R=40,w=8)", 64, 40, 8}, {"couple: 32 x (R=40,w=8)", 32, 40, 8},
                  {"cfg1 leaf: 16 x (R=32,w=20)", 16, 32, 20}};
  long long* cyc; double* sink; cudaMalloc(&cyc, 8 * 8); cudaMalloc(&sink, 8);
  for (auto& cs : cases) {
    std::vector<Op> ops; std::vector<Slot> slots;
    int off = 0, sh = 0; while ((1 << sh) < cs.w && sh < 5) ++sh;
    for (int i = 0; i < cs.nops; ++i) {
      Op o{off, off + cs.R * cs.w, off + cs.R * cs.w + cs.R, cs.R, cs.w, sh};
      off += cs.R * cs.w + cs.R + cs.w;
      ops.push_back(o);
      for (int c = 0; c < cs.w; ++c) slots.push_back({o.pay, o.in, o.out, o.R, o.w, c});
    }
    if (off > 10000 || slots.size() > 1024) { printf("%s: too big\n", cs.name); continue; }
    Op* dops; Slot* dsl; cudaMalloc(&dops, sizeof(Op) * ops.size()); cudaMalloc(&dsl, sizeof(Slot) * slots.size());
    cudaMemcpy(dops, ops.data(), sizeof(Op) * ops.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsl, slots.data(), sizeof(Slot) * slots.size(), cudaMemcpyHostToDevice);
    long long h[9];
    auto run = [&](auto kern, int idx) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      kern<<<1, 256, 10000 * 16>>>(dops, (int)ops.size(), dsl, (int)slots.size(), 200, cyc, sink);
      cudaMemcpy(&h[idx], cyc, 8, cudaMemcpyDeviceToHost);
    };
    run(k<0, 1>, 0); run(k<1, 1>, 1); run(k<1, 2>, 2); run(k<1, 4>, 3); run(k<1, 8>, 4);
    run(k<2, 1>, 5); run(k<2, 2>, 6); run(k<2, 4>, 7); run(k<3, 1>, 8);
    printf("%-32s warp/op %5lld | slot S=1 %5lld S=2 %5lld S=4 %5lld S=8 %5lld | unrolled32 S=1 %5lld S=2 %5lld S=4 %5lld | unr64 S=1 %5lld\n", cs.name,
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
