// HBM streaming micro-benchmark on B200: TMA bulk-copy rings vs LDG.256 loads.
// Each CTA streams a private contiguous slab; aggregate GB/s from CUDA events.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(b)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void arm(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su(b)), "r"(ph) : "memory");
}
// TMA ring: nst stages of chunk bytes; thread 0 issues, all threads wait + touch 1 value
__global__ void k_tma(const char* src, size_t per_cta, int chunk, int nst, double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) for (int i = 0; i < nst; ++i) bar_init(&bars[i]);
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  if (threadIdx.x == 0) for (int i = 0; i < nst && i < n; ++i) { arm(&bars[i], chunk); bulk(sm + i * chunk, base + (size_t)i * chunk, chunk, &bars[i]); }
  uint32_t ph = 0; double acc = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % nst;
    wait(&bars[s], (ph >> s) & 1); ph ^= 1u << s;
    acc += ((const double*)(sm + s * chunk))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && i + nst < n) { arm(&bars[s], chunk); bulk(sm + s * chunk, base + (size_t)(i + nst) * chunk, chunk, &bars[s]); }
  }
  if (acc == 12345.0) sink[0] = acc;
}
// ring variant closer to the near-field task: second small copy per stage and/or L2 hint
template <bool XCOPY, bool HINT>
__global__ void k_tma2(const char* src, const char* xsrc, size_t per_cta, int chunk, int nst, double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) for (int i = 0; i < nst; ++i) bar_init(&bars[i]);
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  const int stg = chunk + (XCOPY ? 512 : 0);
  auto issue = [&](int i, int s) {
    arm(&bars[s], stg);
    if (HINT)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su(sm + s * stg)), "l"(base + (size_t)i * chunk), "r"(chunk), "r"(su(&bars[s])), "l"(pol) : "memory");
    else
      bulk(sm + s * stg, base + (size_t)i * chunk, chunk, &bars[s]);
    if (XCOPY) bulk(sm + s * stg + chunk, xsrc + (size_t)((i * 7919) % 1024) * 512, 512, &bars[s]);
  };
  if (threadIdx.x == 0) for (int i = 0; i < nst && i < n; ++i) issue(i, i);
  uint32_t ph = 0; double acc = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % nst;
    wait(&bars[s], (ph >> s) & 1); ph ^= 1u << s;
    acc += ((const double*)(sm + s * stg))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && i + nst < n) issue(i + nst, s);
  }
  if (acc == 12345.0) sink[0] = acc;
}
// LDG.256 streaming: UNR loads in flight per thread
template <int UNR>
__global__ void k_ldg(const double* src, size_t per_cta, double* sink) {
  const double* base = src + (size_t)blockIdx.x * (per_cta / 8);
  const size_t n4 = per_cta / 32;  // 32-byte chunks
  double acc = 0;
  for (size_t i0 = threadIdx.x; i0 < n4; i0 += (size_t)blockDim.x * UNR) {
    double v[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const size_t i = i0 + (size_t)u * blockDim.x;
      if (i < n4) asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3]) : "l"(base + 4 * i));
      else v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u][0] + v[u][1] + v[u][2] + v[u][3];
  }
  if (acc == 12345.0) sink[0] = acc;
}
int main(int argc, char** argv) {
  const size_t total = argc > 1 ? (size_t)atol(argv[1]) << 20 : (size_t)1 << 30;  // MiB streamed per run
  char* src; double* sink;
  cudaMalloc(&src, total); cudaMemset(src, 0, total); cudaMalloc(&sink, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  char* flush; cudaMalloc(&flush, 256 << 20);
  char* clean; cudaMalloc(&clean, 256 << 20); cudaMemset(clean, 0, 256 << 20);
  const bool clean_flush = getenv("CLEAN_FLUSH") != nullptr;
  auto run = [&](auto launch, const char* name) {
    launch(); cudaDeviceSynchronize();
    float tot = 0;
    for (int r = 0; r < 5; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);  // cold L2 for every rep
      if (clean_flush) k_ldg<4><<<148 * 8, 256>>>((const double*)clean, (size_t)(256 << 20) / (148 * 8) / 32 * 32, sink);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
    }
    printf("%-44s %7.0f GB/s  (%.1f us per rep)\n", name, 5.0 * total / (tot * 1e-3) / 1e9, tot / 5 * 1e3);
  };
  char nm[128];
  for (int ctas_per_sm : {1, 2}) for (int chunk : {16384, 32768, 65536}) for (int nst : {2, 4, 6, 12}) {
    const int grid = 148 * ctas_per_sm;
    const size_t per = total / grid / chunk * chunk;
    if ((size_t)nst * chunk * ctas_per_sm > 220 * 1024) continue;
    snprintf(nm, sizeof nm, "TMA %d CTA/SM chunk %5d stages %d", ctas_per_sm, chunk, nst);
    run([&] { k_tma<<<grid, 256, nst * chunk>>>(src, per, chunk, nst, sink); }, nm);
  }
  cudaFuncSetAttribute(k_tma2<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_tma2<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_tma2<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  {
    const int grid = 296, chunk = 16384, nst = 5;
    const size_t per = total / grid / chunk * chunk;
    run([&] { k_tma2<true, true><<<grid, 256, nst * (chunk + 512)>>>(src, src, per, chunk, nst, sink); }, "ring 16K+512 x-copy + evict_first hint");
    run([&] { k_tma2<true, false><<<grid, 256, nst * (chunk + 512)>>>(src, src, per, chunk, nst, sink); }, "ring 16K+512 x-copy, no hint");
    run([&] { k_tma2<false, true><<<grid, 256, nst * chunk>>>(src, src, per, chunk, nst, sink); }, "ring 16K, evict_first hint");
  }
  for (int ctas_per_sm : {2, 4, 8}) {
    const int grid = 148 * ctas_per_sm;
    const size_t per = total / grid / 32 * 32;
    snprintf(nm, sizeof nm, "LDG.256 UNR4 %d CTA/SM x 256 thr", ctas_per_sm);
    run([&] { k_ldg<4><<<grid, 256>>>((const double*)src, per, sink); }, nm);
    snprintf(nm, sizeof nm, "LDG.256 UNR8 %d CTA/SM x 256 thr", ctas_per_sm);
    run([&] { k_ldg<8><<<grid, 256>>>((const double*)src, per, sink); }, nm);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
