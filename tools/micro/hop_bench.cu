// Inter-SM hand-off latency on B200: a chain of H hops, hop h run by CTA (h * 37) % G, each
// waiting for flag[h-1] and publishing flag[h] (optionally with a 1 KB payload written before
// the release and read after the acquire).  Variants of the poll / publish idiom:
//   0: ld.acquire.gpu poll + nanosleep(64); bar.sync; st.release.gpu        (k_mega today)
//   1: ld.acquire.gpu poll, no sleep;     bar.sync; st.release.gpu
//   2: ld.relaxed.gpu poll, then fence.acq_rel.gpu; bar.sync; fence.acq_rel.gpu + st.relaxed
//   3: ld.relaxed.gpu poll + fence;       bar.sync; red.release.gpu.add
//   4: as 1, plus fence.proxy.async.global after the acquire and fence.proxy.async.shared::cta
//      + bar.sync before the release (k_mega's task frame)
//   5: as 1, the poll done by every thread of warp 0 on the same flag (no bar.sync skew)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hop_bench hop_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V, bool PAYLOAD>
__global__ void k_hops(uint32_t* flags, double2* pay, int H, uint32_t epoch, double* sink) {
  const int G = gridDim.x;
  double acc = 0.0;
  for (int h = 0; h < H; ++h) {
    if ((h * 37) % G != (int)blockIdx.x) continue;
    if (h > 0) {
      if (V == 5) {
        if (threadIdx.x < 32)
          while (ld_acq(flags + h - 1) != epoch) {
          }
      } else if (threadIdx.x == 0) {
        if (V == 0) {
          while (ld_acq(flags + h - 1) != epoch) __nanosleep(64);
        } else if (V == 1 || V == 4) {
          while (ld_acq(flags + h - 1) != epoch) {
          }
        } else {
          while (ld_rlx(flags + h - 1) != epoch) {
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
      }
      __syncthreads();
      if (V == 4) asm volatile("fence.proxy.async.global;" ::: "memory");
      if (PAYLOAD && threadIdx.x < 64) {
        const double2 v = __ldcg(pay + (size_t)(h - 1) * 64 + threadIdx.x);
        acc += v.x + v.y;
      }
    }
    if (PAYLOAD && threadIdx.x < 64) pay[(size_t)h * 64 + threadIdx.x] = make_double2(acc + h, threadIdx.x);
    if (V == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 2) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_rlx(flags + h, epoch);
      } else if (V == 3) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(flags + h), "r"(1u) : "memory");
      } else {
        st_rel(flags + h, epoch);
      }
    }
  }
  if (acc == 12345.0) *sink = acc;
}

template <int V, bool P>
float run(uint32_t* flags, double2* pay, int G, int H, uint32_t& epoch, double* sink) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    if (V == 3) {
      cudaMemset(flags, 0, 4 * H);
      epoch = 1;
    } else {
      ++epoch;
    }
    cudaEventRecord(a);
    k_hops<V, P><<<G, 256>>>(flags, pay, H, V == 3 ? 1u : epoch, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return best;
}

int main() {
  const int G = 148, H = 2000;
  uint32_t* flags;
  double2* pay;
  double* sink;
  cudaMalloc(&flags, 4 * H);
  cudaMemset(flags, 0, 4 * H);
  cudaMalloc(&pay, sizeof(double2) * 64 * H);
  cudaMalloc(&sink, 8);
  uint32_t epoch = 0;
  const char* names[] = {"acquire+nanosleep64 / st.release (k_mega)", "acquire spin / st.release",
                         "relaxed spin + fence / fence + st.relaxed", "relaxed spin + fence / fence + red.add",
                         "acquire spin + proxy fences (k_mega frame)", "warp-wide acquire spin / st.release"};
#define RUN(v)                                                                                   \
  {                                                                                              \
    const float t0 = run<v, false>(flags, pay, G, H, epoch, sink);                               \
    const float t1 = run<v, true>(flags, pay, G, H, epoch, sink);                                \
    printf("variant %d %-46s %.3f us/hop   with 1 KB payload %.3f us/hop\n", v, names[v], t0 * 1e3 / H, \
           t1 * 1e3 / H);                                                                        \
  }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
  return 0;
}
