// FP64 tensor-pipe (DMMA, mma.sync m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 f64) vs DFMA throughput
// on the whole chip, in FLOP/s, timed with CUDA events.  Decides the multi-RHS
// (q = 64) path of the H² matvec: dense complex contractions on DMMA or DFMA.
#include <cstdio>

template <int SHAPE>
__global__ void dmma_loop(int n, double* out) {
  double acc[8][4];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 2; ++i) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (SHAPE == 0) {  // m8n8k4: 2*8*8*4 = 512 flop per warp-instruction
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k4: 1024 flop
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {  // m16n8k8: 2048 flop
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(int n, double* out) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4000;
  for (int threads : {128, 256, 512}) {
    const int blocks = 148 * 4;
    float ms;
    const double warps = blocks * (threads / 32.0);
    dfma_loop<<<blocks, threads>>>(10, out);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA   %4d thr x %d blk: %.2f TFLOP/s\n", threads, blocks,
           2.0 * 8 * n * blocks * threads / (ms * 1e-3) / 1e12);
    const double fl[3] = {512, 1024, 2048};
    const char* nm[3] = {"m8n8k4", "m16n8k4", "m16n8k8"};
    for (int s = 0; s < 3; ++s) {
      if (s == 0) dmma_loop<0><<<blocks, threads>>>(10, out);
      if (s == 1) dmma_loop<1><<<blocks, threads>>>(10, out);
      if (s == 2) dmma_loop<2><<<blocks, threads>>>(10, out);
      cudaEventRecord(e0);
      if (s == 0) dmma_loop<0><<<blocks, threads>>>(n, out);
      if (s == 1) dmma_loop<1><<<blocks, threads>>>(n, out);
      if (s == 2) dmma_loop<2><<<blocks, threads>>>(n, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("DMMA %-8s %4d thr x %d blk: %.2f TFLOP/s\n", nm[s], threads, blocks,
             fl[s] * 8 * n * warps / (ms * 1e-3) / 1e12);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
