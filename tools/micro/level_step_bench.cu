// Warm cost of one level step of the subtree programs (h2b_tree.cu): a bottom subtree of 16
// leaves (32 x 6) and 15 internal nodes (12 x 6 transfers) in shared memory, the upward-pass loop
// exactly as k_far_tree runs it, repeated; cycles per level from clock64.
// nvcc -O3 -std=c++17 -arch=sm_100a level_step_bench.cu
#include <cstdio>
#include "../../paper_1703_01175_b200/csrc/h2b_tree.cu"
void h2b_set_error(const std::string&) {}

__global__ void __launch_bounds__(256, 1) k_lvl(int reps, long long* out, int variant) {
  extern __shared__ __align__(16) double2 sm2[];
  constexpr int NN = 31;
  TNode* nodes = reinterpret_cast<TNode*>(sm2);
  double2* x = sm2 + 4 * NN;           // 512 points
  double2* V = x + 512;                 // 16 x 32 x 6
  double2* T = V + 16 * 32 * 6;         // 15 x 12 x 6
  double2* XH = T + 15 * 12 * 6;        // 31 x 6
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 512 + 16 * 32 * 6 + 15 * 12 * 6; i += 256) x[i] = make_double2(1e-3 * (i % 97), 1.0);
  if (tid < NN) {
    TNode n{};
    n.k = 6;
    n.sh = 3;
    // node order: level 0 (1), 1 (2), 2 (4), 3 (8), 4 (16 leaves)
    int lvl = tid == 0 ? 0 : tid < 3 ? 1 : tid < 7 ? 2 : tid < 15 ? 3 : 4;
    int first = (1 << lvl) - 1, ord = tid - first;
    n.xh = (int)(XH - sm2) + 6 * tid;
    if (lvl == 4) {
      n.kind = 0; n.R = 32; n.pay = (int)(V - sm2) + ord * 192; n.in = (int)(x - sm2) + 32 * ord;
    } else {
      n.kind = 1; n.R = 12; n.pay = (int)(T - sm2) + tid * 72;
      const int lo = (1 << (lvl + 1)) - 1 + 2 * ord;
      n.in = (int)(XH - sm2) + 6 * lo;
    }
    nodes[tid] = n;
  }
  __syncthreads();
  const int lev_first[6] = {0, 1, 3, 7, 15, 31};
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    for (int lv = 4; lv >= 0; --lv) {
      const int a = lev_first[lv], b = lev_first[lv + 1];
      for (int i = a + warp; i < b; i += 8) {
        const TNode nd = nodes[i];
        if (variant == 1) {  // no math: record load only
          if ((tid & 31) == 0) sm2[nd.xh] = make_double2(nd.R, 0);
        } else if (nd.kind != 2 && nd.k > 0) {
          colsum(sm2 + nd.pay, nd.R, nd.k, nd.sh, sm2 + nd.in, sm2 + nd.xh);
        }
      }
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / reps;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  const int smem = 16 * (4 * 31 + 512 + 16 * 192 + 15 * 72 + 31 * 6);
  cudaFuncSetAttribute(k_lvl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v : {0, 1}) {
    k_lvl<<<1, 256, smem>>>(100, d, v);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %lld cycles per 5-level up pass (%.2f us at 1.965 GHz)\n", v ? "record loads only" : "full up pass",
           h, h / 1965.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
