// Orchestration of one H² matvec on sm_100a (B200): y_perm = S x_perm.
//
// Restates the reference `_apply_perm` (/root/reference/pkg/src/h2vie/
// arith.py:52-104).  The near-field phase (h2b_near.cu, byte-dominant) runs
// on the caller's stream and overwrites y; the far field (h2b_far.cu) runs
// concurrently on a high-priority side stream; the last far-field launch,
// which adds the leaf back-transform into y, runs after both joined.  The
// whole sequence is captured once per (x, y, q) into a CUDA graph and
// replayed, so a matvec costs one graph launch on the host.
#include <algorithm>

#include "h2b_common.cuh"

int h2b_launch_near(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st);
int h2b_launch_span(h2b_ctx* h, const SpanLaunch& L, bool up, const double2* xp, double2* yp, int q,
                    cudaStream_t st);
int h2b_launch_coupling(h2b_ctx* h, int q, cudaStream_t st);
int h2b_launch_far_levels_head(h2b_ctx* h, const double2* xp, int q, cudaStream_t st, int* nl);
int h2b_launch_leaf_back(h2b_ctx* h, double2* yp, int q, cudaStream_t st);
int h2b_launch_mega(h2b_ctx* h, const double2* xp, double2* yp, cudaStream_t st);

namespace {

__global__ void k_gather(const int64_t* __restrict__ perm, int64_t n, const double2* __restrict__ in,
                         double2* __restrict__ out, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / q, c = e - i * q;
    out[e] = in[perm[i] * q + c];
  }
}

__global__ void k_scatter(const int64_t* __restrict__ perm, int64_t n, const double2* __restrict__ in,
                          double2* __restrict__ out, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / q, c = e - i * q;
    out[perm[i] * q + c] = in[e];
  }
}

// host <-> device through mapped pinned memory (zero copy): x read over PCIe in the original
// order (contiguous, coalesced) and written to its packed position, y written over PCIe in the
// original order; replaces a DMA node plus a gather / scatter kernel on the host path
__global__ void k_host_in(const double2* __restrict__ xh, const int64_t* __restrict__ iperm, int64_t n,
                          double2* __restrict__ out, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / q, c = e - o * q;
    out[iperm[o] * q + c] = xh[e];
  }
}

__global__ void k_host_out(const double2* __restrict__ in, const int64_t* __restrict__ iperm, int64_t n,
                           double2* __restrict__ yh, int q) {
  const int64_t tot = n * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / q, c = e - o * q;
    yh[e] = in[iperm[o] * q + c];
  }
}

__global__ void k_invert_perm(const int64_t* __restrict__ perm, int64_t n, int64_t* __restrict__ iperm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    iperm[perm[i]] = i;
}

int grid_for(int64_t tot) {
  int64_t g = (tot + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

bool use_programs(const h2b_ctx* h, int q) { return q == 1 && h->span_mode == 1; }

// far field up to the join (everything that does not write y)
int launch_far_head(h2b_ctx* h, const double2* xp, int q, cudaStream_t st, int* nl) {
  if (!use_programs(h, q)) return h2b_launch_far_levels_head(h, xp, q, st, nl);
  for (const SpanLaunch& L : h->up_prog) {
    H2B_TRY(h2b_launch_span(h, L, true, xp, nullptr, q, st));
    ++*nl;
  }
  H2B_TRY(h2b_launch_coupling(h, q, st));
  ++*nl;
  for (const SpanLaunch& L : h->down_prog_head) {
    H2B_TRY(h2b_launch_span(h, L, false, xp, nullptr, q, st));
    ++*nl;
  }
  return H2B_OK;
}

// far field after the join (adds into y)
int launch_far_tail(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl) {
  if (!use_programs(h, q)) {
    H2B_TRY(h2b_launch_leaf_back(h, yp, q, st));
    ++*nl;
    return H2B_OK;
  }
  for (const SpanLaunch& L : h->down_prog_tail) {
    H2B_TRY(h2b_launch_span(h, L, false, xp, yp, q, st));
    ++*nl;
  }
  return H2B_OK;
}

int enqueue_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl) {
  *nl = 0;
  if (q == 1 && h->mega) {  // far-field task graph || near-field stream: two concurrent launches
    H2B_TRY(h2b_launch_mega(h, xp, yp, st));
    *nl = (h->mega_grid > 0 ? 1 : 0) + (h->n_near_tasks > 0 ? 1 : 0);
    return H2B_OK;
  }
  if (q >= 2 && h->use_mrhs)  // all phases as grouped complex GEMMs on DMMA (h2b_mrhs.cu)
    return h2b_launch_mrhs(h, xp, yp, q, st, nl);
  if (h->K == 0) {
    H2B_TRY(h2b_launch_near(h, xp, yp, q, st));
    ++*nl;
    return H2B_OK;
  }
  H2B_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
  H2B_CUDA_TRY(cudaStreamWaitEvent(h->far_stream, h->ev_fork, 0));
  H2B_TRY(h2b_launch_near(h, xp, yp, q, st));
  ++*nl;
  H2B_TRY(launch_far_head(h, xp, q, h->far_stream, nl));
  H2B_CUDA_TRY(cudaEventRecord(h->ev_join, h->far_stream));
  H2B_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
  H2B_TRY(launch_far_tail(h, xp, yp, q, st, nl));
  return H2B_OK;
}

}  // namespace

int h2b_launch_gather(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                      cudaStream_t st) {
  k_gather<<<grid_for(n * q), 256, 0, st>>>(perm, n, in, out, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_scatter(const int64_t* perm, int64_t n, const double2* in, double2* out, int q,
                       cudaStream_t st) {
  k_scatter<<<grid_for(n * q), 256, 0, st>>>(perm, n, in, out, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_host_in(const double2* xh, const int64_t* iperm, int64_t n, double2* out, int q, cudaStream_t st) {
  k_host_in<<<grid_for(n * q), 256, 0, st>>>(xh, iperm, n, out, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_launch_host_out(const double2* in, const int64_t* iperm, int64_t n, double2* yh, int q, cudaStream_t st) {
  k_host_out<<<grid_for(n * q), 256, 0, st>>>(in, iperm, n, yh, q);
  H2B_CHECK_LAUNCH();
  return H2B_OK;
}

int h2b_ensure_iperm(h2b_ctx* h) {
  if (h->iperm) return H2B_OK;
  H2B_CUDA_TRY(cudaMalloc(&h->iperm, sizeof(int64_t) * std::max<int64_t>(h->n, 1)));
  k_invert_perm<<<grid_for(h->n), 256>>>(h->perm, h->n, h->iperm);
  H2B_CHECK_LAUNCH();
  H2B_CUDA_TRY(cudaDeviceSynchronize());
  h->device_bytes += sizeof(int64_t) * h->n;
  return H2B_OK;
}

void h2b_release_graphs(h2b_ctx* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  for (auto& kv : h->gmres_graphs) cudaGraphExecDestroy(kv.second);
  h->gmres_graphs.clear();
}

int h2b_enqueue_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st, int* nl) {
  return enqueue_matvec(h, xp, yp, q, st, nl);
}

int h2b_ensure_workspace(h2b_ctx* h, int q) {
  if (q <= h->ws_q) return H2B_OK;
  h2b_release_graphs(h);  // captured graphs hold the old workspace pointers
  if (h->xhat) cudaFree(h->xhat);
  if (h->yhat) cudaFree(h->yhat);
  h->xhat = h->yhat = nullptr;
  h->device_bytes -= 2 * 16 * std::max<int64_t>(h->K, 1) * h->ws_q;
  h->ws_q = 0;
  const size_t bytes = (size_t)16 * std::max<int64_t>(h->K, 1) * q;
  H2B_CUDA_TRY(cudaMalloc(&h->xhat, bytes));
  H2B_CUDA_TRY(cudaMalloc(&h->yhat, bytes));
  h->ws_q = q;
  h->device_bytes += 2 * 16 * std::max<int64_t>(h->K, 1) * q;
  return H2B_OK;
}

int h2b_order_begin(h2b_ctx* h, cudaStream_t st) {
  if (!h->ev_done) H2B_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming));
  H2B_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_done, 0));  // never recorded yet: a no-op
  return H2B_OK;
}

int h2b_order_end(h2b_ctx* h, cudaStream_t st) {
  H2B_CUDA_TRY(cudaEventRecord(h->ev_done, st));
  return H2B_OK;
}

namespace {
int run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st);
}

// one matvec on `st`, ordered after the handle's previous work on any stream (the graphs of one
// handle share its x̂/ŷ workspace and control flags, so two matvecs must not overlap on the device)
int h2b_run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st) {
  H2B_TRY(h2b_order_begin(h, st));
  H2B_TRY(run_matvec(h, xp, yp, q, st));
  return h2b_order_end(h, st);
}

namespace {
int run_matvec(h2b_ctx* h, const double2* xp, double2* yp, int q, cudaStream_t st) {
  H2B_TRY(h2b_prepare(h));
  H2B_TRY(h2b_ensure_workspace(h, q));
  if (q >= 2 && h->use_mrhs) H2B_TRY(h2b_mrhs_workspace(h, q));  // allocates: never inside a capture
  int nl = 0;
  if (!h->use_graphs) {
    H2B_TRY(enqueue_matvec(h, xp, yp, q, st, &nl));
    if (q == 1) h->launches_q1 = nl;
    return H2B_OK;
  }
  const GraphKey key{xp, yp, q};
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    if (h->graphs.size() >= 64) h2b_release_graphs(h);
    cudaStream_t cs = nullptr;
    H2B_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    H2B_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_matvec(h, xp, yp, q, cs, &nl);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) {
      h2b_set_error(std::string("graph capture: ") + cudaGetErrorString(e));
      return H2B_ECUDA;
    }
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      h2b_set_error(std::string("graph instantiate: ") + cudaGetErrorString(e));
      return H2B_ECUDA;
    }
    if (q == 1) h->launches_q1 = nl;
    it = h->graphs.emplace(key, ex).first;
  }
  H2B_CUDA_TRY(cudaGraphLaunch(it->second, st));
  return H2B_OK;
}
}  // namespace

// phase 0: near-field only (y overwritten); phase 1: far field only (y accumulated);
// both serialised on `st` so they can be timed one by one.
int h2b_run_phase(h2b_ctx* h, int phase, const double2* xp, double2* yp, int q, cudaStream_t st) {
  H2B_TRY(h2b_prepare(h));
  H2B_TRY(h2b_ensure_workspace(h, q));
  int nl = 0;
  if (phase == 0) return h2b_launch_near(h, xp, yp, q, st);
  if (h->K == 0) return H2B_OK;
  H2B_TRY(launch_far_head(h, xp, q, st, &nl));
  return launch_far_tail(h, xp, yp, q, st, &nl);
}
