// extern "C" surface of libh2b.so (declared in include/h2b.h).
#include <stdio.h>
#include <immintrin.h>
#include <vector>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <time.h>
#include <string.h>

#include <algorithm>
#include <iterator>
#include <string>

#include "h2b_common.cuh"

static thread_local std::string g_last_error;

void h2b_set_error(const std::string& msg) { g_last_error = msg; }

#define REQUIRE(cond, code, msg) \
  do {                           \
    if (!(cond)) {               \
      h2b_set_error(msg);        \
      return code;               \
    }                            \
  } while (0)

namespace {

template <typename T>
int upload_table(T** dst, const T* src, int64_t count, int64_t* acc) {
  const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
  H2B_CUDA_TRY(cudaMalloc((void**)dst, bytes));
  if (count > 0) H2B_CUDA_TRY(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  *acc += (int64_t)bytes;
  return H2B_OK;
}

}  // namespace
void h2b_tree_free(TreeDev* d);
int h2b_tree_error(const TreeDev* d, uint32_t* err);
namespace {

void free_ctx(h2b_ctx* h) {
  h2b_release_graphs(h);
  h2b_tree_free(h->tree);
  h->tree = nullptr;
  h2b_mrhs_free(h);
  void* ptrs[] = {h->c_start_d, h->c_size_d, h->c_rank_d, h->c_lo,      h->c_hi,
                  h->c_parent,  h->c_xoff_d, h->c_voff_d, h->c_toff_d,  h->s_row_ptr_d,
                  h->s_off_d,   h->d_row_ptr_d, h->d_off_d, h->s_col_d, h->d_col_d,
                  h->perm,      h->leaves,   h->xhat,     h->yhat,      h->kry,
                  h->buf[0],    h->buf[1],   h->buf[2],   h->buf[3],    h->hxp,
                  h->hyp,       h->vT,       h->tT,       h->s_prow,    h->s_xcol,
                  h->couple_targets, h->span_heads, h->span_copies, h->span_outs,
                  h->span_ops, h->near_items, h->near_blks, h->couple_items, h->tasks, h->deps,
                  h->near_tasks, h->leaf_items, h->couple_groups, h->ctrl, h->flags, h->trace,
                  h->rec_pool, h->l2_prefetch, h->cta_lists, h->task_list, h->near_recs, h->near_idx, h->wbuf, h->ydeep,
                  h->ks_partial, h->ks_vals, h->near_trace, h->iperm};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->far_stream) cudaStreamDestroy(h->far_stream);
  if (h->host_stream) cudaStreamDestroy(h->host_stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  if (h->ks_host) cudaFreeHost(h->ks_host);
  if (h->hpin) cudaFreeHost(h->hpin);
  delete h;
}

int ready(h2b_ctx* h) {
  REQUIRE(h, H2B_EINVAL, "null handle");
  for (int s = 0; s < 4; ++s)
    REQUIRE(h->sec_uploaded[s] >= h->sec_elems[s], H2B_ESTATE,
            "payload section " + std::to_string(s) + " not fully uploaded");
  return H2B_OK;
}

}  // namespace

extern "C" {

int h2b_version(void) { return 1; }

const char* h2b_last_error(void) { return g_last_error.c_str(); }

int h2b_device_ok(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 ? 1 : 0;
}

int h2b_create(const h2b_layout* L, int device, h2b_handle* out) {
  REQUIRE(L && out, H2B_EINVAL, "h2b_create: null argument");
  *out = nullptr;
  REQUIRE(h2b_device_ok(device), H2B_ENODEV,
          "h2b_create: no compute-capability 10.x (B200/sm_100a) device " + std::to_string(device) +
              " — the H2 hot path has no CPU fallback");
  REQUIRE(L->n > 0 && L->depth > 0 && L->num_clusters > 0, H2B_EINVAL, "h2b_create: empty operator");
  REQUIRE(L->n_coupling >= 0 && L->n_near > 0, H2B_EINVAL, "h2b_create: bad block counts");
  H2B_CUDA_TRY(cudaSetDevice(device));
  h2b_ctx* h = new h2b_ctx();
  h->device = device;
  h->n = L->n;
  h->depth = L->depth;
  h->P = L->num_clusters;
  h->K = L->c_xhat_off[L->num_clusters];
  h->n_coupling = L->n_coupling;
  h->n_near = L->n_near;
  h->sec_elems[0] = L->v_elems;
  h->sec_elems[1] = L->t_elems;
  h->sec_elems[2] = L->s_elems;
  h->sec_elems[3] = L->d_elems;
  const int P = h->P;
  h->level_ptr.assign(L->level_ptr, L->level_ptr + h->depth + 1);
  h->c_rank.assign(L->c_rank, L->c_rank + P);
  h->c_child_lo.assign(L->c_child_lo, L->c_child_lo + P);
  h->c_size.assign(L->c_size, L->c_size + P);
  h->c_child_hi.assign(L->c_child_hi, L->c_child_hi + P);
  h->c_start.assign(L->c_start, L->c_start + P);
  h->c_xoff.assign(L->c_xhat_off, L->c_xhat_off + P + 1);
  h->c_voff.assign(L->c_v_off, L->c_v_off + P);
  h->c_toff.assign(L->c_t_off, L->c_t_off + P);
  h->s_row_ptr.assign(L->s_row_ptr, L->s_row_ptr + P + 1);
  h->s_off.assign(L->s_off, L->s_off + L->n_coupling);
  h->s_col.assign(L->s_col, L->s_col + L->n_coupling);
  h->d_row_ptr.assign(L->d_row_ptr, L->d_row_ptr + P + 1);
  h->d_off.assign(L->d_off, L->d_off + L->n_near);
  h->d_col.assign(L->d_col, L->d_col + L->n_near);
  if (h->level_ptr[0] != 0 || h->level_ptr[h->depth] != P) {
    delete h;
    h2b_set_error("h2b_create: level_ptr does not cover the clusters");
    return H2B_EINVAL;
  }
  // leaves, schedule
  int uni = -1;
  for (int p = 0; p < P; ++p)
    if (h->c_child_lo[p] < 0) {
      h->h_leaves.push_back(p);
      const int sz = h->c_size[p];
      uni = (uni == -1 || uni == sz) ? sz : 0;
    }
  h->uniform_leaf = uni > 0 ? uni : 0;
  h->n_leaves = (int)h->h_leaves.size();
  for (int l = h->depth - 1; l >= 0; --l) {
    bool any = false;
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) any |= h->c_rank[p] > 0;
    if (any) h->up_levels.push_back(l);
  }
  for (int l = 0; l < h->depth; ++l) {
    bool any = false;
    for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p)
      any |= (h->c_rank[p] > 0 && h->c_child_lo[p] >= 0);
    if (any) h->down_levels.push_back(l);
  }
  // near-field fast path needs every near block to be uniform (n x n), which holds when all
  // leaves share one size; it also needs 32-byte alignment, guaranteed for even sizes.
  int64_t acc = 0;
  int rc = H2B_OK;
#define UP(dst, src, cnt) \
  if (!rc) rc = upload_table(&h->dst, src, cnt, &acc)
  UP(c_start_d, L->c_start, P);
  UP(c_size_d, L->c_size, P);
  UP(c_rank_d, L->c_rank, P);
  UP(c_lo, L->c_child_lo, P);
  UP(c_hi, L->c_child_hi, P);
  UP(c_parent, L->c_parent, P);
  UP(c_xoff_d, L->c_xhat_off, P + 1);
  UP(c_voff_d, L->c_v_off, P);
  UP(c_toff_d, L->c_t_off, P);
  UP(s_row_ptr_d, L->s_row_ptr, P + 1);
  UP(s_col_d, L->s_col, L->n_coupling);
  UP(s_off_d, L->s_off, L->n_coupling);
  UP(d_row_ptr_d, L->d_row_ptr, P + 1);
  UP(d_col_d, L->d_col, L->n_near);
  UP(d_off_d, L->d_off, L->n_near);
  UP(perm, L->perm, L->n);
  UP(leaves, h->h_leaves.data(), (int64_t)h->h_leaves.size());
#undef UP
  for (int s = 0; s < 4 && !rc; ++s) {
    const size_t bytes = 16 * (size_t)std::max<int64_t>(h->sec_elems[s], 2);
    cudaError_t e = cudaMalloc(&h->buf[s], bytes);
    if (e != cudaSuccess) {
      h2b_set_error(std::string("h2b_create: payload allocation: ") + cudaGetErrorString(e));
      rc = e == cudaErrorMemoryAllocation ? H2B_ENOMEM : H2B_ECUDA;
    }
    acc += bytes;
  }
  if (rc) {
    free_ctx(h);
    return rc;
  }
  h->device_bytes = acc;
  *out = h;
  return H2B_OK;
}

int h2b_upload(h2b_handle h, int sec, const void* src, size_t bytes, size_t offset) {
  REQUIRE(h, H2B_EINVAL, "null handle");
  REQUIRE(!h->prepared, H2B_ESTATE, "h2b_upload: payload is immutable after the first matvec");
  REQUIRE(sec >= 0 && sec < 4, H2B_EINVAL, "h2b_upload: bad section");
  REQUIRE(bytes % 16 == 0 && offset % 16 == 0, H2B_EINVAL, "h2b_upload: unaligned size/offset");
  REQUIRE((int64_t)((offset + bytes) / 16) <= h->sec_elems[sec], H2B_EINVAL,
          "h2b_upload: beyond section end");
  if (bytes == 0) return H2B_OK;
  REQUIRE(src, H2B_EINVAL, "h2b_upload: null source");
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  // host or device source (unified addressing): device-side fills need no host staging
  H2B_CUDA_TRY(cudaMemcpy((char*)h->buf[sec] + offset, src, bytes, cudaMemcpyDefault));
  // record the chunk as a range and merge it with the ones it touches: ready() passes only
  // when the merged ranges cover the whole section (any chunk order, overlaps allowed)
  int64_t b = (int64_t)(offset / 16), e = (int64_t)((offset + bytes) / 16);
  auto& iv = h->sec_iv[sec];
  auto it = iv.upper_bound(b);
  if (it != iv.begin() && std::prev(it)->second >= b) --it;
  while (it != iv.end() && it->first <= e) {
    b = std::min(b, it->first);
    e = std::max(e, it->second);
    it = iv.erase(it);
  }
  iv.emplace(b, e);
  int64_t covered = 0;
  for (const auto& kv : iv) covered += kv.second - kv.first;
  h->sec_uploaded[sec] = covered;
  return H2B_OK;
}

int h2b_destroy(h2b_handle h) {
  if (!h) return H2B_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  free_ctx(h);
  return H2B_OK;
}

int64_t h2b_device_bytes(h2b_handle h) { return h ? h->device_bytes : -1; }

int h2b_matvec_perm(h2b_handle h, const void* x_perm, void* y_perm, int q, void* stream) {
  int rc = ready(h);
  if (rc) return rc;
  REQUIRE(q >= 1, H2B_EINVAL, "h2b_matvec_perm: q must be >= 1");
  REQUIRE(x_perm && y_perm && x_perm != y_perm, H2B_EINVAL,
          "h2b_matvec_perm: null or aliased buffers");
  return h2b_run_matvec(h, (const double2*)x_perm, (double2*)y_perm, q, (cudaStream_t)stream);
}

namespace {
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
}  // namespace


// ---------------------------------------------------------------------------
// parallel host copy for the pageable staging of h2b_matvec_host: one memcpy of a MiB runs at
// ~17-20 GB/s on one core; a few persistent workers split it.  Workers spin briefly after a job
// (tight solver loops keep them hot) and then sleep on a condition variable.
// ---------------------------------------------------------------------------
namespace {
struct CopyPool {
  int nw = 0;
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<uint64_t> gen{0};
  std::atomic<int> done{0};
  char* dst = nullptr;
  const char* src = nullptr;
  size_t bytes = 0;
  int parts = 1;

  void part(int i) {
    const size_t per = (bytes / parts + 63) & ~size_t(63);
    const size_t b = std::min(bytes, per * i), e = std::min(bytes, b + per);
    if (e > b) memcpy(dst + b, src + b, e - b);
  }
  void worker(int w) {
    uint64_t seen = 0;
    for (;;) {
      uint64_t g = gen.load(std::memory_order_acquire);
      const double t0 = wall_us();
      while (g == seen && wall_us() - t0 < 300.0) {
        _mm_pause();
        g = gen.load(std::memory_order_acquire);
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return gen.load(std::memory_order_acquire) != seen; });
        g = gen.load(std::memory_order_acquire);
      }
      seen = g;
      part(w + 1);
      done.fetch_add(1, std::memory_order_acq_rel);
    }
  }
  static double wall_us() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
  }
  std::mutex job_mu;  // one job at a time (handles used from several threads share the pool)
  void copy(void* d, const void* s_, size_t n) {
    if (nw == 0 || n < (256u << 10)) {
      memcpy(d, s_, n);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu);
    dst = (char*)d;
    src = (const char*)s_;
    bytes = n;
    parts = nw + 1;
    done.store(0, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu);
      gen.fetch_add(1, std::memory_order_acq_rel);
    }
    cv.notify_all();
    part(0);
    while (done.load(std::memory_order_acquire) < nw) _mm_pause();
  }
};

CopyPool& copy_pool() {
  static CopyPool* p = [] {
    CopyPool* c = new CopyPool();  // never destroyed: detached workers outlive static destruction
    unsigned hc = std::thread::hardware_concurrency();
    int nw = (int)std::min(5u, hc > 2 ? hc / 2 - 1 : 0u);  // 6 parts on a 16-core host: 233 -> 142 us per cfg2 call
    if (const char* e = getenv("H2B_COPY_THREADS")) nw = std::max(0, std::min(15, atoi(e) - 1));
    c->nw = nw;
    for (int w = 0; w < nw; ++w) {
      c->th.emplace_back([c, w] { c->worker(w); });
      c->th.back().detach();
    }
    return c;
  }();
  return *p;
}
}  // namespace

static double host_now_us() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

int h2b_matvec_host(h2b_handle h, const void* x, void* y, int q) {
  static const bool timing = getenv("H2B_HOST_TIMING") != nullptr;  // development aid
  double tt[6] = {host_now_us(), 0, 0, 0, 0, 0};
  int rc = ready(h);
  if (rc) return rc;
  REQUIRE(q >= 1, H2B_EINVAL, "h2b_matvec_host: q must be >= 1");
  REQUIRE(x && y, H2B_EINVAL, "h2b_matvec_host: null buffer");
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  const size_t bytes = (size_t)16 * h->n * q;
  if (h->hws_q < q) {
    h2b_release_graphs(h);  // host-path graphs hold the staging pointers
    if (h->hxp) cudaFree(h->hxp);
    if (h->hyp) cudaFree(h->hyp);
    h->hxp = h->hyp = nullptr;
    h->hws_q = 0;
    H2B_CUDA_TRY(cudaMalloc(&h->hxp, 2 * bytes));
    H2B_CUDA_TRY(cudaMalloc(&h->hyp, 2 * bytes));
    h->hws_q = q;
  }
  if (!h->host_stream) H2B_CUDA_TRY(cudaStreamCreateWithFlags(&h->host_stream, cudaStreamNonBlocking));
  double2* dx = h->hxp;                  // original order
  double2* dxp = h->hxp + h->n * q;      // permuted
  double2* dyp = h->hyp;                 // permuted
  double2* dy = h->hyp + h->n * q;       // original order
  cudaStream_t st = h->host_stream;
  H2B_TRY(h2b_order_begin(h, st));
  // pageable caller buffers (numpy arrays: the reference-facing drop-in) are staged through the
  // handle's own pinned buffers so the call still runs as one graph with one DMA per direction;
  // H2B_HOST_STAGING=driver leaves pageable copies to the CUDA driver instead (A/B timing)
  const bool x_pinned = is_pinned(x), y_pinned = is_pinned(y);
  static const bool driver_staging = [] {
    const char* e = getenv("H2B_HOST_STAGING");
    return e && !strcmp(e, "driver");
  }();
  const void* xs = x;
  void* ys = y;
  if (h->use_graphs && !driver_staging && (!x_pinned || !y_pinned)) {
    if (h->hpin_bytes < 2 * bytes) {
      h2b_release_graphs(h);  // host-path graphs hold the old staging pointers
      if (h->hpin) cudaFreeHost(h->hpin);
      h->hpin = nullptr;
      h->hpin_bytes = 0;
      H2B_CUDA_TRY(cudaMallocHost(&h->hpin, 2 * bytes));
      h->hpin_bytes = 2 * bytes;
    }
    if (!x_pinned) {
      tt[1] = host_now_us();
      copy_pool().copy(h->hpin, x, bytes);
      tt[2] = host_now_us();
      xs = h->hpin;
    }
    if (!y_pinned) ys = (char*)h->hpin + bytes;
  }
  // pinned buffers are read / written by the permutation kernels themselves over PCIe (zero
  // copy: one kernel per direction instead of a DMA node plus a gather / scatter kernel);
  // H2B_HOST_ZC=0 keeps the DMA path (A/B timing)
  static const bool zc_env = [] {
    const char* e = getenv("H2B_HOST_ZC");
    return !(e && !strcmp(e, "0"));
  }();
  void* xs_dev = nullptr;
  void* ys_dev = nullptr;
  bool zc = zc_env && is_pinned(xs) && is_pinned(ys) && cudaHostGetDevicePointer(&xs_dev, const_cast<void*>(xs), 0) == cudaSuccess &&
            cudaHostGetDevicePointer(&ys_dev, ys, 0) == cudaSuccess;
  if (!zc) cudaGetLastError();
  if (zc) H2B_TRY(h2b_ensure_iperm(h));
  auto enqueue = [&](cudaStream_t s, bool in_graph) -> int {
    int r = H2B_OK;
    if (zc) {
      r = h2b_launch_host_in((const double2*)xs_dev, h->iperm, h->n, dxp, q, s);
    } else {
      H2B_CUDA_TRY(cudaMemcpyAsync(dx, xs, bytes, cudaMemcpyHostToDevice, s));
      r = h2b_launch_gather(h->perm, h->n, dx, dxp, q, s);
    }
    if (!r) {
      int nl = 0;
      r = in_graph ? h2b_enqueue_matvec(h, dxp, dyp, q, s, &nl) : h2b_run_matvec(h, dxp, dyp, q, s);
    }
    if (r) return r;
    if (zc) return h2b_launch_host_out(dyp, h->iperm, h->n, (double2*)ys_dev, q, s);
    r = h2b_launch_scatter(h->perm, h->n, dyp, dy, q, s);
    if (r) return r;
    H2B_CUDA_TRY(cudaMemcpyAsync(ys, dy, bytes, cudaMemcpyDeviceToHost, s));
    return H2B_OK;
  };
  if (h->use_graphs && is_pinned(xs) && is_pinned(ys)) {
    // pinned host buffers: the whole call (H2D, gather, matvec, scatter, D2H) is one graph
    H2B_TRY(h2b_prepare(h));
    H2B_TRY(h2b_ensure_workspace(h, q));
    if (q >= 2 && h->use_mrhs) H2B_TRY(h2b_mrhs_workspace(h, q));
    const GraphKey key{xs, ys, -q};  // negative q: host-path graph
    auto it = h->graphs.find(key);
    if (it == h->graphs.end()) {
      cudaStream_t cs = nullptr;
      H2B_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      H2B_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      rc = enqueue(cs, true);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &g);
      cudaStreamDestroy(cs);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      REQUIRE(e == cudaSuccess, H2B_ECUDA, std::string("host-path capture: ") + cudaGetErrorString(e));
      cudaGraphExec_t ex = nullptr;
      e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      REQUIRE(e == cudaSuccess, H2B_ECUDA, std::string("host-path instantiate: ") + cudaGetErrorString(e));
      if (h->graphs.size() >= 64) h2b_release_graphs(h);
      it = h->graphs.emplace(key, ex).first;
    }
    H2B_CUDA_TRY(cudaGraphLaunch(it->second, st));
    tt[3] = host_now_us();
  } else {
    H2B_TRY(enqueue(st, false));
  }
  H2B_TRY(h2b_order_end(h, st));
  H2B_CUDA_TRY(cudaStreamSynchronize(st));
  tt[4] = host_now_us();
  if (ys != y) copy_pool().copy(y, ys, bytes);
  if (timing) {
    tt[5] = host_now_us();
    fprintf(stderr, "h2b_matvec_host us: pre %.1f copy-in %.1f launch %.1f sync %.1f copy-out %.1f\n",
            tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4]);
  }
  return H2B_OK;
}

int h2b_matvec_phase(h2b_handle h, int phase, const void* x_perm, void* y_perm, int q,
                     void* stream) {
  int rc = ready(h);
  if (rc) return rc;
  REQUIRE(q >= 1 && (phase == 0 || phase == 1), H2B_EINVAL, "h2b_matvec_phase: bad phase/q");
  REQUIRE(x_perm && y_perm && x_perm != y_perm, H2B_EINVAL, "h2b_matvec_phase: bad buffers");
  return h2b_run_phase(h, phase, (const double2*)x_perm, (double2*)y_perm, q, (cudaStream_t)stream);
}

int h2b_prepare_handle(h2b_handle h) {
  int rc = ready(h);
  if (rc) return rc;
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  return h2b_prepare(h);
}

int h2b_set_option(h2b_handle h, int option, int value) {
  REQUIRE(h, H2B_EINVAL, "null handle");
  if (option == H2B_OPT_GRAPHS) {
    h->use_graphs = value ? 1 : 0;
    h2b_release_graphs(h);
    return H2B_OK;
  }
  if (option == H2B_OPT_TRACE) {
    REQUIRE(h->prepared && h->mega, H2B_ESTATE, "h2b_set_option(H2B_OPT_TRACE): needs a prepared "
                                                "persistent-kernel handle");
    h2b_release_graphs(h);  // captured launches hold the old trace pointer
    if (h->trace) cudaFree(h->trace);
    h->trace = nullptr;
    if (value) {
      H2B_CUDA_TRY(cudaMalloc(&h->trace, sizeof(uint64_t) * 8 * std::max(h->n_tasks, 1)));
      H2B_CUDA_TRY(cudaMemset(h->trace, 0, sizeof(uint64_t) * 8 * std::max(h->n_tasks, 1)));
    }
    return H2B_OK;
  }
  if (option == H2B_OPT_DEBUG) {
    h->mega_debug = value;
    h2b_release_graphs(h);
    return H2B_OK;
  }
  if (option == H2B_OPT_MRHS) {
    h->use_mrhs = value ? 1 : 0;
    h2b_release_graphs(h);
    return H2B_OK;
  }
  if (option == H2B_OPT_TREE) {
    REQUIRE(!h->prepared, H2B_ESTATE, "h2b_set_option(H2B_OPT_TREE): set before the first matvec");
    h->use_tree = value ? 1 : 0;
    return H2B_OK;
  }
  if (option == H2B_OPT_MEGA) {
    REQUIRE(!h->prepared, H2B_ESTATE, "h2b_set_option(H2B_OPT_MEGA): set before the first matvec");
    h->use_mega = value ? 1 : 0;
    return H2B_OK;
  }
  h2b_set_error("h2b_set_option: unknown option");
  return H2B_EINVAL;
}

int h2b_query(h2b_handle h, int what, int64_t* out) {
  REQUIRE(h && out, H2B_EINVAL, "h2b_query: null argument");
  switch (what) {
    case H2B_Q_LAUNCHES_Q1: *out = h->launches_q1; return H2B_OK;
    case H2B_Q_SPAN_MODE: *out = h->span_mode; return H2B_OK;
    case H2B_Q_SPLIT_LEVEL: *out = h->ls; return H2B_OK;
    case H2B_Q_TOP_STAGED: *out = h->top_staged; return H2B_OK;
    case H2B_Q_DEVICE_BYTES: *out = h->device_bytes; return H2B_OK;
    case H2B_Q_MEGA: *out = h->mega; return H2B_OK;
    case H2B_Q_MEGA_TASKS: *out = h->n_tasks; return H2B_OK;
    case H2B_Q_MEGA_GRID: *out = h->mega_grid; return H2B_OK;
    case H2B_Q_MEGA_TIERS: *out = h->mega_tiers; return H2B_OK;
    case H2B_Q_NEAR_TASKS: *out = h->n_near_tasks; return H2B_OK;
    case H2B_Q_NEAR_STAGES: *out = h->near_nst; return H2B_OK;
    case H2B_Q_NEAR_SMEM: *out = h->near_smem; return H2B_OK;
    case H2B_Q_MEGA_SMEM: *out = h->mega_smem + 16 * h->mega_blob_slots; return H2B_OK;
    case H2B_Q_NEAR_VARIANT: *out = 100 * h->mega_ns + h->mega_r; return H2B_OK;
    case H2B_Q_MRHS_LAUNCHES: *out = h2b_mrhs_launches(h); return H2B_OK;
    case H2B_Q_DEVICE_ERROR: {
      MegaCtrl c{};
      if (h->ctrl) H2B_CUDA_TRY(cudaMemcpy(&c, h->ctrl, sizeof(c), cudaMemcpyDeviceToHost));
      uint32_t te = 0;
      if (h->tree) H2B_TRY(h2b_tree_error(h->tree, &te));
      *out = c.error | te;
      return H2B_OK;
    }
    case H2B_Q_TREE: *out = h->tree ? (int64_t)h->tree_progs | ((int64_t)h->tree_ls << 16) | ((int64_t)h->tree_lt << 24) | ((int64_t)h->tree_flat << 30) | ((int64_t)h->tree_smem << 32) : 0; return H2B_OK;
    default: break;
  }
  h2b_set_error("h2b_query: unknown key");
  return H2B_EINVAL;
}

int h2b_get_trace(h2b_handle h, int64_t* out, int64_t max_tasks) {
  REQUIRE(h && out, H2B_EINVAL, "h2b_get_trace: null argument");
  REQUIRE(h->trace, H2B_ESTATE, "h2b_get_trace: tracing is off (H2B_OPT_TRACE)");
  const int64_t n = std::min<int64_t>(max_tasks, h->n_tasks);
  std::vector<uint64_t> t(8 * (size_t)n);
  H2B_CUDA_TRY(cudaDeviceSynchronize());
  H2B_CUDA_TRY(cudaMemcpy(t.data(), h->trace, sizeof(uint64_t) * 8 * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) {
    int64_t* o = out + 10 * i;
    o[0] = h->h_tasks[i].type;
    o[1] = h->h_tasks[i].arg;
    o[2] = (int64_t)t[8 * i + 0];  // claim
    o[3] = (int64_t)t[8 * i + 1];  // ready
    o[4] = (int64_t)t[8 * i + 2];  // staged (spans)
    o[5] = (int64_t)t[8 * i + 6];  // end of level 0 (spans)
    o[6] = (int64_t)t[8 * i + 7];  // end of level 1 (spans)
    o[7] = (int64_t)t[8 * i + 5];  // compute done (spans)
    o[8] = (int64_t)t[8 * i + 3];  // done
    o[9] = (int64_t)t[8 * i + 4];  // smid | cta << 32
  }
  return H2B_OK;
}

int h2b_gather_perm(h2b_handle h, const void* in, void* out, int q, void* stream) {
  REQUIRE(h && in && out && q >= 1, H2B_EINVAL, "h2b_gather_perm: bad arguments");
  return h2b_launch_gather(h->perm, h->n, (const double2*)in, (double2*)out, q, (cudaStream_t)stream);
}

int h2b_scatter_perm(h2b_handle h, const void* in, void* out, int q, void* stream) {
  REQUIRE(h && in && out && q >= 1, H2B_EINVAL, "h2b_scatter_perm: bad arguments");
  return h2b_launch_scatter(h->perm, h->n, (const double2*)in, (double2*)out, q, (cudaStream_t)stream);
}

}  // extern "C"
