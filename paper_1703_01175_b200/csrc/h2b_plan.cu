// One-time preparation of an uploaded operator (host side + layout kernels):
//   * Vᵀ, Tᵀ copies and in-place Sᵀ (the panel layout of h2b_panel.cuh)
//   * coupling panel index (x̂ row feeding every panel row) and work items
//   * near-field work items (rows-per-CTA chosen from the block statistics)
//   * the q = 1 far-field schedule: span programs (h2b_common.cuh) chosen by
//     a small cost model over the split level `ls`.
#include <algorithm>
#include <cstring>
#include <functional>
#include <queue>
#include <set>
#include <tuple>

#include "h2b_common.cuh"
#include "h2b_panel.cuh"

int h2b_far_init_attributes(int smem_cap_bytes);
int h2b_mega_set_smem(int ns, int r, int bytes);
int h2b_mega_occupancy(int ns, int r, int smem_bytes, int* blocks_per_sm);
int h2b_mega_regs();
int h2b_tree_regs();
int h2b_near_stream_regs(int ns, int r);
int h2b_mega_static_smem();
int h2b_near_stream_static_smem(int ns, int r, int* bytes);
int h2b_near_stream_set_smem(int ns, int r, int bytes);
int h2b_near_rows_per_item(int ns, int r);
int h2b_tree_prepare(h2b_ctx* h, int max_ctas, int budget_bytes, int64_t* bytes, int* planned);
int h2b_tree_prepare_zero(h2b_ctx* h, TreeDev* d);
int h2b_tree_static_smem();
constexpr int TREE_BUDGET = 168 * 1024;  // shared memory of one subtree program (bytes)

namespace {

constexpr int SPAN_BUDGET = 12800;  // double2 elements (200 KB) of shared memory per span CTA
constexpr int SMEM_CAP = 227 * 1024;

struct BlockDesc {
  int64_t off;
  int32_t rows, cols;
};

// dst[off + c*rows + r] = src[off + r*cols + c]
__global__ void k_transpose_oop(const BlockDesc* __restrict__ bl, const double2* __restrict__ src,
                                double2* __restrict__ dst) {
  const BlockDesc b = bl[blockIdx.x];
  const int64_t n = (int64_t)b.rows * b.cols;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int64_t r = e / b.cols, c = e - r * b.cols;
    dst[b.off + c * b.rows + r] = src[b.off + e];
  }
}

// in-place block transpose through shared memory (the block must fit)
__global__ void k_transpose_inplace(const BlockDesc* __restrict__ bl, double2* buf) {
  extern __shared__ double2 sm[];
  const BlockDesc b = bl[blockIdx.x];
  const int64_t n = (int64_t)b.rows * b.cols;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) sm[e] = buf[b.off + e];
  __syncthreads();
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int64_t c = e / b.rows, r = e - c * b.rows;
    buf[b.off + e] = sm[r * b.cols + c];
  }
}

// flattened bases (prepare time): W rows of one leaf = V_l T_l T_parent(l) ... up to level ls
struct FlatLeaf {
  int64_t v_off, w_off;   // V_l in the V payload; first W element of the leaf's rows
  int32_t n, k0;          // leaf size and rank
  int32_t step_first, n_steps;
};
struct FlatStep {
  int64_t t_off;          // the child's rows inside its parent's T block (rows x cols, row-major)
  int32_t rows, cols;
};
__global__ void k_flatten(const FlatLeaf* __restrict__ leaves, const FlatStep* __restrict__ steps,
                          const double2* __restrict__ vbuf, const double2* __restrict__ tbuf,
                          double2* __restrict__ wbuf, int kmax) {
  extern __shared__ double2 fs[];
  const FlatLeaf L = leaves[blockIdx.x];
  double2* a = fs;
  double2* b = fs + (size_t)L.n * kmax;
  int k = L.k0;
  for (int e = threadIdx.x; e < L.n * k; e += blockDim.x) a[e] = vbuf[L.v_off + e];
  __syncthreads();
  for (int st = 0; st < L.n_steps; ++st) {
    const FlatStep S = steps[L.step_first + st];
    for (int e = threadIdx.x; e < L.n * S.cols; e += blockDim.x) {
      const int i = e / S.cols, j = e - i * S.cols;
      double2 acc = make_double2(0.0, 0.0);
      for (int l = 0; l < S.rows; ++l) cfma(acc, a[i * k + l], tbuf[S.t_off + (int64_t)l * S.cols + j]);
      b[i * S.cols + j] = acc;
    }
    __syncthreads();
    double2* t = a;
    a = b;
    b = t;
    k = S.cols;
  }
  for (int e = threadIdx.x; e < L.n * k; e += blockDim.x) wbuf[L.w_off + e] = a[e];
}

template <typename T>
int to_device(T** dst, const std::vector<T>& v, int64_t* acc) {
  const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  H2B_CUDA_TRY(cudaMalloc((void**)dst, bytes));
  if (!v.empty()) H2B_CUDA_TRY(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  if (acc) *acc += (int64_t)bytes;
  return H2B_OK;
}

// ------------------------------ span programs ------------------------------
struct Prog {
  std::vector<SpanHead> heads;
  std::vector<SpanCopy> copies, outs;
  std::vector<SpanOp> ops;
};

struct SB {  // a span under construction
  std::vector<SpanCopy> cp, out;
  std::vector<std::vector<SpanOp>> lv;
  int smem = 0;
  int alloc(int e) {
    const int o = smem;
    smem += e;
    return o;
  }
  int in(int kind, int64_t src, int64_t e) {
    const int o = alloc((int)e);
    if (e > 0) cp.push_back({src, kind, (int32_t)e, o, 0, 0});
    return o;
  }
  void outc(int kind, int64_t dst, int64_t e, int o) {
    if (e > 0) out.push_back({dst, kind, (int32_t)e, o, 0, 0});
  }
  void level() { lv.emplace_back(); }
  void op(int pay, int in_, int out_, int R, int w, int flags) {
    lv.back().push_back(SpanOp{pay, in_, out_, R, w, flags, panel_shift(w), 0});
  }
};

// append a finished span; returns false when it does not fit
bool finish(Prog& P, SB& s, int* smem_out) {
  int n_ops = 0;
  for (auto& l : s.lv) n_ops += (int)l.size();
  if ((int)s.lv.size() > SPAN_MAXLEV) return false;
  const int op_first = (int)P.ops.size();
  const int ops_smem = s.in(SRC_OPS, 2 * (int64_t)op_first, 2 * (int64_t)n_ops);
  // the write-back descriptors travel with the working set too (no serial global loads later)
  const int outs_smem = s.in(SRC_OUTS, 2 * (int64_t)P.outs.size(), 2 * (int64_t)s.out.size());
  if (s.smem > SPAN_BUDGET) return false;
  SpanHead hd{};
  hd.pad[1] = outs_smem;
  hd.copy_first = (int)P.copies.size();
  hd.n_copy = (int)s.cp.size();
  hd.out_first = (int)P.outs.size();
  hd.n_out = (int)s.out.size();
  hd.ops_smem = ops_smem;
  hd.n_ops = n_ops;
  hd.smem_elems = s.smem;
  hd.nlev = (int)s.lv.size();
  int64_t bytes = 0;
  for (auto& c : s.cp) bytes += 16 * (int64_t)c.elems;
  hd.pad[0] = (int32_t)bytes;  // expected transaction bytes of the span's staging
  int acc = 0;
  hd.lvl[0] = 0;
  for (size_t i = 0; i < s.lv.size(); ++i) {
    for (auto& o : s.lv[i]) P.ops.push_back(o);
    acc += (int)s.lv[i].size();
    hd.lvl[i + 1] = acc;
  }
  P.copies.insert(P.copies.end(), s.cp.begin(), s.cp.end());
  P.outs.insert(P.outs.end(), s.out.begin(), s.out.end());
  P.heads.push_back(hd);
  *smem_out = std::max(*smem_out, s.smem);
  return true;
}

struct Lvl {  // a contiguous packed range [a, b) of one level
  int a, b;
};

std::vector<Lvl> desc_ranges(const h2b_ctx* h, int r, int max_levels) {
  std::vector<Lvl> out;
  int a = r, b = r + 1;
  while (a < b && (int)out.size() < max_levels) {
    out.push_back({a, b});
    int na = -1, nb = -1;
    for (int p = a; p < b; ++p)
      if (h->c_child_lo[p] >= 0) {
        if (na < 0) na = h->c_child_lo[p];
        nb = h->c_child_hi[p] + 1;
      }
    if (na < 0) break;
    a = na;
    b = nb;
  }
  return out;
}

int m_of(const h2b_ctx* h, int p) { return h->c_rank[h->c_child_lo[p]] + h->c_rank[h->c_child_hi[p]]; }

int level_of(const h2b_ctx* h, int p) {
  return (int)(std::upper_bound(h->level_ptr.begin(), h->level_ptr.end(), p) - h->level_ptr.begin()) - 1;
}

// payload ranges of a level range: V of its leaves, T of its non-leaves
void pay_ranges(const h2b_ctx* h, Lvl L, int64_t& vb, int64_t& ve, int64_t& tb, int64_t& te) {
  vb = ve = tb = te = 0;
  int fl = -1, ll = -1, fn = -1, ln = -1;
  for (int p = L.a; p < L.b; ++p) {
    if (h->c_child_lo[p] < 0) {
      if (fl < 0) fl = p;
      ll = p;
    } else {
      if (fn < 0) fn = p;
      ln = p;
    }
  }
  if (fl >= 0) {
    vb = h->c_voff[fl];
    ve = h->c_voff[ll] + (int64_t)h->c_size[ll] * h->c_rank[ll] - vb;
  }
  if (fn >= 0) {
    tb = h->c_toff[fn];
    te = h->c_toff[ln] + (int64_t)m_of(h, ln) * h->c_rank[ln] - tb;
  }
}

struct Plan {
  Prog prog;
  std::vector<SpanLaunch> up, down_head, down_tail;
  double cost = 1e30;
  int ls = -1, top_staged = 0;
};

// cost of one launch (microseconds): launch + staging + in-CTA levels
double launch_cost(int smem_elems, int nlev) { return 2.0 + 16.0 * smem_elems / 100e3 + 0.3 * nlev; }

// subtree span rooted at r covering levels [level(r), level(r) + nl): UP or DOWN program
// deep (flattened bottom tier): the root's own level is left to the flat tasks: no x̂ output
// for the root (up), no propagation from the root and leaf results into y_deep (down)
bool build_subtree_span(const h2b_ctx* h, Prog& P, int r, int nl, bool up, bool input_last,
                        int* smem_max, bool deep = false) {
  SB s;
  auto R = desc_ranges(h, r, nl);
  const int n = (int)R.size();
  const int ncomp = input_last ? n - 1 : n;  // levels computed by this span
  std::vector<int> vs(n, 0), ts(n, 0), xh(n, 0);
  std::vector<int64_t> vb(n), ve(n), tb(n), te(n);
  int x_sm = 0;
  bool has_leaf = false;
  for (int i = 0; i < ncomp; ++i)
    for (int p = R[i].a; p < R[i].b; ++p) has_leaf |= h->c_child_lo[p] < 0;
  if (up && has_leaf) x_sm = s.in(SRC_X, h->c_start[r], h->c_size[r]);
  for (int i = 0; i < n; ++i) {
    pay_ranges(h, R[i], vb[i], ve[i], tb[i], te[i]);
    const int64_t xb = h->c_xoff[R[i].a], xe = h->c_xoff[R[i].b] - xb;
    if (i < ncomp) {
      vs[i] = s.in(up ? SRC_V : SRC_VT, vb[i], ve[i]);
      ts[i] = s.in(up ? SRC_T : SRC_TT, tb[i], te[i]);
    }
    if (up)
      xh[i] = (i < ncomp) ? s.alloc((int)xe) : s.in(SRC_XHAT, xb, xe);
    else
      xh[i] = (deep && i == 0) ? s.alloc((int)xe) : s.in(SRC_YHAT, xb, xe);
  }
  auto emit_level = [&](int i) {
    s.level();
    const int64_t xb = h->c_xoff[R[i].a];
    for (int p = R[i].a; p < R[i].b; ++p) {
      const int k = h->c_rank[p];
      if (k == 0) continue;
      const int out_here = xh[i] + (int)(h->c_xoff[p] - xb);
      const int lo = h->c_child_lo[p];
      if (lo < 0) {
        const int pay = vs[i] + (int)(h->c_voff[p] - vb[i]);
        if (up)
          s.op(pay, x_sm + (h->c_start[p] - h->c_start[r]), out_here, h->c_size[p], k, 0);
        else
          s.op(pay, out_here, h->c_start[p], k, h->c_size[p], deep ? (OP_OUT_Y | OP_OUT_YD) : (OP_ACC | OP_OUT_Y));
      } else {
        const int m = m_of(h, p);
        const int pay = ts[i] + (int)(h->c_toff[p] - tb[i]);
        const int child = xh[i + 1] + (int)(h->c_xoff[lo] - h->c_xoff[R[i + 1].a]);
        if (up)
          s.op(pay, child, out_here, m, k, 0);
        else if (m > 0)
          s.op(pay, out_here, child, k, m, OP_ACC);
      }
    }
  };
  const int first = deep ? 1 : 0;  // deep: the root level belongs to the flat tasks
  if (up)
    for (int i = ncomp - 1; i >= first; --i) emit_level(i);
  else
    for (int i = first; i < ncomp; ++i) emit_level(i);
  if (up) {
    for (int i = first; i < ncomp; ++i)
      s.outc(SRC_XHAT, h->c_xoff[R[i].a], h->c_xoff[R[i].b] - h->c_xoff[R[i].a], xh[i]);
  } else if (input_last) {
    const int i = n - 1;
    s.outc(SRC_YHAT, h->c_xoff[R[i].a], h->c_xoff[R[i].b] - h->c_xoff[R[i].a], xh[i]);
  }
  return finish(P, s, smem_max);
}

// single-cluster spans of level l (one CTA per cluster); false if one does not fit
bool build_level_spans(const h2b_ctx* h, Prog& P, int l, bool up, SpanLaunch& L) {
  L = SpanLaunch{(int)P.heads.size(), 0, 0, 0, -1};
  int smem = 0;
  for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) {
    const int k = h->c_rank[p];
    if (k == 0) continue;
    const int lo = h->c_child_lo[p];
    SB s;
    s.level();
    if (lo < 0) {
      const int n = h->c_size[p];
      if (up) {
        const int v = s.in(SRC_V, h->c_voff[p], (int64_t)n * k);
        const int xi = s.in(SRC_X, h->c_start[p], n);
        const int xo = s.alloc(k);
        s.op(v, xi, xo, n, k, 0);
        s.outc(SRC_XHAT, h->c_xoff[p], k, xo);
      } else {
        const int v = s.in(SRC_VT, h->c_voff[p], (int64_t)n * k);
        const int yi = s.in(SRC_YHAT, h->c_xoff[p], k);
        s.op(v, yi, h->c_start[p], k, n, OP_ACC | OP_OUT_Y);
      }
    } else {
      const int m = m_of(h, p);
      if (up) {
        const int t = s.in(SRC_T, h->c_toff[p], (int64_t)m * k);
        const int xi = s.in(SRC_XHAT, h->c_xoff[lo], m);
        const int xo = s.alloc(k);
        s.op(t, xi, xo, m, k, 0);
        s.outc(SRC_XHAT, h->c_xoff[p], k, xo);
      } else {
        if (m == 0) continue;
        const int t = s.in(SRC_TT, h->c_toff[p], (int64_t)m * k);
        const int yi = s.in(SRC_YHAT, h->c_xoff[p], k);
        const int yc = s.in(SRC_YHAT, h->c_xoff[lo], m);
        s.op(t, yi, yc, k, m, OP_ACC);
        s.outc(SRC_YHAT, h->c_xoff[lo], m, yc);
      }
    }
    if (!finish(P, s, &smem)) return false;
    ++L.n_heads;
  }
  L.smem_elems = smem;
  return true;
}

bool level_active(const h2b_ctx* h, int l, bool up) {
  for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) {
    if (h->c_rank[p] == 0) continue;
    if (up || h->c_child_lo[p] < 0 || m_of(h, p) > 0) return true;
  }
  return false;
}

// per-level launches for levels in [l0, l1) (up: deepest first); fallback kernels if needed
void per_level(const h2b_ctx* h, Prog& P, int l0, int l1, bool up, std::vector<SpanLaunch>& out,
               double& cost, bool& ok_leaves) {
  std::vector<int> lv;
  for (int l = l0; l < l1; ++l) lv.push_back(l);
  if (up) std::reverse(lv.begin(), lv.end());
  for (int l : lv) {
    if (!level_active(h, l, up)) continue;
    SpanLaunch L;
    const size_t h0 = P.heads.size(), c0 = P.copies.size(), o0 = P.outs.size(), op0 = P.ops.size();
    if (build_level_spans(h, P, l, up, L)) {
      if (L.n_heads > 0) {
        out.push_back(L);
        cost += launch_cost(L.smem_elems, 1);
      }
    } else {  // roll back and fall back to the per-level kernel
      P.heads.resize(h0);
      P.copies.resize(c0);
      P.outs.resize(o0);
      P.ops.resize(op0);
      bool has_leaf = false;
      for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p) has_leaf |= h->c_child_lo[p] < 0;
      if (has_leaf) ok_leaves = false;  // leaf levels have no per-level fallback in span mode
      out.push_back(SpanLaunch{0, 0, 0, 0, l});
      cost += 8.0;
    }
  }
}

bool plan_with_split(const h2b_ctx* h, int ls, Plan& pl) {
  pl = Plan();
  pl.ls = ls;
  Prog& P = pl.prog;
  const int L = h->depth;
  // bottom spans: every cluster at level ls roots one span over all deeper levels
  SpanLaunch up_b{(int)P.heads.size(), 0, 0, 0, -1};
  for (int r = h->level_ptr[ls]; r < h->level_ptr[ls + 1]; ++r) {
    if (!build_subtree_span(h, P, r, L - ls, true, false, &up_b.smem_elems)) return false;
    ++up_b.n_heads;
  }
  SpanLaunch dn_b{(int)P.heads.size(), 0, 0, 0, -1};
  for (int r = h->level_ptr[ls]; r < h->level_ptr[ls + 1]; ++r) {
    if (!build_subtree_span(h, P, r, L - ls, false, false, &dn_b.smem_elems)) return false;
    ++dn_b.n_heads;
  }
  int nlev_b = 0;
  for (int r = h->level_ptr[ls]; r < h->level_ptr[ls + 1]; ++r)
    nlev_b = std::max(nlev_b, (int)desc_ranges(h, r, L).size());
  pl.up.push_back(up_b);
  pl.down_tail.push_back(dn_b);
  double cost = launch_cost(up_b.smem_elems, nlev_b) + launch_cost(dn_b.smem_elems, nlev_b);
  if (ls > 0) {
    // leaves above the split would belong to no span
    for (int p = 0; p < h->level_ptr[ls]; ++p)
      if (h->c_child_lo[p] < 0) return false;
    bool any_up = false, any_dn = false;
    for (int l = 0; l < ls; ++l) {
      any_up |= level_active(h, l, true);
      any_dn |= level_active(h, l, false);
    }
    const size_t h0 = P.heads.size(), c0 = P.copies.size(), o0 = P.outs.size(), op0 = P.ops.size();
    int su = 0, sd = 0;
    const int root = h->level_ptr[0];
    const bool top_ok = (!any_up || build_subtree_span(h, P, root, ls + 1, true, true, &su)) &&
                        (!any_dn || build_subtree_span(h, P, root, ls + 1, false, true, &sd));
    if (top_ok) {
      pl.top_staged = 1;
      int hi = (int)h0;
      if (any_up) {
        pl.up.push_back(SpanLaunch{hi++, 1, su, 1, -1});
        cost += launch_cost(su, ls);
      }
      if (any_dn) {
        pl.down_head.push_back(SpanLaunch{hi++, 1, sd, 1, -1});
        cost += launch_cost(sd, ls);
      }
    } else {
      P.heads.resize(h0);
      P.copies.resize(c0);
      P.outs.resize(o0);
      P.ops.resize(op0);
      bool ok = true;
      per_level(h, P, 0, ls, true, pl.up, cost, ok);
      per_level(h, P, 0, ls, false, pl.down_head, cost, ok);
    }
  }
  pl.cost = cost;
  return true;
}

// ------------------------- persistent-kernel task graph -------------------------
constexpr int MEGA_BUDGET = 7000;  // double2 elements (112 KB): largest work area of a far CTA
                                   // (5800 / 8200 measured 2-3 us slower at cfg2: profiles/r01_budget_ab.txt)
constexpr int MEGA_BUDGET_MAX = 12000;  // tuning override ceiling (the near ring shrinks to fit)
constexpr int MEGA_BLOB_MAX = 1024;  // 16-byte slots (16 KB) of per-CTA task blob
constexpr double NEAR_TASK_BYTES = 64e3;  // target D bytes per near-field task

std::vector<DepRange> to_ranges(std::vector<int> ids) {
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  std::vector<DepRange> out;
  for (int v : ids) {
    if (!out.empty() && out.back().hi == v)
      out.back().hi = v + 1;
    else
      out.push_back({v, v + 1});
  }
  return out;
}

// does every span of a tier fit the budget?  (built into a scratch program)
bool tier_fits(const h2b_ctx* h, int root_level, int nl, bool input_last, int budget) {
  Prog P;
  int sm = 0;
  for (int r = h->level_ptr[root_level]; r < h->level_ptr[root_level + 1]; ++r) {
    if (!build_subtree_span(h, P, r, nl, true, input_last, &sm)) return false;
    if (!build_subtree_span(h, P, r, nl, false, input_last, &sm)) return false;
  }
  return sm <= budget;
}

struct MegaPlan {
  Prog prog;
  std::vector<Task> tasks;
  std::vector<DepRange> deps;
  std::vector<NearTask> near_tasks;
  std::vector<NearItem> leaf_items;
  std::vector<CoupleGroup> groups;
  std::vector<CoupleItem> citems;
  std::vector<int4> recs;
  std::vector<int2> cta_lists;
  std::vector<int> task_list;
  std::vector<int4> near_recs;  // near-field task records (claimed dynamically by the stream kernel)
  std::vector<int2> near_idx;   // per near task {first slot, slots} in near_recs
  int ns = 0, r = 1, smem = 0, tiers = 0, blob_slots = 0, near_rec_max = 0;
  bool flat = false;
  std::vector<FlatRec> flat_recs;  // per split-level cluster (flat mode)
  int64_t flat_elems = 0;          // W buffer size (double2)
  int flat_level = -1;             // ls
  double est_makespan = 0.0;
};

bool plan_mega(const h2b_ctx* h, const std::vector<CoupleItem>& citems_all,
               const std::vector<int32_t>& targets, int grid_est, int budget, MegaPlan& mp) {
  const int L = h->depth;
  int min_leaf = L - 1;
  for (int p = 0; p < h->P; ++p)
    if (h->c_child_lo[p] < 0) min_leaf = std::min(min_leaf, level_of(h, p));
  // ---- tiers: bottom split ls, then upper splits up to the root -----------------
  int ls = -1;
  int ls_min = 0;
  if (const char* e = getenv("H2B_DEBUG_LS")) ls_min = std::max(0, atoi(e));  // tuning aid
  for (int l = ls_min; l <= min_leaf && ls < 0; ++l)
    if (tier_fits(h, l, L - l, false, budget)) ls = l;
  if (ls < 0) return false;
  std::vector<int> splits = {ls};  // bottom-up list of tier roots
  while (splits.back() > 0) {
    const int cur = splits.back();
    int s = -1;
    for (int c = 0; c < cur && s < 0; ++c)
      if (tier_fits(h, c, cur - c + 1, true, budget)) s = c;
    if (s < 0) return false;
    splits.push_back(s);
  }
  const int m = (int)splits.size();  // tier 0 = bottom
  mp.tiers = m;
  // Flattened bottom tier: the critical chain then enters the upper tiers through one
  // W_cᵀ x_c per split-level cluster instead of a sweep over all the levels below it, and
  // leaves them through one W_c ŷ_c (plus y_deep from the deep spans, off the critical
  // chain).  Needs every leaf on the deepest level, a few levels below ls and W_c (plus x_c)
  // in the work area.
  bool flat = m >= 2 && min_leaf == L - 1 && h->uniform_leaf > 0 && ls <= L - 3 && !getenv("H2B_NO_FLAT");
  for (int r = h->level_ptr[ls]; flat && r < h->level_ptr[ls + 1]; ++r)
    flat = h->c_rank[r] > 0 && (int64_t)h->c_size[r] * (h->c_rank[r] + 1) <= budget;
  for (int p = h->level_ptr[ls]; flat && p < h->P; ++p)
    if (h->c_child_lo[p] < 0) flat = h->c_rank[p] > 0;
  if (flat) {  // the prepare-time product kernel keeps two (leaf x max rank) tiles in smem
    int kmax = 1;
    for (int p = 0; p < h->P; ++p) kmax = std::max(kmax, h->c_rank[p]);
    flat = 2 * 16 * h->uniform_leaf * kmax <= 200 * 1024;
  }
  mp.flat = flat;
  mp.flat_level = ls;
  // ---- span programs ---------------------------------------------------------------
  struct SpanRef {
    int root, up_head, dn_head;  // head index or -1 when the span has no ops
  };
  std::vector<std::vector<SpanRef>> tier(m);
  Prog& P = mp.prog;
  int smem = 0;
  for (int i = 0; i < m; ++i) {
    const int rl = splits[i];
    const bool bottom = i == 0;
    const int nl = bottom ? L - rl : splits[i - 1] - rl + 1;
    for (int r = h->level_ptr[rl]; r < h->level_ptr[rl + 1]; ++r) {
      SpanRef s{r, -1, -1};
      for (int dir = 0; dir < 2; ++dir) {
        const size_t h0 = P.heads.size();
        if (!build_subtree_span(h, P, r, nl, dir == 0, !bottom, &smem, flat && bottom)) return false;
        if (P.heads.back().n_ops == 0) {  // nothing to do: drop it again
          P.ops.resize(P.ops.size() - 0);
          P.copies.resize(P.heads.back().copy_first);
          P.outs.resize(P.heads.back().out_first);
          P.heads.resize(h0);
        } else {
          (dir == 0 ? s.up_head : s.dn_head) = (int)h0;
        }
      }
      tier[i].push_back(s);
    }
  }
  mp.smem = 16 * smem;
  // ---- task list -------------------------------------------------------------------
  // self-contained task records (see Task in h2b_common.cuh)
  std::vector<int4>* rec_out = &mp.recs;
  auto push_slots = [&](const void* data, size_t bytes) {
    const size_t n = (bytes + 15) / 16;
    const size_t at = rec_out->size();
    rec_out->resize(at + n, int4{0, 0, 0, 0});
    std::memcpy(rec_out->data() + at, data, bytes);
  };
  auto make_record = [&](int type, int arg) -> bool {
    if (type == T_SPAN) {
      SpanHead hd = mp.prog.heads[arg];
      const int c0 = hd.copy_first;
      hd.copy_first = 0;  // copies follow the head inside the record
      push_slots(&hd, sizeof(SpanHead));
      push_slots(mp.prog.copies.data() + c0, sizeof(SpanCopy) * hd.n_copy);
    } else if (type == T_FLAT_UP || type == T_FLAT_DOWN) {
      push_slots(&mp.flat_recs[arg], sizeof(FlatRec));
    } else if (type == T_COUPLE) {
      const CoupleGroup& g = mp.groups[arg];
      const int4 hdr{g.n_items, g.cta_mode, 0, 0};
      push_slots(&hdr, sizeof(hdr));
      push_slots(mp.citems.data() + g.item_first, sizeof(CoupleItem) * g.n_items);
    } else if (mp.ns == 0) {
      const int4 hdr{arg, 0, 0, 0};
      push_slots(&hdr, sizeof(hdr));
    } else {
      const NearTask& nt = mp.near_tasks[arg];
      std::vector<int64_t> lv, bl;
      for (int li = nt.leaf_first; li < nt.leaf_first + nt.n_leaves; ++li) {
        const int t = h->h_leaves[li];
        const int64_t b0 = h->d_row_ptr[t], b1 = h->d_row_ptr[t + 1];
        lv.push_back(h->c_start[t]);
        lv.push_back(b1 - b0);
        for (int64_t b = b0; b < b1; ++b) {
          bl.push_back(h->d_off[b] + (int64_t)nt.row0 * mp.ns);
          bl.push_back(h->c_start[h->d_col[b]]);
        }
      }
      const int4 hdr{(int)(bl.size() / 2), nt.n_leaves, nt.row0, 0};
      push_slots(&hdr, sizeof(hdr));
      push_slots(lv.data(), 8 * lv.size());
      push_slots(bl.data(), 8 * bl.size());
    }
    return true;
  };
  // ---- logical task graph; the queue order is decided afterwards by a simulation --------
  struct LTask {
    int type, arg;
    std::vector<int> deps;  // logical ids
    double dur;             // estimated run time (us)
  };
  std::vector<LTask> lt;
  const double G = (double)std::max(1, grid_est);
  const double cta_bw = 6.5e6 / G;  // bytes per microsecond per CTA when all CTAs stream
  auto add_l = [&](int type, int arg, std::vector<int> deps, double dur) {
    lt.push_back({type, arg, std::move(deps), dur});
    return (int)lt.size() - 1;
  };
  // the clusters a span computes (for producer / consumer maps)
  auto span_clusters = [&](int tier_i, int root, bool with_input) {
    const bool bottom = tier_i == 0;
    const int nl = bottom ? L - splits[tier_i] : splits[tier_i - 1] - splits[tier_i] + 1;
    auto R = desc_ranges(h, root, nl);
    std::vector<int> cl;
    const int n = (int)R.size() - ((bottom || with_input) ? 0 : 1);
    for (int i = 0; i < n; ++i)
      for (int p = R[i].a; p < R[i].b; ++p) cl.push_back(p);
    return cl;
  };
  // estimated run times (us), calibrated on B200 traces: staging + ~1 us per level + write-back
  auto span_dur = [&](int head) { return 3.5 + 1.0 * mp.prog.heads[head].nlev; };
  // ---- near-field work list (leaf order) --------------------------------------------
  const int ns = h->uniform_leaf;
  const int nleaves = (int)h->h_leaves.size();
  for (int i = 0; i < nleaves; ++i) {
    const int t = h->h_leaves[i];
    mp.leaf_items.push_back({(int64_t)h->c_start[t], (int32_t)h->d_row_ptr[t],
                             (int32_t)(h->d_row_ptr[t + 1] - h->d_row_ptr[t]), 0, 0});
  }
  std::vector<NearTask>& nts = mp.near_tasks;
  std::vector<double> nt_bytes;
  auto leaf_nb = [&](int i) {
    const int t = h->h_leaves[i];
    return (int)(h->d_row_ptr[t + 1] - h->d_row_ptr[t]);
  };
  if (ns == 32 || ns == 64) {
    const double avg_nb = (double)h->n_near / std::max(1, nleaves);
    const double row_bytes = ns * 16.0 * avg_nb;
    const int rpp = 256 / (ns / 2);  // rows per pass of a 256-thread CTA
    int R = 1;
    // tasks of ~NEAR_TASK_BYTES: small tasks keep the tail of the static split short.  (Choosing
    // the slice height by an estimated near-field makespan made cfg1's near field 37 -> 25 us
    // but its step 43 -> 46 us: the faster stream slows the concurrent far field more.)
    double task_bytes = NEAR_TASK_BYTES;
    if (const char* e = getenv("H2B_NEAR_TASK_BYTES")) task_bytes = std::max(4e3, atof(e));  // tuning aid
    while (R * 2 * rpp <= ns && R * 2 <= (ns == 32 ? 2 : 8) && R * 2 * rpp * row_bytes <= task_bytes) R *= 2;
    if (const char* e = getenv("H2B_NEAR_R")) R = std::max(1, std::min(ns == 32 ? 2 : 8, atoi(e)));  // tuning aid
    mp.ns = ns;
    mp.r = R;
    const int rb = R * rpp;
    if (rb < ns) {
      for (int i = 0; i < nleaves; ++i)
        for (int r0 = 0; r0 < ns; r0 += rb) {
          nts.push_back({i, 1, r0, 0});
          nt_bytes.push_back(16.0 * rb * ns * leaf_nb(i));
        }
    } else {
      // group whole leaves into tasks (the ring streams on across task boundaries)
      const int per = std::max(1, (int)(task_bytes / (ns * row_bytes) + 0.5));
      int i = 0;
      while (i < nleaves) {
        int c = 0, blocks = 0;
        while (i + c < nleaves && c < per && c < 64) {
          const int nb = leaf_nb(i + c);
          if (c > 0 && blocks + nb > NEAR_REC_MAXB) break;
          blocks += nb;
          ++c;
        }
        nts.push_back({i, c, 0, 0});
        nt_bytes.push_back(16.0 * ns * ns * blocks);
        i += c;
      }
    }
    for (int i = 0; i < nleaves; ++i)  // a single leaf must fit a record too
      if (leaf_nb(i) > NEAR_REC_MAXB) return false;
  } else {
    mp.ns = 0;
    mp.r = 1;
    for (int i = 0; i < nleaves; ++i) {
      nts.push_back({i, 1, 0, 0});
      nt_bytes.push_back(16.0 * h->c_size[h->h_leaves[i]] * 64.0 * leaf_nb(i));
    }
  }
  // the near field runs in its own streaming kernel, concurrently with the far-field task
  // graph (both accumulate into a zeroed y): its tasks are not part of the graph below
  for (size_t k = 0; k < nts.size(); ++k) {
    std::vector<int4> rec;
    rec_out = &rec;
    make_record(T_NEAR, ns == 32 || ns == 64 ? (int)k : nts[k].leaf_first);
    mp.near_idx.push_back({(int)mp.near_recs.size(), (int)rec.size()});
    mp.near_recs.insert(mp.near_recs.end(), rec.begin(), rec.end());
    mp.near_rec_max = std::max(mp.near_rec_max, (int)rec.size());
  }
  rec_out = &mp.recs;
  const int n_near = 0;
  // ---- far-field tasks in topological order ---------------------------------------------
  std::vector<int> up_task(h->P, -1), up_of_span_root(h->P, -1), flat_of(h->P, -1);
  if (flat) {  // the flattened bases' records, one per split-level cluster
    int64_t w = 0;
    for (int r = h->level_ptr[ls]; r < h->level_ptr[ls + 1]; ++r) {
      flat_of[r] = (int)mp.flat_recs.size();
      mp.flat_recs.push_back(FlatRec{w, (int64_t)h->c_start[r], h->c_xoff[r], h->c_size[r], h->c_rank[r]});
      w += (int64_t)h->c_size[r] * h->c_rank[r];
      mp.smem = std::max(mp.smem, 16 * h->c_size[r] * (h->c_rank[r] + 1));
    }
    mp.flat_elems = w;
  }
  auto flat_dur = [&](int r) { return 3.0 + 16.0 * h->c_size[r] * h->c_rank[r] / 2e4; };
  for (int i = 0; i < m; ++i)  // A. forward spans, bottom tier first
    for (auto& s : tier[i]) {
      std::vector<int> deps;
      if (i > 0)  // children spans: tier i-1 spans rooted inside this span's input level
        for (int p : span_clusters(i, s.root, true))
          if (up_of_span_root[p] >= 0 && level_of(h, p) == splits[i - 1]) deps.push_back(up_of_span_root[p]);
      if (flat && i == 0) {  // x̂ of the root straight from x; the deep span does the levels below
        const int fid = add_l(T_FLAT_UP, flat_of[s.root], {}, flat_dur(s.root));
        up_of_span_root[s.root] = fid;
        up_task[s.root] = fid;
        if (s.up_head < 0) continue;
        const int id = add_l(T_SPAN, s.up_head, {}, span_dur(s.up_head));
        for (int p : span_clusters(0, s.root, false))
          if (p != s.root) up_task[p] = id;
        continue;
      }
      if (s.up_head < 0) continue;
      const int id = add_l(T_SPAN, s.up_head, deps, span_dur(s.up_head));
      up_of_span_root[s.root] = id;
      for (int p : span_clusters(i, s.root, false)) up_task[p] = id;
    }
  // B. coupling groups (targets in packed order; panels + gathered x̂ bounded by the budget)
  std::vector<int> group_task(h->P, -1);
  std::vector<std::vector<int>> group_members;  // targets of each coupling group (plan check)
  int couple_smem = 0;
  {
    const int64_t cap = 4000;  // double2 elements per warp-mode group (64 KB)
    int couple_items = 8, couple_items_deep = 32;
    if (const char* e = getenv("H2B_DEBUG_COUPLE_ITEMS")) couple_items = std::max(1, atoi(e));  // profiling
    if (const char* e = getenv("H2B_DEBUG_COUPLE_DEEP")) couple_items_deep = std::max(1, atoi(e));
    size_t i = 0;
    while (i < citems_all.size()) {
      const int64_t e0 = (int64_t)citems_all[i].R * citems_all[i].w + citems_all[i].R;
      CoupleGroup g{(int)mp.citems.size(), 0, 0, 0};
      std::vector<int> members;
      int64_t elems = 0, pelems = 0;
      if (e0 > 3000) {  // a big panel: the whole CTA streams it
        if (citems_all[i].R > budget) return false;
        g.cta_mode = 1;
        mp.citems.push_back(citems_all[i]);
        members.push_back(targets[i]);
        elems = citems_all[i].R;
        pelems = (int64_t)citems_all[i].R * citems_all[i].w;
        ++i;
      } else {
        // a group is one round of the CTA's warps (8 panels), within one level: the coupling
        // tasks sit on the far-field critical path, so many small tasks beat few big ones
        const int lvl0 = level_of(h, targets[i]);
        // below the split level the couplings are off the critical chain (they only have to be
        // done before the deep down spans): bigger groups there amortise the per-task overhead
        const int max_items = lvl0 > ls ? couple_items_deep : couple_items;
        while (i < citems_all.size() && (int)members.size() < max_items) {
          const int64_t e = (int64_t)citems_all[i].R * citems_all[i].w + citems_all[i].R;
          if (e > 3000 || elems + e > cap || level_of(h, targets[i]) != lvl0) break;
          mp.citems.push_back(citems_all[i]);
          members.push_back(targets[i]);
          elems += e;
          pelems += (int64_t)citems_all[i].R * citems_all[i].w;
          ++i;
        }
      }
      couple_smem = std::max<int>(couple_smem, (int)elems);
      g.n_items = (int)members.size();
      std::vector<int> deps;
      for (int t : members)
        for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
          const int sc = h->s_col[b];
          if (h->c_rank[sc] > 0 && up_task[sc] >= 0) deps.push_back(up_task[sc]);
        }
      mp.groups.push_back(g);
      group_members.push_back(members);
      const int id = add_l(T_COUPLE, (int)mp.groups.size() - 1, deps, 3.5 + 16.0 * pelems / 2e4);
      for (int t : members) group_task[t] = id;
    }
  }
  mp.smem = std::max(mp.smem, 16 * couple_smem);
  // C. backward spans, root tier first; D. bottom tier after the near tasks of its leaves
  std::vector<int> dn_writer(h->P, -1);  // task that last wrote ŷ of a tier root
  auto down_deps = [&](int tier_i, const SpanRef& s) {
    std::vector<int> deps;
    if (dn_writer[s.root] >= 0) deps.push_back(dn_writer[s.root]);
    for (int p : span_clusters(tier_i, s.root, true))
      if (group_task[p] >= 0) deps.push_back(group_task[p]);
    return deps;
  };
  for (int i = m - 1; i >= 1; --i)
    for (auto& s : tier[i]) {
      if (s.dn_head < 0) continue;
      const int id = add_l(T_SPAN, s.dn_head, down_deps(i, s), span_dur(s.dn_head));
      auto R = desc_ranges(h, s.root, splits[i - 1] - splits[i] + 1);
      for (int p = R.back().a; p < R.back().b; ++p) dn_writer[p] = id;  // writes back the input level
    }
  for (auto& s : tier[0]) {
    if (flat) {
      // deep span: the levels below the root, from their couplings only, into y_deep; then the
      // flat task adds W ŷ_root (ŷ_root complete once the tier above wrote it back) and y_deep
      std::vector<int> deps, fdeps;
      for (int p : span_clusters(0, s.root, true))
        if (p != s.root && group_task[p] >= 0) deps.push_back(group_task[p]);
      if (s.dn_head >= 0) fdeps.push_back(add_l(T_SPAN, s.dn_head, deps, span_dur(s.dn_head)));
      if (dn_writer[s.root] >= 0) fdeps.push_back(dn_writer[s.root]);
      if (group_task[s.root] >= 0) fdeps.push_back(group_task[s.root]);
      add_l(T_FLAT_DOWN, flat_of[s.root], fdeps, flat_dur(s.root));
      continue;
    }
    if (s.dn_head < 0) continue;
    std::vector<int> deps = down_deps(0, s);
    add_l(T_SPAN, s.dn_head, deps, span_dur(s.dn_head));
  }
  // ---- static schedule -----------------------------------------------------------------
  // CTA roles: the first g_near CTAs stream the near field (contiguous runs of row panels of
  // ~equal bytes, never waiting); the others run the far-field tasks, assigned by list
  // scheduling (earliest-ready task to the earliest-free CTA) against estimated durations.
  // Global order = near panels, then far tasks in assignment order; every CTA's list is
  // sorted by it and every dependency points to an earlier task.
  const int nl_all = (int)lt.size();
  const int n_far = nl_all - n_near;
  const int g_total = std::max(2, grid_est);
  int g_near = 0;
  int g_far = n_far > 0 ? g_total : 0;
  std::vector<double> fin(nl_all, 0.0);
  std::vector<std::vector<int>> lists(g_near + g_far);
  {
    double tot = 0.0;
    for (int k = 0; k < n_near; ++k) tot += nt_bytes[k];
    const double per_cta = tot / g_near, bw = 6.5e6 / g_near;
    double acc = 0.0, cta_t = 0.0;
    int c = 0;
    for (int k = 0; k < n_near; ++k) {
      if (c < g_near - 1 && acc >= per_cta * (c + 1)) {
        ++c;
        cta_t = 0.0;
      }
      acc += nt_bytes[k];
      cta_t += 1.0 + nt_bytes[k] / bw;
      fin[k] = cta_t;
      lists[c].push_back(k);
    }
  }
  std::vector<int> order;  // far tasks in assignment order
  if (n_far > 0) {
    std::vector<int> missing(nl_all, 0);
    std::vector<std::vector<int>> users(nl_all);
    for (int id = n_near; id < nl_all; ++id)
      for (int d : lt[id].deps)
        if (d >= n_near) {
          ++missing[id];
          users[d].push_back(id);
        }
    auto ready_time = [&](int id) {
      double r = 0.0;
      for (int d : lt[id].deps) r = std::max(r, fin[d]);
      return r;
    };
    // upward rank: the longest estimated path from a task to the end (ids are topological)
    std::vector<double> rank(nl_all, 0.0);
    for (int id = nl_all - 1; id >= n_near; --id) {
      double m = 0.0;
      for (int u : users[id]) m = std::max(m, rank[u]);
      rank[id] = lt[id].dur + m;
    }
    // list scheduling: the earliest-ready task first (the more critical one on ties), placed on
    // a CTA that is free by then and whose previous task ends latest (best fit), so the
    // critical chain never queues behind a task of another branch that waits for its inputs
    double slack = 2.0;
    if (const char* e = getenv("H2B_DEBUG_SLACK")) slack = atof(e);  // profiling
    using QE = std::tuple<double, double, int>;  // ready time, -rank, id
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> cand;
    std::multiset<std::pair<double, int>> cta_free;
    for (int id = n_near; id < nl_all; ++id)
      if (missing[id] == 0) cand.push({ready_time(id), -rank[id], id});
    for (int c = 0; c < g_far; ++c) cta_free.insert({0.0, g_near + c});
    while (!cand.empty()) {
      const auto [rt, nr, id] = cand.top();
      cand.pop();
      auto it = cta_free.upper_bound({rt, 1 << 30});
      if (it != cta_free.begin()) --it;  // best fit: free by rt, latest such
      const auto [ft, c] = *it;
      cta_free.erase(it);
      fin[id] = std::max(rt, ft) + lt[id].dur;
      // the CTA counts as busy for `slack` times the estimate: run times vary under load, and a
      // task that runs late must not hold up a critical one queued behind it on the same CTA
      cta_free.insert({std::max(rt, ft) + slack * lt[id].dur, c});
      lists[c].push_back(id);
      order.push_back(id);
      for (int u : users[id])
        if (--missing[u] == 0) cand.push({ready_time(u), -rank[u], u});
    }
    if ((int)order.size() != n_far) return false;  // cycle: cannot happen
  }
  // ---- emit: global task table (flags, tracing) + one self-contained blob per CTA --------
  std::vector<int> qid(nl_all, -1);
  for (int k = 0; k < n_near; ++k) qid[k] = k;
  for (int i = 0; i < n_far; ++i) qid[order[i]] = n_near + i;
  std::vector<int> by_q(nl_all);
  for (int id = 0; id < nl_all; ++id) by_q[qid[id]] = id;
  for (int pos = 0; pos < nl_all; ++pos) {
    const LTask& l = lt[by_q[pos]];
    mp.tasks.push_back(Task{l.type, l.arg, 0, 0, 0, 0, 0});
  }
  std::vector<int> near_run_last(n_near, -1);  // last panel of the near CTA run holding k
  for (int c = 0; c < g_near; ++c)
    for (int k : lists[c]) near_run_last[k] = lists[c].back();
  mp.blob_slots = 0;
  for (auto& l : lists) {
    // [header][2 entry slots per task][dependency ranges][records]
    std::vector<int4> blob(1 + 2 * l.size(), int4{0, 0, 0, 0});
    blob[0] = int4{(int)l.size(), 0, 0, 0};
    for (size_t i = 0; i < l.size(); ++i) {
      const LTask& lk = lt[l[i]];
      std::vector<int> dq;
      for (int d : lk.deps) dq.push_back(qid[d < n_near ? near_run_last[d] : d]);
      const auto rg = to_ranges(dq);
      const int dep_off = (int)blob.size();
      for (size_t j = 0; j < rg.size(); j += 2) {
        int4 v{rg[j].lo, rg[j].hi, 0, 0};
        if (j + 1 < rg.size()) v.z = rg[j + 1].lo, v.w = rg[j + 1].hi;
        blob.push_back(v);
      }
      std::vector<int4> rec;
      rec_out = &rec;
      make_record(lk.type, lk.arg);
      const int rec_off = (int)blob.size();
      blob.insert(blob.end(), rec.begin(), rec.end());
      blob[1 + 2 * i] = int4{qid[l[i]], lk.type, rec_off, (int)rec.size()};
      // near panels publish completion only at the end of their CTA's run
      const bool publish = l[i] >= n_near || near_run_last[l[i]] == l[i];
      blob[2 + 2 * i] = int4{dep_off, (int)rg.size(), publish ? 1 : 0, 0};
    }
    if ((int)blob.size() > MEGA_BLOB_MAX) return false;
    mp.cta_lists.push_back({(int)mp.recs.size(), l.empty() ? 0 : (int)blob.size()});
    if (!l.empty()) mp.recs.insert(mp.recs.end(), blob.begin(), blob.end());
    mp.blob_slots = std::max(mp.blob_slots, (int)blob.size());
  }
  mp.est_makespan = fin.empty() ? 0.0 : *std::max_element(fin.begin(), fin.end());
  if (const char* path = getenv("H2B_DUMP_PLAN")) {  // profiling aid: the schedule as text
    if (FILE* f = fopen(path, "w")) {
      fprintf(f, "# flat %d splits", (int)mp.flat);
      for (int sp : splits) fprintf(f, " %d", sp);
      fprintf(f, "\n# qid type arg cta est_dur est_fin nlev : deps (queue ids)\n");
      std::vector<int> cta_of(nl_all, -1);
      for (size_t c = 0; c < lists.size(); ++c)
        for (int id : lists[c]) cta_of[id] = (int)c;
      for (int pos = 0; pos < nl_all; ++pos) {
        const int id = by_q[pos];
        const LTask& l = lt[id];
        fprintf(f, "%d %d %d %d %.2f %.2f %d :", pos, l.type, l.arg, cta_of[id], l.dur, fin[id],
                l.type == T_SPAN ? mp.prog.heads[l.arg].nlev : 0);
        for (int d : l.deps) fprintf(f, " %d", qid[d < n_near ? near_run_last[d] : d]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  if (getenv("H2B_VERIFY_PLAN")) {
    // self-check (debugging aid): every two tasks that touch the same x̂ / ŷ / y elements, one
    // of them writing, must be ordered by the schedule (CTA list order + dependency edges)
    struct Acc {
      int space;  // 0 x̂, 1 ŷ, 2 y, 3 y_deep
      int64_t lo, hi;
      bool w;
      int q;
    };
    std::vector<Acc> acc;
    for (int id = 0; id < nl_all; ++id) {
      const LTask& l = lt[id];
      const int q = qid[id];
      if (l.type == T_NEAR) {
        const int lf = ns == 32 || ns == 64 ? nts[l.arg].leaf_first : l.arg;
        const int nlf = ns == 32 || ns == 64 ? nts[l.arg].n_leaves : 1;
        const int rb = ns == 32 || ns == 64 ? mp.r * (256 / (ns / 2)) : 1 << 30;
        for (int li = lf; li < lf + nlf; ++li) {
          const int t = h->h_leaves[li];
          const int64_t r0 = (int64_t)h->c_start[t] + (ns == 32 || ns == 64 ? nts[l.arg].row0 : 0);
          acc.push_back({2, r0, std::min<int64_t>(r0 + rb, (int64_t)h->c_start[t] + h->c_size[t]), true, q});
        }
      } else if (l.type == T_SPAN) {
        const SpanHead& hd = mp.prog.heads[l.arg];
        int op_first = -1;
        for (int c = hd.copy_first; c < hd.copy_first + hd.n_copy; ++c) {
          const SpanCopy& cp = mp.prog.copies[c];
          if (cp.kind == SRC_XHAT || cp.kind == SRC_YHAT)
            acc.push_back({cp.kind == SRC_XHAT ? 0 : 1, cp.src, cp.src + cp.elems, false, q});
          if (cp.kind == SRC_OPS) op_first = (int)(cp.src / 2);
        }
        for (int c = hd.out_first; c < hd.out_first + hd.n_out; ++c) {
          const SpanCopy& cp = mp.prog.outs[c];
          acc.push_back({cp.kind == SRC_XHAT ? 0 : 1, cp.src, cp.src + cp.elems, true, q});
        }
        for (int o = op_first; o >= 0 && o < op_first + hd.n_ops; ++o) {
          const SpanOp& op = mp.prog.ops[o];
          if (op.flags & OP_OUT_Y)
            acc.push_back({(op.flags & OP_OUT_YD) ? 3 : 2, op.out, (int64_t)op.out + op.w, true, q});
        }
      } else if (l.type == T_FLAT_UP || l.type == T_FLAT_DOWN) {
        const FlatRec& f = mp.flat_recs[l.arg];
        if (l.type == T_FLAT_UP) {
          acc.push_back({0, f.hat_off, f.hat_off + f.k, true, q});
        } else {
          acc.push_back({1, f.hat_off, f.hat_off + f.k, false, q});
          acc.push_back({3, f.x_off, f.x_off + f.n, false, q});
        }
      } else {
        for (int t : group_members[l.arg]) {
          acc.push_back({1, h->c_xoff[t], h->c_xoff[t] + h->c_rank[t], true, q});
          for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
            const int sc = h->s_col[b];
            acc.push_back({0, h->c_xoff[sc], h->c_xoff[sc] + h->c_rank[sc], false, q});
          }
        }
      }
    }
    // happens-before closure over queue ids (every edge goes to a larger id)
    const int W = (nl_all + 63) / 64;
    std::vector<std::vector<uint64_t>> reach(nl_all, std::vector<uint64_t>(W, 0));
    std::vector<std::vector<int>> preds(nl_all);
    for (auto& l : lists)
      for (size_t i = 1; i < l.size(); ++i) preds[qid[l[i]]].push_back(qid[l[i - 1]]);
    for (int id = 0; id < nl_all; ++id)
      for (int d : lt[id].deps) preds[qid[id]].push_back(qid[d < n_near ? near_run_last[d] : d]);
    for (int v = 0; v < nl_all; ++v)
      for (int p : preds[v]) {
        for (int w = 0; w < W; ++w) reach[v][w] |= reach[p][w];
        reach[v][p / 64] |= 1ull << (p % 64);
      }
    auto before = [&](int a, int b) { return (reach[b][a / 64] >> (a % 64)) & 1ull; };
    int bad = 0;
    for (size_t i = 0; i < acc.size(); ++i) {
      if (!acc[i].w) continue;
      for (size_t j = 0; j < acc.size(); ++j) {
        const Acc &a = acc[i], &b = acc[j];
        if (i == j || a.space != b.space || a.q == b.q || b.hi <= a.lo || a.hi <= b.lo) continue;
        if (b.w && j < i) continue;  // write/write pairs once
        if (before(a.q, b.q) || before(b.q, a.q)) continue;
        if (++bad <= 20)
          fprintf(stderr, "plan check: unordered %s task %d (type %d arg %d) / %s task %d (type %d arg %d) on %s [%lld, %lld)\n",
                  "write", a.q, mp.tasks[a.q].type, mp.tasks[a.q].arg, b.w ? "write" : "read", b.q,
                  mp.tasks[b.q].type, mp.tasks[b.q].arg,
                  a.space == 0 ? "xhat" : a.space == 1 ? "yhat" : a.space == 2 ? "y" : "y_deep",
                  (long long)std::max(a.lo, b.lo), (long long)std::min(a.hi, b.hi));
      }
    }
    fprintf(stderr, "plan check: %d tasks, %zu accesses, %d unordered conflicts\n", nl_all, acc.size(), bad);
  }
  return true;
}

bool plan_per_level(const h2b_ctx* h, Plan& pl) {
  pl = Plan();
  pl.ls = -1;
  double cost = 0.0;
  bool ok = true;
  per_level(h, pl.prog, 0, h->depth, true, pl.up, cost, ok);
  per_level(h, pl.prog, 0, h->depth, false, pl.down_tail, cost, ok);
  pl.cost = cost;
  return ok;
}

}  // namespace

int h2b_prepare(h2b_ctx* h) {
  if (h->prepared) return H2B_OK;
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  int64_t acc = 0;
  const int P = h->P;
  // ---- Vᵀ, Tᵀ (out of place), Sᵀ (in place) --------------------------------
  std::vector<BlockDesc> vb, tbl, sb;
  for (int p = 0; p < P; ++p) {
    const int k = h->c_rank[p];
    if (k == 0) continue;
    if (h->c_child_lo[p] < 0)
      vb.push_back({h->c_voff[p], h->c_size[p], k});
    else if (m_of(h, p) > 0)
      tbl.push_back({h->c_toff[p], m_of(h, p), k});
  }
  int max_s = 0;
  for (int t = 0; t < P; ++t)
    for (int64_t b = h->s_row_ptr[t]; b < h->s_row_ptr[t + 1]; ++b) {
      const int kt = h->c_rank[t], ks = h->c_rank[h->s_col[b]];
      if (kt * ks == 0) continue;
      sb.push_back({h->s_off[b], kt, ks});
      max_s = std::max(max_s, kt * ks);
    }
  H2B_CUDA_TRY(cudaMalloc(&h->vT, 16 * (size_t)std::max<int64_t>(h->sec_elems[0], 2)));
  H2B_CUDA_TRY(cudaMalloc(&h->tT, 16 * (size_t)std::max<int64_t>(h->sec_elems[1], 2)));
  acc += 16 * (std::max<int64_t>(h->sec_elems[0], 2) + std::max<int64_t>(h->sec_elems[1], 2));
  BlockDesc* dbl = nullptr;
  const size_t nmax = std::max(vb.size(), std::max(tbl.size(), sb.size()));
  H2B_CUDA_TRY(cudaMalloc(&dbl, sizeof(BlockDesc) * std::max<size_t>(std::min<size_t>(nmax, 65535), 1)));
  auto run_list = [&](const std::vector<BlockDesc>& l, std::function<void(int)> launch) -> int {
    for (size_t i = 0; i < l.size(); i += 65535) {
      const int cnt = (int)std::min<size_t>(65535, l.size() - i);
      H2B_CUDA_TRY(cudaMemcpy(dbl, l.data() + i, sizeof(BlockDesc) * cnt, cudaMemcpyHostToDevice));
      launch(cnt);
      H2B_CHECK_LAUNCH();
      H2B_CUDA_TRY(cudaDeviceSynchronize());
    }
    return H2B_OK;
  };
  int rc = run_list(vb, [&](int c) { k_transpose_oop<<<c, 256>>>(dbl, h->buf[0], h->vT); });
  if (!rc) rc = run_list(tbl, [&](int c) { k_transpose_oop<<<c, 256>>>(dbl, h->buf[1], h->tT); });
  if (!rc && !sb.empty()) {
    if ((size_t)max_s * 16 <= (size_t)SMEM_CAP) {
      H2B_CUDA_TRY(cudaFuncSetAttribute(k_transpose_inplace, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SMEM_CAP));
      rc = run_list(sb, [&](int c) { k_transpose_inplace<<<c, 256, max_s * 16>>>(dbl, h->buf[2]); });
    } else {  // very large ranks: bounce through a temporary copy
      double2* tmp = nullptr;
      H2B_CUDA_TRY(cudaMalloc(&tmp, 16 * (size_t)h->sec_elems[2]));
      H2B_CUDA_TRY(cudaMemcpy(tmp, h->buf[2], 16 * (size_t)h->sec_elems[2], cudaMemcpyDeviceToDevice));
      rc = run_list(sb, [&](int c) { k_transpose_oop<<<c, 256>>>(dbl, tmp, h->buf[2]); });
      cudaFree(tmp);
    }
  }
  cudaFree(dbl);
  if (rc) return rc;
  // ---- coupling panel index and work items ------------------------------------
  std::vector<int64_t> prow(P + 1, 0);
  std::vector<int32_t> xcol, targets;
  std::vector<CoupleItem> citems;
  int64_t celems = 0;
  for (int t = 0; t < P; ++t) {
    prow[t] = (int64_t)xcol.size();
    const int kt = h->c_rank[t];
    if (kt == 0) continue;
    targets.push_back(t);
    const int64_t b0 = h->s_row_ptr[t], b1 = h->s_row_ptr[t + 1];
    for (int64_t b = b0; b < b1; ++b) {
      const int s = h->s_col[b];
      for (int j = 0; j < h->c_rank[s]; ++j) xcol.push_back((int32_t)(h->c_xoff[s] + j));
    }
    CoupleItem it{};
    it.panel = b1 > b0 ? h->s_off[b0] : 0;
    it.xcol = prow[t];
    it.out = h->c_xoff[t];
    it.R = (int32_t)((int64_t)xcol.size() - prow[t]);
    it.w = kt;
    celems += (int64_t)it.R * it.w;
    citems.push_back(it);
  }
  prow[P] = (int64_t)xcol.size();
  H2B_TRY(to_device(&h->s_prow, prow, &acc));
  H2B_TRY(to_device(&h->s_xcol, xcol, &acc));
  H2B_TRY(to_device(&h->couple_targets, targets, &acc));
  H2B_TRY(to_device(&h->couple_items, citems, &acc));
  h->n_couple_targets = (int)targets.size();
  h->n_couple_items = (int)citems.size();
  h->couple_warp_mode = (!citems.empty() && celems / (int64_t)citems.size() < 4096) ? 1 : 0;
  // ---- near-field work items (q = 1, uniform leaves of 32 or 64) ---------------
  h->near_rb = 0;
  const int ns = h->uniform_leaf;
  if (ns == 32 || ns == 64) {
    const double avg_blocks = (double)h->n_near / std::max(1, h->n_leaves);
    int R = 1;
    while (R < 4 && h2b_near_rows_per_item(ns, R) * ns * 16.0 * avg_blocks < 24e3) R *= 2;
    const int rb = h2b_near_rows_per_item(ns, R);
    std::vector<NearBlk> blks;
    std::vector<NearItem> items;
    for (int t : h->h_leaves) {
      const int64_t b0 = h->d_row_ptr[t], b1 = h->d_row_ptr[t + 1];
      const int first = (int)blks.size();
      for (int64_t b = b0; b < b1; ++b) blks.push_back({h->d_off[b], (int64_t)h->c_start[h->d_col[b]]});
      for (int r0 = 0; r0 < ns; r0 += rb)
        items.push_back({(int64_t)h->c_start[t] + r0, first, (int32_t)(b1 - b0), r0, 0});
    }
    H2B_TRY(to_device(&h->near_blks, blks, &acc));
    H2B_TRY(to_device(&h->near_items, items, &acc));
    h->n_near_items = (int)items.size();
    h->near_rb = rb;
  }
  // ---- q = 1 persistent single-launch task graph ----------------------------------------
  h->mega = 0;
  if (h->use_mega) {
    MegaPlan mp;
    int sms_est = 148;
    cudaDeviceGetAttribute(&sms_est, cudaDevAttrMultiProcessorCount, h->device);
    // far-field CTAs per SM (each with a smaller work area) vs one: more CTAs keep the many
    // short far-field tasks from queueing behind each other
    int far_per_sm = 1;
    if (const char* e = getenv("H2B_FAR_PER_SM")) far_per_sm = std::max(1, std::min(2, atoi(e)));
    int budget = far_per_sm == 1 ? MEGA_BUDGET : 3900;
    if (const char* e = getenv("H2B_MEGA_BUDGET")) budget = std::max(1000, std::min(MEGA_BUDGET_MAX, atoi(e)));
    if (plan_mega(h, citems, targets, far_per_sm * sms_est, budget, mp)) {
      H2B_TRY(to_device(&h->span_heads, mp.prog.heads, &acc));
      H2B_TRY(to_device(&h->span_copies, mp.prog.copies, &acc));
      H2B_TRY(to_device(&h->span_outs, mp.prog.outs, &acc));
      H2B_TRY(to_device(&h->span_ops, mp.prog.ops, &acc));
      H2B_TRY(to_device(&h->tasks, mp.tasks, &acc));
      H2B_TRY(to_device(&h->deps, mp.deps, &acc));
      H2B_TRY(to_device(&h->near_tasks, mp.near_tasks, &acc));
      H2B_TRY(to_device(&h->leaf_items, mp.leaf_items, &acc));
      H2B_TRY(to_device(&h->couple_groups, mp.groups, &acc));
      H2B_TRY(to_device(&h->rec_pool, mp.recs, &acc));
      H2B_TRY(to_device(&h->cta_lists, mp.cta_lists, &acc));
      H2B_TRY(to_device(&h->near_recs, mp.near_recs, &acc));
      H2B_TRY(to_device(&h->near_idx, mp.near_idx, &acc));
      h->n_near_tasks = (int)mp.near_idx.size();
      h->mega_flat = 0;
      if (mp.flat) {  // flattened bases W (and the deep spans' y_deep)
        std::vector<FlatLeaf> fl;
        std::vector<FlatStep> fst;
        int kmax = 1, nmax = 1;
        for (int p = 0; p < P; ++p) kmax = std::max(kmax, h->c_rank[p]);
        std::vector<int> parent(P, -1);
        for (int p = 0; p < P; ++p)
          if (h->c_child_lo[p] >= 0) parent[h->c_child_lo[p]] = parent[h->c_child_hi[p]] = p;
        for (int t : h->h_leaves) {
          int c = t;
          FlatLeaf L{h->c_voff[t], 0, h->c_size[t], h->c_rank[t], (int)fst.size(), 0};
          nmax = std::max(nmax, L.n);
          while (level_of(h, c) > mp.flat_level) {
            const int pp = parent[c];
            const bool hi = h->c_child_hi[pp] == c;
            const int64_t off = h->c_toff[pp] + (hi ? (int64_t)h->c_rank[h->c_child_lo[pp]] * h->c_rank[pp] : 0);
            fst.push_back(FlatStep{off, h->c_rank[c], h->c_rank[pp]});
            ++L.n_steps;
            c = pp;
          }
          int64_t w0 = -1;
          for (const FlatRec& r : mp.flat_recs)
            if (r.x_off == h->c_start[c]) w0 = r.w_off;
          L.w_off = w0 + (int64_t)(h->c_start[t] - h->c_start[c]) * h->c_rank[c];
          fl.push_back(L);
        }
        const int fsm = 2 * 16 * nmax * kmax;  // <= 200 KB (checked by the planner)
        {
          H2B_CUDA_TRY(cudaMalloc(&h->wbuf, 16 * std::max<int64_t>(mp.flat_elems, 1)));
          H2B_CUDA_TRY(cudaMalloc(&h->ydeep, 16 * std::max<int64_t>(h->n, 1)));
          acc += 16 * (mp.flat_elems + h->n);
          FlatLeaf* dl = nullptr;
          FlatStep* ds = nullptr;
          H2B_TRY(to_device(&dl, fl, nullptr));
          H2B_TRY(to_device(&ds, fst, nullptr));
          H2B_CUDA_TRY(cudaFuncSetAttribute(k_flatten, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm));
          k_flatten<<<(int)fl.size(), 256, fsm>>>(dl, ds, h->buf[H2B_SEC_V], h->buf[H2B_SEC_T], h->wbuf, kmax);
          H2B_CHECK_LAUNCH();
          H2B_CUDA_TRY(cudaDeviceSynchronize());
          cudaFree(dl);
          cudaFree(ds);
          h->mega_flat = 1;
        }
      }
      h->near_rec_max = mp.near_rec_max;
      h->mega_blob_slots = mp.blob_slots;
      {  // far-field operands that may be warmed into L2 at launch (64 KB pieces; off by default)
        std::vector<int4> pf;
        auto add = [&](const void* p, int64_t bytes) {
          for (int64_t o = 0; o < bytes; o += 65536) {
            const uint64_t a = (uint64_t)p + o;
            pf.push_back(int4{(int)(uint32_t)a, (int)(uint32_t)(a >> 32),
                              (int)std::min<int64_t>(65536, bytes - o), 0});
          }
        };
        add(h->buf[H2B_SEC_V], 16 * h->sec_elems[0]);
        add(h->buf[H2B_SEC_T], 16 * h->sec_elems[1]);
        add(h->vT, 16 * h->sec_elems[0]);
        add(h->tT, 16 * h->sec_elems[1]);
        add(h->buf[H2B_SEC_S], 16 * h->sec_elems[2]);
        add(h->s_xcol, 4 * (int64_t)xcol.size() / 16 * 16);
        H2B_TRY(to_device(&h->l2_prefetch, pf, &acc));
        h->n_prefetch = (int)pf.size();
      }
      if (!mp.citems.empty()) {  // grouped order of the coupling work items
        cudaFree(h->couple_items);
        h->couple_items = nullptr;
        H2B_TRY(to_device(&h->couple_items, mp.citems, &acc));
      }
      H2B_CUDA_TRY(cudaMalloc(&h->ctrl, sizeof(MegaCtrl)));
      H2B_CUDA_TRY(cudaMemset(h->ctrl, 0, sizeof(MegaCtrl)));
      H2B_CUDA_TRY(cudaMalloc(&h->flags, sizeof(uint32_t) * std::max<size_t>(mp.tasks.size(), 1)));
      H2B_CUDA_TRY(cudaMemset(h->flags, 0, sizeof(uint32_t) * std::max<size_t>(mp.tasks.size(), 1)));
      h->n_tasks = (int)mp.tasks.size();
      h->h_tasks = mp.tasks;
      h->mega_ns = mp.ns;
      h->mega_r = mp.r;
      h->mega_tiers = mp.tiers;
      int sms = 0;
      H2B_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
      // far-field task graph: one CTA per SM, all co-resident (they wait on one another)
      h->mega_smem = std::max(mp.smem, 16);
      h->mega_grid = (int)mp.cta_lists.size();
      const int far_bytes = h->mega_smem + 16 * h->mega_blob_slots;
      H2B_TRY(h2b_mega_set_smem(0, 0, 16 * (std::max(budget, MEGA_BUDGET) + MEGA_BLOB_MAX)));
      int per_sm = 1;
      if (h->mega_grid > 0) H2B_TRY(h2b_mega_occupancy(0, 0, far_bytes, &per_sm));
      // near-field stream: one CTA per SM beside the far-field CTA, ring in the shared memory left
      int near_static = 0;
      H2B_TRY(h2b_near_stream_static_smem(mp.ns, mp.r, &near_static));
      const int sm_total = 233472 - 2048;  // per SM, minus the per-CTA reservations of both kernels
      const int far_total = h->mega_grid > 0 ? far_per_sm * (far_bytes + h2b_mega_static_smem() + 1024) : 0;
      const int rec_bytes = NEAR_NRB * 16 * std::max(1, mp.near_rec_max);  // NRB record buffers
      const int stg = mp.ns > 0 ? 16 * (mp.r * (256 / (mp.ns / 2)) * mp.ns + mp.ns) : 0;
      int nst = stg > 0 ? std::min(8, (sm_total - far_total - near_static - rec_bytes) / stg) : 0;
      if (const char* e = getenv("H2B_DEBUG_NEAR_NST")) nst = std::min(nst, std::max(2, atoi(e)));  // tuning aid
      if (mp.ns > 0 && nst < 2) nst = 2;  // still correct; the two kernels then share SMs less well
      h->near_nst = nst;
      h->near_smem = nst * stg + rec_bytes;
      // the attribute is per kernel and process-wide: set the maximum, never a per-handle size
      H2B_TRY(h2b_near_stream_set_smem(mp.ns, mp.r, 232448 - near_static));
      h->near_grid = sms;
      if (const char* e = getenv("H2B_DEBUG_NEAR_DELAY_NS")) h->near_delay_ns = (uint32_t)std::max(0, atoi(e));  // tuning aid
      // near tasks split statically over the CTAs: no claim atomics on the producer's path
      // (measured 32.8 vs 34.8 us for the cfg2 near field alone, step 45.6 vs 46.3 us)
      h->near_static = 1;
      if (const char* e = getenv("H2B_NEAR_STATIC")) h->near_static = atoi(e) ? 1 : 0;  // tuning aid
      if (const char* e = getenv("H2B_NEAR_DBG")) h->near_dbg = atoi(e);  // profiling only
      if (const char* e = getenv("H2B_NEAR_GRID")) h->near_grid = std::max(1, std::min(NEAR_MAXG, atoi(e)));  // tuning aid
      // each CTA's first record and first block (static split): kernel parameters
      auto near_cta_tables = [&]() {  // (again below when the tree plan changes the grid)
      h->near_early = 0;
      auto leaf_has_near = [&](int t) { return h->d_row_ptr[t + 1] > h->d_row_ptr[t]; };
      h->near_first_rec.assign(h->near_grid, int2{0, 0});
      h->near_first_blk.assign(h->near_grid, longlong2{0, 0});
      if (mp.ns > 0 && h->near_grid <= NEAR_MAXG && !getenv("H2B_NEAR_NO_EARLY")) {
        const int nt = (int)mp.near_idx.size();
        for (int c = 0; c < h->near_grid; ++c) {
          const int t = (int)((int64_t)c * nt / h->near_grid);
          if (t >= (int)((int64_t)(c + 1) * nt / h->near_grid)) continue;  // no task
          const int2 ix = mp.near_idx[t];
          const int4 head = mp.near_recs[ix.x];
          const int4 b0 = mp.near_recs[ix.x + 1 + head.y];  // {D offset, x offset} as two int64
          h->near_first_rec[c] = ix;
          h->near_first_blk[c] = longlong2{(long long)(uint32_t)b0.x | ((long long)b0.y << 32),
                                           (long long)(uint32_t)b0.z | ((long long)b0.w << 32)};
        }
        h->near_early = 1;
      }
      // rows of y per CTA of the static split (tasks are in row order: whole leaves, or row
      // slices of one leaf): valid when the ranges tile [0, n)
      h->near_zero_ok = 0;
      h->near_zero_row.assign(h->near_grid, int2{0, 0});
      if (h->near_static && mp.ns > 0 && h->near_grid <= NEAR_MAXG && h->n < (int64_t)1 << 31 &&
          mp.near_tasks.size() == mp.near_idx.size()) {
        const int nt = (int)mp.near_tasks.size();
        const int rb = mp.r * (256 / (mp.ns / 2));
        int64_t next = 0;
        bool ok = true;
        for (int c = 0; c < h->near_grid && ok; ++c) {
          const int t0 = (int)((int64_t)c * nt / h->near_grid), t1 = (int)((int64_t)(c + 1) * nt / h->near_grid);
          int64_t first = next;
          for (int t = t0; t < t1 && ok; ++t) {
            const NearTask& k = mp.near_tasks[t];
            for (int i = 0; i < k.n_leaves && ok; ++i) {
              const int leaf = h->h_leaves[k.leaf_first + i];
              const bool sliced = rb < mp.ns;
              const int64_t a = h->c_start[leaf] + (sliced ? k.row0 : 0);
              const int64_t b = sliced ? a + rb : a + h->c_size[leaf];
              ok = a == next && leaf_has_near(leaf);
              next = b;
            }
          }
          h->near_zero_row[c] = int2{(int)first, (int)(next - first)};
        }
        h->near_zero_ok = ok && next == h->n ? 1 : 0;
      }
      };
      near_cta_tables();
      if (getenv("H2B_NEAR_TRACE") && !h->near_trace) {  // development aid (h2b_near_trace)
        H2B_CUDA_TRY(cudaMalloc(&h->near_trace, sizeof(uint64_t) * 24 * std::max(sms, NEAR_MAXG)));
        H2B_CUDA_TRY(cudaMemset(h->near_trace, 0, sizeof(uint64_t) * 24 * std::max(sms, NEAR_MAXG)));
      }
      h->mega = (per_sm > 0 && h->mega_grid <= per_sm * sms) ? 1 : 0;
      h->mega_est_us = mp.est_makespan;
      // far field as subtree programs (h2b_tree.cu) when the tree qualifies: it takes k_mega's
      // place beside the near-field stream, whose ring gets the shared memory left over
      int planned = 0;
      int64_t tb = 0;
      if (h->mega && h->use_tree) H2B_TRY(h2b_tree_prepare(h, sms, TREE_BUDGET, &tb, &planned));
      if (planned) {
        acc += tb;
        // one more near-field CTA on every SM without a program: a program's 174 KB leave room
        // for exactly one near-field CTA beside it, so the extra CTAs can only land on the free
        // SMs, which then stream with two consumer chains (cfg2: 168 CTAs, the near CTAs' last
        // exit 31.9 -> 30.8 us in the step)
        if (!getenv("H2B_NEAR_GRID") && mp.ns > 0 && h->near_static) {
          const int extra = std::max(0, sms - h->tree_progs);
          if (extra > 0 && sms + extra <= NEAR_MAXG) {
            h->near_grid = sms + extra;
            near_cta_tables();
          }
        }
        H2B_TRY(h2b_tree_prepare_zero(h, h->tree));
        const int tree_total = h->tree_smem + h2b_tree_static_smem() + 1024;
        int tnst = stg > 0 ? std::min(8, (sm_total - tree_total - near_static - rec_bytes) / stg) : 0;
        if (const char* e = getenv("H2B_DEBUG_NEAR_NST")) tnst = std::min(tnst, std::max(2, atoi(e)));
        if (mp.ns > 0 && tnst < 2) tnst = 2;
        h->near_nst = tnst;
        h->near_smem = tnst * stg + rec_bytes;
      }
      // both kernels must fit one SM's register file per scheduler (warp w runs on scheduler
      // w % 4: 3 of the near kernel's 9 warps share scheduler 0 with 2 far warps); otherwise
      // the near CTAs wait for the far kernel to exit (correct, but the step nearly doubles)
      if (h->near_grid > 0) {
        auto warp_regs = [](int regs) { return ((regs + 7) / 8 * 8) * 32; };
        const int far_regs = planned ? h2b_tree_regs() : h2b_mega_regs();
        const int need = 3 * warp_regs(h2b_near_stream_regs(mp.ns, mp.r)) + 2 * warp_regs(far_regs);
        if (need > 16384) {
          static bool warned = false;
          if (!warned)
            fprintf(stderr, "h2b: near-field and far-field kernels exceed a scheduler's registers (%d > 16384): "
                            "they will not run concurrently\n", need);
          warned = true;
        }
      }
    }
  }
  if (h->mega) {  // the multi-kernel programs below are still planned for phase timing
    h->device_bytes += acc;
    acc = 0;
  }
  // ---- q = 1 far-field schedule ---------------------------------------------------
  h->span_mode = 0;
  if (h->K > 0 && !h->mega) {
    Plan best;
    int min_leaf_level = h->depth;
    for (int l = 0; l < h->depth; ++l)
      for (int p = h->level_ptr[l]; p < h->level_ptr[l + 1]; ++p)
        if (h->c_child_lo[p] < 0) min_leaf_level = std::min(min_leaf_level, l);
    for (int ls = 0; ls <= std::min(min_leaf_level, h->depth - 1); ++ls) {
      Plan pl;
      if (plan_with_split(h, ls, pl) && pl.cost < best.cost) best = std::move(pl);
    }
    {
      Plan pl;
      if (plan_per_level(h, pl) && pl.cost < best.cost) best = std::move(pl);
    }
    if (best.cost < 1e29) {
      h->span_mode = 1;
      h->ls = best.ls;
      h->top_staged = best.top_staged;
      h->up_prog = best.up;
      h->down_prog_head = best.down_head;
      h->down_prog_tail = best.down_tail;
      H2B_TRY(to_device(&h->span_heads, best.prog.heads, &acc));
      H2B_TRY(to_device(&h->span_copies, best.prog.copies, &acc));
      H2B_TRY(to_device(&h->span_outs, best.prog.outs, &acc));
      H2B_TRY(to_device(&h->span_ops, best.prog.ops, &acc));
      H2B_TRY(h2b_far_init_attributes(16 * SPAN_BUDGET));
    }
  }
  // ---- streams ------------------------------------------------------------------
  int lo_prio = 0, hi_prio = 0;
  H2B_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  H2B_CUDA_TRY(cudaStreamCreateWithPriority(&h->far_stream, cudaStreamNonBlocking, hi_prio));
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  H2B_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  h->device_bytes += acc;
  h->prepared = true;
  return H2B_OK;
}
