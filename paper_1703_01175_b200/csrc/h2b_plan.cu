// One-time preparation of an uploaded operator (host side + layout kernels):
//   * Vᵀ, Tᵀ copies and in-place Sᵀ (the panel layout of h2b_panel.cuh)
//   * coupling panel index (x̂ row feeding every panel row) and work items
//   * near-field work items (rows-per-CTA chosen from the block statistics)
//   * the q = 1 far-field schedule: span programs (h2b_common.cuh) chosen by
//     a small cost model over the split level `ls`.
#include <algorithm>
#include <functional>

#include "h2b_common.cuh"

int h2b_far_init_attributes(int smem_cap_bytes);
int h2b_near_rows_per_item(int ns, int r);

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
    if (e > 0) cp.push_back({src, kind, (int32_t)e, o, 0});
    return o;
  }
  void outc(int kind, int64_t dst, int64_t e, int o) {
    if (e > 0) out.push_back({dst, kind, (int32_t)e, o, 0});
  }
  void level() { lv.emplace_back(); }
  void op(int pay, int in_, int out_, int R, int w, int flags) {
    lv.back().push_back(SpanOp{pay, in_, out_, R, w, flags, 0, 0});
  }
};

// append a finished span; returns false when it does not fit
bool finish(Prog& P, SB& s, int* smem_out) {
  int n_ops = 0;
  for (auto& l : s.lv) n_ops += (int)l.size();
  if ((int)s.lv.size() > SPAN_MAXLEV) return false;
  const int op_first = (int)P.ops.size();
  const int ops_smem = s.in(SRC_OPS, 2 * (int64_t)op_first, 2 * (int64_t)n_ops);
  if (s.smem > SPAN_BUDGET) return false;
  SpanHead hd{};
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
bool build_subtree_span(const h2b_ctx* h, Prog& P, int r, int nl, bool up, bool input_last,
                        int* smem_max) {
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
      xh[i] = s.in(SRC_YHAT, xb, xe);
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
          s.op(pay, out_here, h->c_start[p], k, h->c_size[p], OP_ACC | OP_OUT_Y);
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
  if (up)
    for (int i = ncomp - 1; i >= 0; --i) emit_level(i);
  else
    for (int i = 0; i < ncomp; ++i) emit_level(i);
  if (up) {
    for (int i = 0; i < ncomp; ++i)
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
  // ---- q = 1 far-field schedule ---------------------------------------------------
  h->span_mode = 0;
  if (h->K > 0) {
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
