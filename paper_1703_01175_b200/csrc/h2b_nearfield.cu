// Near-field payload generated on the device from the voxel geometry.
//
// The near-field blocks are plain samples of the system matrix, so instead of
// uploading them (5.45 GB at BASELINE cfg3, 113 GB at cfg4) the handle can
// assemble them in HBM directly.  Restates the reference block sampler
//   assemble_block_raw   /root/reference/pkg/src/h2vie/_kernel_core.pyx:13-47
//     S[m, n] = 1 - chi_n * diag                       m == n
//             = -chi_n * (amp cos(k0 r) - j amp sin(k0 r)),  amp = k0^2 V / (4 pi r)
// with diag = k0^2 * self_term(V, k0) (kernel.py:170-187, computed by the host), for every
// inadmissible pair in the packed CSR order (build.py:321-324).  Values agree with the
// reference's libm path to a few ulp (CUDA's sin/cos/sqrt are within 1-2 ulp).
#include "h2b_common.cuh"

namespace {

constexpr int NF_THREADS = 256;

__global__ void __launch_bounds__(NF_THREADS) k_assemble_near(
    const int32_t* __restrict__ leaves, const int32_t* __restrict__ c_start,
    const int32_t* __restrict__ c_size, const int64_t* __restrict__ d_row_ptr,
    const int32_t* __restrict__ d_col, const int64_t* __restrict__ d_off,
    const int64_t* __restrict__ perm, const double* __restrict__ centers,
    const double2* __restrict__ chi, double k0, double coef, double2 diag, double2* __restrict__ dbuf,
    unsigned long long* bad) {
  const int t = leaves[blockIdx.x];
  const int nt = c_size[t];
  const int64_t t0 = c_start[t];
  for (int64_t b = d_row_ptr[t]; b < d_row_ptr[t + 1]; ++b) {
    const int s = d_col[b];
    const int ns = c_size[s];
    const int64_t s0 = c_start[s];
    double2* out = dbuf + d_off[b];
    for (int e = threadIdx.x; e < nt * ns; e += NF_THREADS) {
      const int i = e / ns, j = e - i * ns;
      const int64_t m = perm[t0 + i], n = perm[s0 + j];
      const double2 cn = chi[n];
      double2 v;
      if (m == n) {
        v = make_double2(1.0 - (cn.x * diag.x - cn.y * diag.y), -(cn.x * diag.y + cn.y * diag.x));
      } else {
        const double dx = centers[3 * m] - centers[3 * n];
        const double dy = centers[3 * m + 1] - centers[3 * n + 1];
        const double dz = centers[3 * m + 2] - centers[3 * n + 2];
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        if (r == 0.0) {
          atomicMin(bad, (unsigned long long)(b << 20) | (unsigned long long)e);
          v = make_double2(0.0, 0.0);
        } else {
          const double amp = coef / r;
          double sn, cs;
          sincos(k0 * r, &sn, &cs);
          const double ar = amp * cs, ai = -(amp * sn);  // amp e^{-j k0 r}
          v = make_double2(-(cn.x * ar - cn.y * ai), -(cn.x * ai + cn.y * ar));
        }
      }
      out[e] = v;
    }
  }
}

}  // namespace

int h2b_assemble_near(h2b_handle h, const double* centers, const double* chi, double k0, double volume,
                      double diag_re, double diag_im) {
  if (!h || !centers || !chi || !(volume > 0.0) || k0 < 0.0) {
    h2b_set_error("h2b_assemble_near: bad arguments");
    return H2B_EINVAL;
  }
  if (h->prepared) {
    h2b_set_error("h2b_assemble_near: payload is immutable after the first matvec");
    return H2B_ESTATE;
  }
  H2B_CUDA_TRY(cudaSetDevice(h->device));
  double* cd = nullptr;
  double2* xd = nullptr;
  unsigned long long* bad = nullptr;
  const unsigned long long none = ~0ull;
  H2B_CUDA_TRY(cudaMalloc(&cd, 24 * (size_t)h->n));
  H2B_CUDA_TRY(cudaMalloc(&xd, 16 * (size_t)h->n));
  H2B_CUDA_TRY(cudaMalloc(&bad, sizeof(unsigned long long)));
  H2B_CUDA_TRY(cudaMemcpy(cd, centers, 24 * (size_t)h->n, cudaMemcpyHostToDevice));
  H2B_CUDA_TRY(cudaMemcpy(xd, chi, 16 * (size_t)h->n, cudaMemcpyHostToDevice));
  H2B_CUDA_TRY(cudaMemcpy(bad, &none, sizeof(none), cudaMemcpyHostToDevice));
  const double coef = k0 * k0 * volume / 12.566370614359172953850573533118;
  k_assemble_near<<<h->n_leaves, NF_THREADS>>>(h->leaves, h->c_start_d, h->c_size_d, h->d_row_ptr_d,
                                                h->d_col_d, h->d_off_d, h->perm, cd, xd, k0, coef,
                                                make_double2(diag_re, diag_im), h->buf[H2B_SEC_D], bad);
  H2B_CHECK_LAUNCH();
  unsigned long long first = none;
  H2B_CUDA_TRY(cudaMemcpy(&first, bad, sizeof(first), cudaMemcpyDeviceToHost));
  cudaFree(cd);
  cudaFree(xd);
  cudaFree(bad);
  if (first != none) {
    h2b_set_error("h2b_assemble_near: coincident voxel centres in near-field block " +
                  std::to_string(first >> 20) + " (kernel singular; reference raises CoincidentCentersError)");
    return H2B_EINVAL;
  }
  h->sec_iv[H2B_SEC_D].clear();
  h->sec_iv[H2B_SEC_D].emplace(0, h->sec_elems[H2B_SEC_D]);
  h->sec_uploaded[H2B_SEC_D] = h->sec_elems[H2B_SEC_D];
  return H2B_OK;
}

// ===========================================================================
// Exact rows of the system matrix times a vector, summed directly over all N columns (entries
// sampled from the geometry as above, self term included): the reference for the device-built
// operators that the reference builder cannot produce (BASELINE cfg4/cfg5).  One CTA per row.
// ===========================================================================
namespace {
__global__ void __launch_bounds__(256) k_exact_rows(const int64_t* __restrict__ rows, int64_t n,
                                                    const double* __restrict__ centers,
                                                    const double2* __restrict__ chi, double k0, double coef,
                                                    double2 diag, const double2* __restrict__ x,
                                                    double2* __restrict__ out) {
  __shared__ double2 red[256];
  const int64_t m = rows[blockIdx.x];
  const double mx = centers[3 * m], my = centers[3 * m + 1], mz = centers[3 * m + 2];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t j = threadIdx.x; j < n; j += 256) {
    const double2 cn = chi[j];
    double2 v;
    if (j == m) {
      v = make_double2(1.0 - (cn.x * diag.x - cn.y * diag.y), -(cn.x * diag.y + cn.y * diag.x));
    } else {
      const double dx = mx - centers[3 * j], dy = my - centers[3 * j + 1], dz = mz - centers[3 * j + 2];
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double amp = coef / r;
      double sn, cs;
      sincos(k0 * r, &sn, &cs);
      const double ar = amp * cs, ai = -(amp * sn);
      v = make_double2(-(cn.x * ar - cn.y * ai), -(cn.x * ai + cn.y * ar));
    }
    cfma(acc, v, x[j]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}
}  // namespace

// out[i] = Σ_j S[rows[i], j] x[j] (original point order, host arrays in and out)
extern "C" int h2b_exact_rows(const int64_t* rows, int nrows, int64_t n, const double* centers, const void* chi,
                              double k0, double volume, double diag_re, double diag_im, const void* x, void* out,
                              int device) {
  if (!rows || !centers || !chi || !x || !out || nrows < 1 || n < 1) {
    h2b_set_error("h2b_exact_rows: bad arguments");
    return H2B_EINVAL;
  }
  H2B_CUDA_TRY(cudaSetDevice(device));
  int64_t* dr = nullptr;
  double* dc = nullptr;
  double2 *dchi = nullptr, *dx = nullptr, *dout = nullptr;
  auto fin = [&](int rc) {
    void* ptrs[] = {dr, dc, dchi, dx, dout};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    return rc;
  };
  if (cudaMalloc(&dr, 8 * (size_t)nrows) != cudaSuccess || cudaMalloc(&dc, 24 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&dchi, 16 * (size_t)n) != cudaSuccess || cudaMalloc(&dx, 16 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&dout, 16 * (size_t)nrows) != cudaSuccess) {
    cudaGetLastError();
    h2b_set_error("h2b_exact_rows: allocation failed");
    return fin(H2B_ENOMEM);
  }
  cudaMemcpy(dr, rows, 8 * (size_t)nrows, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, centers, 24 * (size_t)n, cudaMemcpyHostToDevice);
  cudaMemcpy(dchi, chi, 16 * (size_t)n, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x, 16 * (size_t)n, cudaMemcpyHostToDevice);
  const double coef = k0 * k0 * volume / (4.0 * 3.14159265358979323846);
  k_exact_rows<<<nrows, 256>>>(dr, n, dc, dchi, k0, coef, make_double2(diag_re, diag_im), dx, dout);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, 16 * (size_t)nrows, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    h2b_set_error(std::string("h2b_exact_rows: ") + cudaGetErrorString(e));
    return fin(H2B_ECUDA);
  }
  return fin(H2B_OK);
}
