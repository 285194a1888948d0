// Per-subsystem kernels behind the per-op C-ABI entry points (unit parity of
// the pieces the iteration kernel fuses; see include/vfpi.h).
#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

inline int nblk(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// apply_jc (contacts.py:402-411)
__global__ void k_apply_jc(int64_t n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                           const double* __restrict__ fr, const double* __restrict__ v, double* __restrict__ eta) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  const int i = ci[m], j = cj[m];
  double rel[3], e[3];
  for (int t = 0; t < 3; ++t) rel[t] = (j >= 0) ? dsub(v[i + t], v[j + t]) : v[i + t];
  frame_apply(fr + 9 * m, rel, e);
  for (int t = 0; t < 3; ++t) eta[3 * m + t] = e[t];
}

// apply_jc_t (contacts.py:414-423), unique columns: plain stores
__global__ void k_apply_jc_t(int64_t n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                             const double* __restrict__ fr, const double* __restrict__ lam, double* __restrict__ out) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  const int i = ci[m], j = cj[m];
  double l[3], w[3];
  for (int t = 0; t < 3; ++t) l[t] = lam[3 * m + t];
  frame_apply_t(fr + 9 * m, l, w);
  for (int t = 0; t < 3; ++t) out[i + t] = dadd(0.0, w[t]);
  if (j >= 0)
    for (int t = 0; t < 3; ++t) out[j + t] = dsub(0.0, w[t]);
}

// overlapping columns: np.add.at then np.subtract.at in contact order, one thread
__global__ void k_apply_jc_t_ordered(int64_t n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                                     const double* __restrict__ fr, const double* __restrict__ lam,
                                     double* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t m = 0; m < n_c; ++m) {
    double l[3], w[3];
    for (int t = 0; t < 3; ++t) l[t] = lam[3 * m + t];
    frame_apply_t(fr + 9 * m, l, w);
    for (int t = 0; t < 3; ++t) out[ci[m] + t] = dadd(out[ci[m] + t], w[t]);
  }
  for (int64_t m = 0; m < n_c; ++m) {
    if (cj[m] < 0) continue;
    double l[3], w[3];
    for (int t = 0; t < 3; ++t) l[t] = lam[3 * m + t];
    frame_apply_t(fr + 9 * m, l, w);
    for (int t = 0; t < 3; ++t) out[cj[m] + t] = dsub(out[cj[m] + t], w[t]);
  }
}

// contact_solve_oneshot (solver.py:262-281)
__global__ void k_oneshot(int64_t n_c, const double* __restrict__ gamma, const double* __restrict__ eta,
                          const double* __restrict__ phi, const double* __restrict__ mu,
                          const double* __restrict__ mu2, int op, double* __restrict__ lam) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  double e[3], l[3];
  for (int t = 0; t < 3; ++t) e[t] = eta[3 * m + t];
  trial_impulse(e, phi[m], gamma[m], l);
  project(op, l, mu[m], mu2[m]);
  for (int t = 0; t < 3; ++t) lam[3 * m + t] = l[t];
}

// scc_residual (solver.py:304-334)
__global__ void k_scc(int64_t n_c, const double* __restrict__ vc, const double* __restrict__ lam,
                      const double* __restrict__ phi, const double* __restrict__ mu, double* __restrict__ out) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  out[m] = scc_one(vc + 3 * m, lam + 3 * m, phi[m], mu[m]);
}

// y_i = sum over row i's numeric entries in increasing column order (sparse.py:97-102)
__global__ void k_spmv_rows(int64_t n, const int64_t* __restrict__ row_ptr, const int* __restrict__ perm,
                            const int* __restrict__ colof, const double* __restrict__ data,
                            const double* __restrict__ x, double* __restrict__ y) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double acc = 0.0;
  for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
    const int e = perm[k];
    acc = dadd(acc, dmul(data[e], x[colof[e]]));
  }
  y[r] = acc;
}

__global__ void k_const(double* p, double v, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}

}  // namespace

void launch_apply_jc(int64_t n_c, const int* ci, const int* cj, const double* fr, const double* v, double* eta,
                     cudaStream_t st) {
  if (n_c > 0) k_apply_jc<<<nblk(n_c), 256, 0, st>>>(n_c, ci, cj, fr, v, eta);
}

void launch_apply_jc_t(int64_t n, int64_t n_c, const int* ci, const int* cj, const double* fr, const double* lam,
                       double* out, bool overlap, cudaStream_t st) {
  cudaMemsetAsync(out, 0, 8 * (size_t)n, st);
  if (n_c <= 0) return;
  if (overlap) k_apply_jc_t_ordered<<<1, 1, 0, st>>>(n_c, ci, cj, fr, lam, out);
  else k_apply_jc_t<<<nblk(n_c), 256, 0, st>>>(n_c, ci, cj, fr, lam, out);
}

void launch_oneshot(int64_t n_c, const double* gamma, const double* eta, const double* phi, const double* mu,
                    const double* mu2, int op, double* lam, cudaStream_t st) {
  if (n_c > 0) k_oneshot<<<nblk(n_c), 256, 0, st>>>(n_c, gamma, eta, phi, mu, mu2, op, lam);
}

void launch_scc(int64_t n_c, const double* vc, const double* lam, const double* phi, const double* mu, double* out,
                cudaStream_t st) {
  if (n_c > 0) k_scc<<<nblk(n_c), 256, 0, st>>>(n_c, vc, lam, phi, mu, out);
}

void launch_spmv_csr_rows(int64_t n, const int64_t* row_ptr, const int* perm, const int* colof, const double* data,
                          const double* x, double* y, cudaStream_t st) {
  if (n > 0) k_spmv_rows<<<nblk(n), 256, 0, st>>>(n, row_ptr, perm, colof, data, x, y);
}

void launch_const_fill(double* p, double v, int64_t n, cudaStream_t st) {
  if (n > 0) k_const<<<nblk(n), 256, 0, st>>>(p, v, n);
}

}  // namespace vfpi
