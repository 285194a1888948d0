// Contact-free fallback step of a diverged V-FPI solve on the device.
//
// The reference harness (harness.py:586-593) answers a DivergenceError with a
// flagged zero-impulse step: v_hat = scipy.sparse.linalg.cg(A, b,
// rtol=1e-10, maxiter=10 n) on the contact-free system, padded with zeros for
// the virtual rows, lam = 0. This is that conjugate-gradient solve (scipy's
// unpreconditioned recurrence, x0 = 0: stop when ||r|| < rtol ||b||, checked
// before each iteration; ||b|| = 0 returns b) in two shapes:
//   * one CTA per scene of a block-diagonal batch (FEM batches: only the
//     diverged scenes are launched), CTA barriers only;
//   * one system over a cooperative grid (single large systems), grid barriers.
// Rows are read from A's CSC arrays (column i as row i: A is symmetric up to
// the assembly's last-bit asymmetry, far below the CG tolerance). Dot products
// are reduced in a fixed order, so the result is deterministic run to run; it
// is tolerance-equal to scipy's (whose dots are BLAS-order dependent), which is
// the same bar the reference's own fallback meets across hosts.
#include <cooperative_groups.h>

#include "vfpi_internal.cuh"

namespace vfpi {

namespace {

namespace cgr = cooperative_groups;

constexpr int kCgThreads = 512;

struct CgArgs {
  const int32_t* indptr;
  const int32_t* indices;
  const double* data;
  const double* b;
  double* x;
  double* r;
  double* p;
  double* q;
  double* partial;     // [2][G] (grid mode)
  int32_t* iters_out;  // per scene (scene mode) or [1] (grid mode)
  const int32_t* scene_list;
  const SolveStatus* status;  // scene mode without a list: CTA b runs iff scene b diverged
  const int* cts;             //   its contacts' impulses [cts[b], cts[b+1]) are zeroed
  double* lam;
  int64_t n;           // rows per scene (scene mode) / of the system (grid mode)
  double rtol;
  int64_t maxiter;
};

// Block-wide sum in a fixed order (warp shuffle tree, then warps in order);
// every thread returns the total.
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

template <bool GRID>
__device__ double all_sum(double v, double* sh, double* partial) {
  const double s = block_sum(v, sh);
  if (!GRID) return s;
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
  cgr::this_grid().sync();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int g = 0; g < (int)gridDim.x; ++g) t += partial[g];
    sh[33] = t;
  }
  __syncthreads();
  return sh[33];
}

template <bool GRID>
__device__ void all_sync() {
  if (GRID) cgr::this_grid().sync();
  else __syncthreads();
}

template <bool GRID>
__global__ void __launch_bounds__(kCgThreads) k_cg(CgArgs a) {
  __shared__ double sh[34];
  int64_t lo, hi;
  double* part0 = a.partial;
  double* part1 = a.partial ? a.partial + gridDim.x : nullptr;
  if (GRID) {
    lo = a.n * blockIdx.x / gridDim.x;
    hi = a.n * (blockIdx.x + 1) / gridDim.x;
  } else if (a.scene_list) {
    lo = (int64_t)a.scene_list[blockIdx.x] * a.n;
    hi = lo + a.n;
  } else {  // device-driven: every scene's CTA checks its own status
    if (!a.status[blockIdx.x].diverged) return;
    lo = (int64_t)blockIdx.x * a.n;
    hi = lo + a.n;
    for (int64_t t = 3 * (int64_t)a.cts[blockIdx.x] + threadIdx.x; t < 3 * (int64_t)a.cts[blockIdx.x + 1];
         t += blockDim.x)
      a.lam[t] = 0.0;
  }
  const double* b = a.b;
  double *x = a.x, *r = a.r, *p = a.p, *q = a.q;
  double rr = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double bi = b[i];
    r[i] = bi;
    x[i] = 0.0;
    rr += bi * bi;
  }
  rr = all_sum<GRID>(rr, sh, part1);
  const double bnrm = sqrt(rr);
  int64_t it = 0;
  if (bnrm == 0.0) {
    // scipy returns b itself (zero here) -- x already holds it
  } else {
    const double atol = a.rtol * bnrm;
    double rho_prev = 1.0;
    for (; it < a.maxiter; ++it) {
      if (sqrt(rr) < atol) break;
      const double rho = rr;
      const double beta = it > 0 ? rho / rho_prev : 0.0;
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = it > 0 ? r[i] + beta * p[i] : r[i];
      all_sync<GRID>();
      double pq = 0.0;
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        double s = 0.0;
        for (int32_t e = a.indptr[i]; e < a.indptr[i + 1]; ++e) s += a.data[e] * p[a.indices[e]];
        q[i] = s;
        pq += p[i] * s;
      }
      pq = all_sum<GRID>(pq, sh, part0);
      const double alpha = rho / pq;
      double rn = 0.0;
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        rn += ri * ri;
      }
      rr = all_sum<GRID>(rn, sh, part1);
      rho_prev = rho;
    }
  }
  if (threadIdx.x == 0 && a.iters_out) {
    if (GRID) {
      if (blockIdx.x == 0) a.iters_out[0] = (int32_t)it;
    } else {
      a.iters_out[blockIdx.x] = (int32_t)it;
    }
  }
}

}  // namespace

int launch_cg_scenes(int num, const int32_t* scene_list, int64_t rows_per_scene, const int32_t* indptr,
                     const int32_t* indices, const double* data, const double* b, double* x, double* r, double* p,
                     double* q, double rtol, int64_t maxiter, int32_t* iters_out, cudaStream_t st) {
  if (num <= 0) return 0;
  CgArgs a{indptr, indices, data, b, x, r, p, q, nullptr, iters_out, scene_list, nullptr, nullptr, nullptr,
           rows_per_scene, rtol, maxiter};
  k_cg<false><<<num, kCgThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_cg_scenes_status(int S, int64_t rows_per_scene, const int32_t* indptr, const int32_t* indices,
                            const double* data, const double* b, double* x, double* r, double* p, double* q,
                            double rtol, int64_t maxiter, const SolveStatus* status, const int* cts, double* lam,
                            cudaStream_t st) {
  if (S <= 0) return 0;
  CgArgs a{indptr, indices, data, b, x, r, p, q, nullptr, nullptr, nullptr, status, cts, lam, rows_per_scene, rtol,
           maxiter};
  k_cg<false><<<S, kCgThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int cg_grid_partials(int device) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg<true>, kCgThreads, 0);
  return sms * std::max(1, std::min(per, 2));
}

int launch_cg_grid(int G, int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                   const double* b, double* x, double* r, double* p, double* q, double* partial, double rtol,
                   int64_t maxiter, int32_t* iters_out, cudaStream_t st) {
  CgArgs a{indptr, indices, data, b, x, r, p, q, partial, iters_out, nullptr, nullptr, nullptr, nullptr, n, rtol,
           maxiter};
  void* args[] = {&a};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_cg<true>, dim3(G), dim3(kCgThreads), args, 0, st);
  return e == cudaSuccess ? 0 : 1;
}

}  // namespace vfpi
