// configs[3] step pieces on the device: node-vs-heightfield contact detection
// and the external-load term of the right-hand side.
//
// The reference has no heightfield (its detect_contacts, contacts.py:159-227,
// knows planes and spheres); this is the same contract for the surface
// z = amp sin(freq x) sin(freq y): every node with z < h + margin becomes an
// S-contact on its own node (nodalize, contacts.py:271-321: col_i = 3 node,
// col_j = -1), in node order, with depth max(0, h - z), phi = -(beta/dt)
// depth (stabilization_term, :230-239, no restitution), normal
// (-hx, -hy, 1)/norm and frame contact_frame(normal) (:131-149). The sine and
// cosine are a fixed Cody-Waite + fdlibm-polynomial sequence (hf_sincos), the
// same as scenes.hf_sincos on the host, so the device contact set, frames and
// phi equal the host restatement (oracle/fem_host.heightfield_contacts) bit
// for bit. One thread per node; compaction by an exclusive scan of flags;
// one host read of the contact count.
#include <cub/cub.cuh>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

constexpr int kT = 256;
inline unsigned gridn(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

__device__ __forceinline__ void hf_sincos(double t, double* sn, double* cs) {
  const double kTwoOverPi = 6.36619772367581382433e-01;
  const double kPio2_1 = 1.57079632673412561417e+00;
  const double kPio2_1t = 6.07710050650619224932e-11;
  const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
               S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
               S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
               C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
               C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double k = rint(dmul(t, kTwoOverPi));
  const double r = dsub(dsub(t, dmul(k, kPio2_1)), dmul(k, kPio2_1t));
  const double z = dmul(r, r);
  const double ps = dadd(S1, dmul(z, dadd(S2, dmul(z, dadd(S3, dmul(z, dadd(S4, dmul(z, dadd(S5, dmul(z, S6))))))))));
  const double s = dadd(r, dmul(dmul(z, r), ps));
  const double pc = dadd(C1, dmul(z, dadd(C2, dmul(z, dadd(C3, dmul(z, dadd(C4, dmul(z, dadd(C5, dmul(z, C6))))))))));
  const double c = dsub(1.0, dsub(dmul(0.5, z), dmul(z, dmul(z, pc))));
  // np.mod(k, 4.0): the quadrant, 0..3 for any sign of k
  double q = fmod(k, 4.0);
  if (q < 0) q += 4.0;
  const int qi = (int)q;
  *sn = qi == 0 ? s : qi == 1 ? c : qi == 2 ? -s : -c;
  *cs = qi == 0 ? c : qi == 1 ? -s : qi == 2 ? -c : s;
}

__device__ __forceinline__ double hf_height(double x, double y, double amp, double freq, double* sx, double* cx,
                                            double* sy, double* cy) {
  hf_sincos(dmul(freq, x), sx, cx);
  hf_sincos(dmul(freq, y), sy, cy);
  return dmul(dmul(amp, *sx), *sy);
}

__global__ void k_hf_flags(int64_t N, const double* __restrict__ x, double amp, double freq, double margin,
                           int* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  double sx, cx, sy, cy;
  const double h = hf_height(x[3 * i], x[3 * i + 1], amp, freq, &sx, &cx, &sy, &cy);
  flag[i] = x[3 * i + 2] < dadd(h, margin) ? 1 : 0;
}

__global__ void k_hf_contacts(int64_t N, const int* __restrict__ flag, const int* __restrict__ pos,
                              const double* __restrict__ x, double amp, double freq, double slope, double neg_beta_dt,
                              double mu, int* __restrict__ ci, int* __restrict__ cj, double* __restrict__ fr,
                              double* __restrict__ muv, double* __restrict__ phi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N || !flag[i]) return;
  const int64_t m = pos[i];
  double sx, cx, sy, cy;
  const double h = hf_height(x[3 * i], x[3 * i + 1], amp, freq, &sx, &cx, &sy, &cy);
  const double depth = np_max(0.0, dsub(h, x[3 * i + 2]));
  const double hx = dmul(dmul(slope, cx), sy);
  const double hy = dmul(dmul(slope, sx), cy);
  const double norm = dsqrt(dadd(dadd(dmul(hx, hx), dmul(hy, hy)), 1.0));
  const double n[3] = {ddiv(-hx, norm), ddiv(-hy, norm), ddiv(1.0, norm)};
  double F[9];
  frame_of(n, F);
  for (int q = 0; q < 9; ++q) fr[9 * m + q] = F[q];
  ci[m] = (int)(3 * i);
  cj[m] = -1;
  muv[m] = mu;
  phi[m] = dmul(neg_beta_dt, depth);
}

__global__ void k_add_inplace(int64_t n, const double* __restrict__ f, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = dadd(b[i], f[i]);
}

}  // namespace

int heightfield_contacts_device(HfWork& w, const HfParams& p, int64_t N, const double* x, cudaStream_t st,
                                HfContactsOut& out, std::string& err, int64_t& launches) {
  auto fail = [&](cudaError_t e) {
    err = std::string("heightfield contacts: ") + cudaGetErrorString(e);
    return VFPI_CUDA_ERROR;
  };
  cudaError_t e;
  if (!w.h_small && (e = cudaMallocHost(&w.h_small, 16)) != cudaSuccess) return fail(e);
  const size_t n = (size_t)std::max<int64_t>(N, 1);
  if ((e = ensure(w.flag, 4 * n)) || (e = ensure(w.pos, 4 * n))) return fail(e);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (int*)w.flag.p, (int*)w.pos.p, (int)n, st);
  if ((e = ensure(w.tmp, std::max<size_t>(tb, 16)))) return fail(e);
  int* flag = (int*)w.flag.p;
  int* pos = (int*)w.pos.p;
  k_hf_flags<<<gridn(N), kT, 0, st>>>(N, x, p.amp, p.freq, p.margin, flag);
  tb = w.tmp.cap;
  if ((e = cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, flag, pos, (int)n, st))) return fail(e);
  launches += 3;
  if ((e = cudaMemcpyAsync(w.h_small, pos + (n - 1), 4, cudaMemcpyDeviceToHost, st)) ||
      (e = cudaMemcpyAsync((int*)w.h_small + 1, flag + (n - 1), 4, cudaMemcpyDeviceToHost, st)) ||
      (e = cudaStreamSynchronize(st)))
    return fail(e);
  const int64_t nc = N > 0 ? (int64_t)((int*)w.h_small)[0] + ((int*)w.h_small)[1] : 0;
  const size_t c = (size_t)std::max<int64_t>(nc, 1);
  if ((e = ensure(w.ci, 4 * c)) || (e = ensure(w.cj, 4 * c)) || (e = ensure(w.fr, 72 * c)) ||
      (e = ensure(w.mu, 8 * c)) || (e = ensure(w.phi, 8 * c)))
    return fail(e);
  k_hf_contacts<<<gridn(N), kT, 0, st>>>(N, flag, pos, x, p.amp, p.freq, p.slope, p.neg_beta_dt, p.mu,
                                         (int*)w.ci.p, (int*)w.cj.p, (double*)w.fr.p, (double*)w.mu.p,
                                         (double*)w.phi.p);
  ++launches;
  if ((e = cudaGetLastError())) return fail(e);
  out.n_c = nc;
  out.col_i = (int*)w.ci.p;
  out.col_j = (int*)w.cj.p;
  out.frames = (double*)w.fr.p;
  out.mu = (double*)w.mu.p;
  out.phi = (double*)w.phi.p;
  return VFPI_OK;
}

void launch_add_inplace(int64_t n, const double* f, double* b, cudaStream_t st) {
  if (n > 0) k_add_inplace<<<gridn(n), kT, 0, st>>>(n, f, b);
}

}  // namespace vfpi
