// Contact nodalization on the device: the reference's
// nodalize (condsim/contacts.py:271-321) with _slot_and_jv (:242-268),
// contact_frame (:131-149), _normal_velocity (:333-340) and
// stabilization_term (:230-239), producing the same slots, virtual nodes,
// J_v (canonical CSR, every block entry stored, signed zeros included),
// frames and phi bit for bit.
//
//   * a node side keeps its own slot on its first use in processing order
//     (contact m, first side then second); later uses move to an identity
//     virtual node: first uses are found with an atomicMin of 2m+side per
//     node offset (order-independent result);
//   * virtual nodes are numbered in processing order (exclusive scan);
//   * rigid sides: J_v block [I, -[r]x] with r = point - body position;
//   * norms and 3-term dots are numpy's: np.linalg.norm / x @ y on 3-vectors
//     go through OpenBLAS ddot, whose 3-element result is
//     fma(x2, y2, fma(x1, y1, x0 * y0)) (pinned by tests/golden); cross
//     products follow np.cross.
#include <climits>

#include <cub/cub.cuh>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

constexpr int kT = 256;
inline unsigned gridn(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

__device__ __forceinline__ double blas_dot3(const double* a, const double* b) {
  return __fma_rn(a[2], b[2], __fma_rn(a[1], b[1], dmul(a[0], b[0])));
}
__device__ __forceinline__ void np_cross(const double* a, const double* b, double* c) {
  c[0] = dsub(dmul(a[1], b[2]), dmul(a[2], b[1]));
  c[1] = dsub(dmul(a[2], b[0]), dmul(a[0], b[2]));
  c[2] = dsub(dmul(a[0], b[1]), dmul(a[1], b[0]));
}

__global__ void k_nod_fill_int(int64_t n, int* __restrict__ p, int v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// first use of every node offset (processing order 2m + side)
// (also validates the sides: kinds, node offsets inside [0, n_o - 3], body ids
// inside [0, n_bodies); a static first side is not a contact)
__global__ void k_nod_first_use(int64_t n_c, int n_o, int n_bodies, int64_t n_q, const int* __restrict__ fk,
                                const int* __restrict__ fr, const int* __restrict__ sk, const int* __restrict__ sr,
                                const int* __restrict__ body_q, const int* __restrict__ body_v,
                                int* __restrict__ first, int* __restrict__ bad) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  for (int s = 0; s < 2; ++s) {
    const int kind = s ? sk[m] : fk[m], ref = s ? sr[m] : fr[m];
    // a rigid side reads q[body_q .. +2] (position) and writes J_v columns body_v .. +5
    const bool rigid_ok = kind == 1 && ref >= 0 && ref < n_bodies && body_q[ref] >= 0 &&
                          (int64_t)body_q[ref] + 3 <= n_q && body_v[ref] >= 0 && body_v[ref] + 6 <= n_o;
    const bool ok = (kind == 0 && ref >= 0 && ref <= n_o - 3) || rigid_ok || (kind == -1 && s == 1);
    if (!ok) {
      atomicExch(bad, 1);
      continue;
    }
    if (kind == 0) atomicMin(first + ref, (int)(2 * m + s));
  }
}

// per (contact, side): 1 if it needs a virtual node; its J_v entry count
__global__ void k_nod_virtual_flags(int64_t n_c, int n_o, const int* __restrict__ fk, const int* __restrict__ fr,
                                    const int* __restrict__ sk, const int* __restrict__ sr,
                                    const int* __restrict__ first, int* __restrict__ vflag, int* __restrict__ jcnt) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o > 2 * n_c) return;
  if (o == 2 * n_c) { vflag[o] = 0; jcnt[o] = 0; return; }
  const int64_t m = o >> 1;
  const int kind = (o & 1) ? sk[m] : fk[m];
  const int ref = (o & 1) ? sr[m] : fr[m];
  int f = 0, c = 0;
  if (kind == 1) { f = 1; c = 18; }                            // rigid: [I, -[r]x]
  else if (kind == 0 && ref >= 0 && ref <= n_o - 3 && first[ref] != (int)o) { f = 1; c = 9; }  // node, later use
  vflag[o] = f;
  jcnt[o] = c;
}

__global__ void k_nod_contacts(int64_t n_c, int n_o, const int* __restrict__ fk, const int* __restrict__ fr,
                               const int* __restrict__ sk, const int* __restrict__ sr,
                               const double* __restrict__ point, const double* __restrict__ normal,
                               const double* __restrict__ depth, const double* __restrict__ q,
                               const double* __restrict__ v, const int* __restrict__ body_q,
                               const int* __restrict__ body_v, const int* __restrict__ vflag,
                               const int* __restrict__ vpos, const int* __restrict__ jpos, double mu, double mu2,
                               double neg_beta_dt, double e_rest, double thr, int* __restrict__ ci,
                               int* __restrict__ cj, double* __restrict__ frames, double* __restrict__ phi,
                               double* __restrict__ muv, double* __restrict__ mu2v, int* __restrict__ jrp,
                               int* __restrict__ jci, double* __restrict__ jcx, int* __restrict__ bad) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  const double pt[3] = {point[3 * m], point[3 * m + 1], point[3 * m + 2]};
  double vside[2][3];
  for (int s = 0; s < 2; ++s) {
    const int64_t o = 2 * m + s;
    const int kind = s ? sk[m] : fk[m];
    const int ref = s ? sr[m] : fr[m];
    int col = -1;
    if (kind == 0) {
      for (int a = 0; a < 3; ++a) vside[s][a] = v[ref + a];
      if (!vflag[o]) {
        col = ref;
      } else {  // identity virtual node (contacts.py:251-255)
        const int vn = vpos[o];
        col = n_o + 3 * vn;
        int e = jpos[o];
        for (int r = 0; r < 3; ++r) {
          jrp[3 * vn + r] = e;
          for (int c = 0; c < 3; ++c) {
            jci[e] = ref + c;
            jcx[e] = (r == c) ? 1.0 : 0.0;
            ++e;
          }
        }
      }
    } else if (kind == 1) {
      const int qo = body_q[ref], vo = body_v[ref];
      const double lever[3] = {dsub(pt[0], q[qo]), dsub(pt[1], q[qo + 1]), dsub(pt[2], q[qo + 2])};
      const double om[3] = {v[vo + 3], v[vo + 4], v[vo + 5]};
      double cr[3];
      np_cross(om, lever, cr);
      for (int a = 0; a < 3; ++a) vside[s][a] = dadd(v[vo + a], cr[a]);
      const int vn = vpos[o];
      col = n_o + 3 * vn;
      // -lx with lx = [[0, -r2, r1], [r2, 0, -r0], [-r1, r0, 0]] (negated zeros are -0.0)
      const double nlx[3][3] = {{-0.0, lever[2], -lever[1]}, {-lever[2], -0.0, lever[0]},
                                {lever[1], -lever[0], -0.0}};
      int e = jpos[o];
      for (int r = 0; r < 3; ++r) {
        jrp[3 * vn + r] = e;
        for (int c = 0; c < 6; ++c) {
          jci[e] = vo + c;
          jcx[e] = c < 3 ? ((r == c) ? 1.0 : 0.0) : nlx[r][c - 3];
          ++e;
        }
      }
    } else {
      vside[s][0] = vside[s][1] = vside[s][2] = 0.0;
    }
    if (s == 0) ci[m] = col;
    else cj[m] = col;
  }
  // contact_frame (contacts.py:131-149)
  double n[3] = {normal[3 * m], normal[3 * m + 1], normal[3 * m + 2]};
  const double norm = dsqrt(blas_dot3(n, n));
  if (norm < 1e-12) {
    atomicExch(bad, 1);
    return;
  }
  if (fabs(dsub(norm, 1.0)) > 1e-9)
    for (int a = 0; a < 3; ++a) n[a] = ddiv(n[a], norm);
  int ax = 0;
  double am = fabs(n[0]);
  for (int a = 1; a < 3; ++a)
    if (fabs(n[a]) < am) { am = fabs(n[a]); ax = a; }
  double e3[3] = {0.0, 0.0, 0.0};
  e3[ax] = 1.0;
  double ne[3], t1[3], t2[3];
  np_cross(n, e3, ne);
  np_cross(ne, n, t1);
  const double tn = dsqrt(blas_dot3(t1, t1));
  for (int a = 0; a < 3; ++a) t1[a] = ddiv(t1[a], tn);
  np_cross(n, t1, t2);
  double* F = frames + 9 * m;
  for (int a = 0; a < 3; ++a) {
    F[a] = n[a];
    F[3 + a] = t1[a];
    F[6 + a] = t2[a];
  }
  // _normal_velocity + stabilization_term
  const double vr[3] = {dsub(vside[0][0], vside[1][0]), dsub(vside[0][1], vside[1][1]),
                        dsub(vside[0][2], vside[1][2])};
  const double vnp = blas_dot3(n, vr);
  double ph = dmul(neg_beta_dt, depth[m]);
  if (fabs(vnp) > thr) ph = dadd(ph, dmul(e_rest, vnp < 0.0 ? vnp : 0.0));
  phi[m] = ph;
  muv[m] = mu;
  mu2v[m] = mu2;
}

__global__ void k_nod_set(int* p, int v) { *p = v; }

template <class T>
T* Bn(Workspace::Buf& b) { return reinterpret_cast<T*>(b.p); }

}  // namespace

#define NK(x)                                                         \
  do {                                                                \
    cudaError_t e_ = (x);                                             \
    if (e_ != cudaSuccess) {                                          \
      err = std::string("nodalize: ") + #x + ": " + cudaGetErrorString(e_); \
      return VFPI_CUDA_ERROR;                                         \
    }                                                                 \
  } while (0)

int nodalize_device(NodalizeWork& w, const NodalizeIn& in, cudaStream_t st, NodalizeOut& out, std::string& err,
                    int64_t& launches) {
  const int64_t n_c = in.n_c;
  const int64_t S = 2 * n_c;
  NK(ensure(w.first, sizeof(int) * (size_t)std::max(in.n_o, 1)));
  NK(ensure(w.vflag, sizeof(int) * (size_t)(S + 1)));
  NK(ensure(w.vpos, sizeof(int) * (size_t)(S + 1)));
  NK(ensure(w.jcnt, sizeof(int) * (size_t)(S + 1)));
  NK(ensure(w.jpos, sizeof(int) * (size_t)(S + 1)));
  NK(ensure(w.flag, sizeof(int)));
  k_nod_fill_int<<<gridn(in.n_o), kT, 0, st>>>(in.n_o, Bn<int>(w.first), INT_MAX);
  k_nod_set<<<1, 1, 0, st>>>(Bn<int>(w.flag), 0);
  k_nod_first_use<<<gridn(n_c), kT, 0, st>>>(n_c, in.n_o, in.n_bodies, in.n_q, in.first_kind, in.first_ref,
                                              in.second_kind, in.second_ref, in.body_q, in.body_v, Bn<int>(w.first),
                                              Bn<int>(w.flag));
  k_nod_virtual_flags<<<gridn(S + 1), kT, 0, st>>>(n_c, in.n_o, in.first_kind, in.first_ref, in.second_kind, in.second_ref,
                                                   Bn<int>(w.first), Bn<int>(w.vflag), Bn<int>(w.jcnt));
  size_t tb = 0;
  NK(cub::DeviceScan::ExclusiveSum(nullptr, tb, Bn<int>(w.vflag), Bn<int>(w.vpos), S + 1, st));
  NK(ensure(w.tmp, tb));
  NK(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, Bn<int>(w.vflag), Bn<int>(w.vpos), S + 1, st));
  NK(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, Bn<int>(w.jcnt), Bn<int>(w.jpos), S + 1, st));
  int* hs = reinterpret_cast<int*>(w.h_small);
  NK(cudaMemcpyAsync(hs, Bn<int>(w.vpos) + S, sizeof(int), cudaMemcpyDeviceToHost, st));
  NK(cudaMemcpyAsync(hs + 1, Bn<int>(w.jpos) + S, sizeof(int), cudaMemcpyDeviceToHost, st));
  NK(cudaMemcpyAsync(hs + 2, Bn<int>(w.flag), sizeof(int), cudaMemcpyDeviceToHost, st));
  NK(cudaStreamSynchronize(st));
  if (hs[2]) {
    err = "nodalize: bad contact side (kind, node offset, body index or body q/v offsets out of range)";
    return VFPI_BAD_ARGUMENT;
  }
  const int nv = hs[0], nj = hs[1];
  NK(ensure(w.ci, sizeof(int) * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.cj, sizeof(int) * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.fr, sizeof(double) * 9 * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.phi, sizeof(double) * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.mu, sizeof(double) * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.mu2, sizeof(double) * (size_t)std::max<int64_t>(n_c, 1)));
  NK(ensure(w.jrp, sizeof(int) * (size_t)(3 * nv + 1)));
  NK(ensure(w.jci, sizeof(int) * (size_t)std::max(nj, 1)));
  NK(ensure(w.jcx, sizeof(double) * (size_t)std::max(nj, 1)));
  k_nod_contacts<<<gridn(n_c), kT, 0, st>>>(
      n_c, in.n_o, in.first_kind, in.first_ref, in.second_kind, in.second_ref, in.point, in.normal, in.depth, in.q,
      in.v, in.body_q, in.body_v, Bn<int>(w.vflag), Bn<int>(w.vpos), Bn<int>(w.jpos), in.mu, in.mu2, in.neg_beta_dt,
      in.e_rest, in.rest_threshold, Bn<int>(w.ci), Bn<int>(w.cj), Bn<double>(w.fr), Bn<double>(w.phi),
      Bn<double>(w.mu), Bn<double>(w.mu2), Bn<int>(w.jrp), Bn<int>(w.jci), Bn<double>(w.jcx), Bn<int>(w.flag));
  k_nod_set<<<1, 1, 0, st>>>(Bn<int>(w.jrp) + 3 * nv, nj);
  NK(cudaMemcpyAsync(hs + 2, Bn<int>(w.flag), sizeof(int), cudaMemcpyDeviceToHost, st));
  NK(cudaStreamSynchronize(st));
  launches += 9;
  if (hs[2]) {
    err = "nodalize: contact normal is zero (contacts.py:139-140)";
    return VFPI_BAD_ARGUMENT;
  }
  out.n_virtual = nv;
  out.jv_nnz = nj;
  out.col_i = Bn<int>(w.ci);
  out.col_j = Bn<int>(w.cj);
  out.frames = Bn<double>(w.fr);
  out.phi = Bn<double>(w.phi);
  out.mu = Bn<double>(w.mu);
  out.mu2 = Bn<double>(w.mu2);
  out.jv_indptr = Bn<int>(w.jrp);
  out.jv_indices = Bn<int>(w.jci);
  out.jv_data = Bn<double>(w.jcx);
  return VFPI_OK;
}

}  // namespace vfpi
