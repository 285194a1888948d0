// Contact detection and nodalization of the configs[4] cube pile on the device
// (SURVEY §8(f) items 2-3). Restates pile.CubePile.detect / .nodalize
// operation for operation (same candidate rule, same floating-point
// expressions in the same order -- numpy's einsum over 3 terms and np.cross
// evaluate sequentially), so the contact set, frames, phi and J_v are
// bit-identical to the host pipeline (tests/test_pile.py).
//
//   1. spatial hash: every surface triangle -> the cells (edge `cell`) its
//      bounding box grown by `reach` overlaps; (cell key, triangle) pairs
//      sorted by key (CUB radix sort);
//   2. one thread per surface node: binary search of its own cell, narrow
//      phase against every triangle of another body listed there, best
//      candidate = largest signed distance d, then lowest triangle index;
//   3. plane contacts (z < margin, node order) first, then face contacts in
//      node order (surface list ascending); a node with both gets an identity
//      virtual node for its face contact (contacts.py:249-255);
//   4. J_v in canonical CSR (identity rows: 3 stored entries; face rows: 9,
//      columns ascending), frames contact_frame(n) (contacts.py:131-149),
//      phi = stabilization_term (contacts.py:230-239).
#include <cub/cub.cuh>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

constexpr int kT = 256;
inline unsigned gridn(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

__device__ __forceinline__ long long cell_of(double c, double cell) { return (long long)floor(ddiv(c, cell)); }
__device__ __forceinline__ unsigned long long cell_key(long long cx, long long cy, long long cz) {
  const unsigned long long o = 1ull << 20;
  return ((unsigned long long)(cx + o) << 42) | ((unsigned long long)(cy + o) << 21) | (unsigned long long)(cz + o);
}

__global__ void k_tri_count(int64_t T, const int* __restrict__ tris, const double* __restrict__ x, double reach,
                            double cell, int64_t* __restrict__ cnt, int* __restrict__ bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > T) return;
  if (t == T) { cnt[t] = 0; return; }
  long long span = 1;
  for (int a = 0; a < 3; ++a) {
    const double p0 = x[3 * (int64_t)tris[3 * t] + a], p1 = x[3 * (int64_t)tris[3 * t + 1] + a];
    const double p2 = x[3 * (int64_t)tris[3 * t + 2] + a];
    const double mn = fmin(fmin(p0, p1), p2), mx = fmax(fmax(p0, p1), p2);
    const long long lo = cell_of(dsub(mn, reach), cell), hi = cell_of(dadd(mx, reach), cell);
    if (hi - lo > 7) atomicExch(bad, 1);
    span *= (hi - lo + 1);
  }
  cnt[t] = span;
}

__global__ void k_tri_fill(int64_t T, const int* __restrict__ tris, const double* __restrict__ x, double reach,
                           double cell, const int64_t* __restrict__ off, unsigned long long* __restrict__ key,
                           int* __restrict__ owner) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  long long lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    const double p0 = x[3 * (int64_t)tris[3 * t] + a], p1 = x[3 * (int64_t)tris[3 * t + 1] + a];
    const double p2 = x[3 * (int64_t)tris[3 * t + 2] + a];
    const double mn = fmin(fmin(p0, p1), p2), mx = fmax(fmax(p0, p1), p2);
    lo[a] = cell_of(dsub(mn, reach), cell);
    hi[a] = min(cell_of(dadd(mx, reach), cell), lo[a] + 7);
  }
  int64_t o = off[t];
  for (long long cx = lo[0]; cx <= hi[0]; ++cx)
    for (long long cy = lo[1]; cy <= hi[1]; ++cy)
      for (long long cz = lo[2]; cz <= hi[2]; ++cz) {
        key[o] = cell_key(cx, cy, cz);
        owner[o] = (int)t;
        ++o;
      }
}

// one surface node: best face candidate (pile.CubePile.detect narrow phase)
__global__ void k_node_query(int64_t S, const int* __restrict__ surf, const double* __restrict__ x,
                             const int* __restrict__ tris, const int* __restrict__ node_body,
                             const int* __restrict__ tri_body, const unsigned long long* __restrict__ key,
                             const int* __restrict__ owner, int64_t E, double cell, double neg_half_h, double margin,
                             int* __restrict__ best_tri, double* __restrict__ best) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int node = surf[s];
  const double p[3] = {x[3 * (int64_t)node], x[3 * (int64_t)node + 1], x[3 * (int64_t)node + 2]};
  const unsigned long long k = cell_key(cell_of(p[0], cell), cell_of(p[1], cell), cell_of(p[2], cell));
  int64_t lo = 0, hi = E;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  const int body = node_body[node];
  int bt = -1;
  double bd = 0.0, bw[3] = {0, 0, 0}, bn[3] = {0, 0, 0};
  for (int64_t e = lo; e < E && key[e] == k; ++e) {
    const int t = owner[e];
    if (tri_body[t] >= body) continue;  // one pass: later body's nodes on earlier body's faces
    const int ia = tris[3 * (int64_t)t], ib = tris[3 * (int64_t)t + 1], ic = tris[3 * (int64_t)t + 2];
    double a[3], b[3], c[3];
    for (int q = 0; q < 3; ++q) {
      a[q] = x[3 * (int64_t)ia + q];
      b[q] = x[3 * (int64_t)ib + q];
      c[q] = x[3 * (int64_t)ic + q];
    }
    double ba[3], ca[3], pa[3], n[3];
    for (int q = 0; q < 3; ++q) {
      ba[q] = dsub(b[q], a[q]);
      ca[q] = dsub(c[q], a[q]);
      pa[q] = dsub(p[q], a[q]);
    }
    cross3(ba, ca, n);
    const double nn = dsqrt(dot3(n, n));
    for (int q = 0; q < 3; ++q) n[q] = ddiv(n[q], nn);
    const double d = dot3(pa, n);
    if (!(d > neg_half_h && d < margin)) continue;
    double qv[3], v2[3];
    for (int q = 0; q < 3; ++q) {
      qv[q] = dsub(p[q], dmul(d, n[q]));
      v2[q] = dsub(qv[q], a[q]);
    }
    const double d00 = dot3(ba, ba), d01 = dot3(ba, ca), d11 = dot3(ca, ca);
    const double d20 = dot3(v2, ba), d21 = dot3(v2, ca);
    const double den = dsub(dmul(d00, d11), dmul(d01, d01));
    const double w1 = ddiv(dsub(dmul(d11, d20), dmul(d01, d21)), den);
    const double w2 = ddiv(dsub(dmul(d00, d21), dmul(d01, d20)), den);
    const double w0 = dsub(dsub(1.0, w1), w2);
    if (!(w0 >= 0.0 && w1 >= 0.0 && w2 >= 0.0)) continue;
    if (bt < 0 || d > bd || (d == bd && t < bt)) {
      bt = t;
      bd = d;
      bw[0] = w0;
      bw[1] = w1;
      bw[2] = w2;
      bn[0] = n[0];
      bn[1] = n[1];
      bn[2] = n[2];
    }
  }
  best_tri[s] = bt;
  double* o = best + 7 * s;
  o[0] = bd;
  o[1] = bw[0];
  o[2] = bw[1];
  o[3] = bw[2];
  o[4] = bn[0];
  o[5] = bn[1];
  o[6] = bn[2];
}

__global__ void k_ground_flags(int64_t N, const double* __restrict__ x, double margin, int* __restrict__ g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > N) return;
  g[i] = (i < N && x[3 * i + 2] < margin) ? 1 : 0;
}

// face flags per surface node + the per-face-contact virtual and J_v sizes
__global__ void k_face_sizes(int64_t S, const int* __restrict__ surf, const int* __restrict__ best_tri,
                             const int* __restrict__ gflag, int* __restrict__ fflag, int* __restrict__ nvirt,
                             int* __restrict__ njv) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s > S) return;
  if (s == S) { fflag[s] = 0; nvirt[s] = 0; njv[s] = 0; return; }
  const bool f = best_tri[s] >= 0;
  const int hg = f ? gflag[surf[s]] : 0;
  fflag[s] = f;
  nvirt[s] = f ? 1 + hg : 0;
  njv[s] = f ? 27 + 9 * hg : 0;
}

__device__ __forceinline__ double phi_of(double depth, double vn, double neg_beta_dt, double e_rest, double thr) {
  double phi = dmul(neg_beta_dt, depth);
  if (fabs(vn) > thr) phi = dadd(phi, dmul(e_rest, fmin(0.0, vn)));
  return phi;
}

__global__ void k_ground_contacts(int64_t N, const int* __restrict__ gflag, const int* __restrict__ gpos,
                                  const double* __restrict__ x, const double* __restrict__ v, double mu,
                                  double neg_beta_dt, double e_rest, double thr, int* __restrict__ ci,
                                  int* __restrict__ cj, double* __restrict__ fr, double* __restrict__ muv,
                                  double* __restrict__ phi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N || !gflag[i]) return;
  const int m = gpos[i];
  ci[m] = (int)(3 * i);
  cj[m] = -1;
  const double up[3] = {0.0, 0.0, 1.0};
  double F[9];
  frame_of(up, F);
  for (int q = 0; q < 9; ++q) fr[9 * (int64_t)m + q] = F[q];
  const double vr[3] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  const double vn = dot3(F, vr);
  muv[m] = mu;
  phi[m] = phi_of(fmax(0.0, -x[3 * i + 2]), vn, neg_beta_dt, e_rest, thr);
}

__global__ void k_face_contacts(int64_t S, int n_o, int n_ground, const int* __restrict__ surf,
                                const int* __restrict__ tris, const int* __restrict__ best_tri,
                                const double* __restrict__ best, const int* __restrict__ gflag,
                                const int* __restrict__ fpos, const int* __restrict__ vpos,
                                const int* __restrict__ jpos, const double* __restrict__ v, double mu,
                                double neg_beta_dt, double e_rest, double thr, int* __restrict__ ci,
                                int* __restrict__ cj, double* __restrict__ fr, double* __restrict__ muv,
                                double* __restrict__ phi, int* __restrict__ jrp, int* __restrict__ jci,
                                double* __restrict__ jcx) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S || best_tri[s] < 0) return;
  const int node = surf[s];
  const int m = n_ground + fpos[s];
  const int hg = gflag[node];
  const int vb = vpos[s];
  ci[m] = hg ? n_o + 3 * vb : 3 * node;
  const int vf = vb + hg;
  cj[m] = n_o + 3 * vf;
  const double* o = best + 7 * s;
  double F[9];
  frame_of(o + 4, F);
  for (int q = 0; q < 9; ++q) fr[9 * (int64_t)m + q] = F[q];
  const int t = best_tri[s];
  const int tn[3] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
  const double w[3] = {o[1], o[2], o[3]};
  double vr[3];
  for (int q = 0; q < 3; ++q) {  // v[node] - einsum('fk,fkj->fj', w, v[tri])
    const double vs = dadd(dadd(dmul(w[0], v[3 * (int64_t)tn[0] + q]), dmul(w[1], v[3 * (int64_t)tn[1] + q])),
                           dmul(w[2], v[3 * (int64_t)tn[2] + q]));
    vr[q] = dsub(v[3 * (int64_t)node + q], vs);
  }
  const double vn = dot3(F, vr);
  muv[m] = mu;
  phi[m] = phi_of(fmax(0.0, -o[0]), vn, neg_beta_dt, e_rest, thr);
  // J_v rows (canonical CSR): identity node first, then the face node
  int e = jpos[s];
  if (hg) {
    for (int r = 0; r < 3; ++r) {
      jrp[3 * vb + r] = e;
      for (int c = 0; c < 3; ++c) {
        jci[e] = 3 * node + c;
        jcx[e] = (r == c) ? 1.0 : 0.0;
        ++e;
      }
    }
  }
  int ord[3] = {0, 1, 2};  // face nodes by ascending column
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2 - i; ++j)
      if (tn[ord[j]] > tn[ord[j + 1]]) { const int tmp = ord[j]; ord[j] = ord[j + 1]; ord[j + 1] = tmp; }
  for (int r = 0; r < 3; ++r) {
    jrp[3 * vf + r] = e;
    for (int k = 0; k < 3; ++k)
      for (int c = 0; c < 3; ++c) {
        jci[e] = 3 * tn[ord[k]] + c;
        jcx[e] = dmul(w[ord[k]], (r == c) ? 1.0 : 0.0);
        ++e;
      }
  }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

template <class T>
T* Bp(Workspace::Buf& b) { return reinterpret_cast<T*>(b.p); }

}  // namespace

#define PK(x)                                                            \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                             \
      err = std::string("pile contacts: ") + #x + ": " + cudaGetErrorString(e_); \
      return VFPI_CUDA_ERROR;                                            \
    }                                                                    \
  } while (0)

template <class T>
static cudaError_t scan_excl(PileWork& w, const T* in, T* out, int64_t n, cudaStream_t st) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, st);
  if (e != cudaSuccess) return e;
  e = ensure(w.tmp, tb);
  if (e != cudaSuccess) return e;
  return cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, in, out, n, st);
}

int pile_contacts_device(PileWork& w, const PileGeometry& g, const double* x, const double* v, cudaStream_t st,
                         PileContactsOut& out, std::string& err, int64_t& launches) {
  const int64_t N = g.nodes, S = g.n_surf, T = g.n_tris;
  // 1. spatial hash of the triangles
  PK(ensure(w.tcnt, sizeof(int64_t) * (size_t)(T + 1)));
  PK(ensure(w.toff, sizeof(int64_t) * (size_t)(T + 1)));
  PK(ensure(w.flag, sizeof(int) * 4));
  k_set_int<<<1, 1, 0, st>>>(Bp<int>(w.flag), 0);
  k_tri_count<<<gridn(T + 1), kT, 0, st>>>(T, g.tris, x, g.reach, g.cell, Bp<int64_t>(w.tcnt), Bp<int>(w.flag));
  PK(scan_excl(w, Bp<int64_t>(w.tcnt), Bp<int64_t>(w.toff), T + 1, st));
  PK(cudaMemcpyAsync(w.h_small, Bp<int64_t>(w.toff) + T, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PK(cudaMemcpyAsync(w.h_small + 1, Bp<int>(w.flag), sizeof(int), cudaMemcpyDeviceToHost, st));
  PK(cudaStreamSynchronize(st));
  const int64_t E = w.h_small[0];
  if (reinterpret_cast<int*>(w.h_small + 1)[0]) {
    err = "pile contacts: a surface triangle spans more than 8 hash cells (mesh too deformed)";
    return VFPI_BAD_ARGUMENT;
  }
  PK(ensure(w.key, sizeof(unsigned long long) * (size_t)std::max<int64_t>(E, 1)));
  PK(ensure(w.key2, sizeof(unsigned long long) * (size_t)std::max<int64_t>(E, 1)));
  PK(ensure(w.own, sizeof(int) * (size_t)std::max<int64_t>(E, 1)));
  PK(ensure(w.own2, sizeof(int) * (size_t)std::max<int64_t>(E, 1)));
  k_tri_fill<<<gridn(T), kT, 0, st>>>(T, g.tris, x, g.reach, g.cell, Bp<int64_t>(w.toff),
                                      Bp<unsigned long long>(w.key), Bp<int>(w.own));
  if (E > 0) {
    size_t tb = 0;
    PK(cub::DeviceRadixSort::SortPairs(nullptr, tb, Bp<unsigned long long>(w.key), Bp<unsigned long long>(w.key2),
                                       Bp<int>(w.own), Bp<int>(w.own2), E, 0, 63, st));
    PK(ensure(w.tmp, tb));
    PK(cub::DeviceRadixSort::SortPairs(w.tmp.p, tb, Bp<unsigned long long>(w.key), Bp<unsigned long long>(w.key2),
                                       Bp<int>(w.own), Bp<int>(w.own2), E, 0, 63, st));
  }
  // 2. narrow phase per surface node
  PK(ensure(w.btri, sizeof(int) * (size_t)std::max<int64_t>(S, 1)));
  PK(ensure(w.best, sizeof(double) * 7 * (size_t)std::max<int64_t>(S, 1)));
  k_node_query<<<gridn(S), kT, 0, st>>>(S, g.surf, x, g.tris, g.node_body, g.tri_body,
                                        Bp<unsigned long long>(w.key2), Bp<int>(w.own2), E, g.cell, g.neg_half_h,
                                        g.margin, Bp<int>(w.btri), Bp<double>(w.best));
  // 3. compaction: plane contacts, face contacts, virtual nodes, J_v entries
  PK(ensure(w.gflag, sizeof(int) * (size_t)(N + 1)));
  PK(ensure(w.gpos, sizeof(int) * (size_t)(N + 1)));
  PK(ensure(w.fflag, sizeof(int) * (size_t)(S + 1)));
  PK(ensure(w.fpos, sizeof(int) * (size_t)(S + 1)));
  PK(ensure(w.nvirt, sizeof(int) * (size_t)(S + 1)));
  PK(ensure(w.vpos, sizeof(int) * (size_t)(S + 1)));
  PK(ensure(w.njv, sizeof(int) * (size_t)(S + 1)));
  PK(ensure(w.jpos, sizeof(int) * (size_t)(S + 1)));
  k_ground_flags<<<gridn(N + 1), kT, 0, st>>>(N, x, g.margin, Bp<int>(w.gflag));
  PK(scan_excl(w, Bp<int>(w.gflag), Bp<int>(w.gpos), N + 1, st));
  k_face_sizes<<<gridn(S + 1), kT, 0, st>>>(S, g.surf, Bp<int>(w.btri), Bp<int>(w.gflag), Bp<int>(w.fflag),
                                            Bp<int>(w.nvirt), Bp<int>(w.njv));
  PK(scan_excl(w, Bp<int>(w.fflag), Bp<int>(w.fpos), S + 1, st));
  PK(scan_excl(w, Bp<int>(w.nvirt), Bp<int>(w.vpos), S + 1, st));
  PK(scan_excl(w, Bp<int>(w.njv), Bp<int>(w.jpos), S + 1, st));
  int* hs = reinterpret_cast<int*>(w.h_small);
  PK(cudaMemcpyAsync(hs + 0, Bp<int>(w.gpos) + N, sizeof(int), cudaMemcpyDeviceToHost, st));
  PK(cudaMemcpyAsync(hs + 1, Bp<int>(w.fpos) + S, sizeof(int), cudaMemcpyDeviceToHost, st));
  PK(cudaMemcpyAsync(hs + 2, Bp<int>(w.vpos) + S, sizeof(int), cudaMemcpyDeviceToHost, st));
  PK(cudaMemcpyAsync(hs + 3, Bp<int>(w.jpos) + S, sizeof(int), cudaMemcpyDeviceToHost, st));
  PK(cudaStreamSynchronize(st));
  const int ng = hs[0], nf = hs[1], nv = hs[2], nj = hs[3];
  const int nc = ng + nf;
  PK(ensure(w.ci, sizeof(int) * (size_t)std::max(nc, 1)));
  PK(ensure(w.cj, sizeof(int) * (size_t)std::max(nc, 1)));
  PK(ensure(w.fr, sizeof(double) * 9 * (size_t)std::max(nc, 1)));
  PK(ensure(w.mu, sizeof(double) * (size_t)std::max(nc, 1)));
  PK(ensure(w.phi, sizeof(double) * (size_t)std::max(nc, 1)));
  PK(ensure(w.jrp, sizeof(int) * (size_t)(3 * nv + 1)));
  PK(ensure(w.jci, sizeof(int) * (size_t)std::max(nj, 1)));
  PK(ensure(w.jcx, sizeof(double) * (size_t)std::max(nj, 1)));
  k_ground_contacts<<<gridn(N), kT, 0, st>>>(N, Bp<int>(w.gflag), Bp<int>(w.gpos), x, v, g.mu, g.neg_beta_dt,
                                             g.e_rest, g.rest_threshold, Bp<int>(w.ci), Bp<int>(w.cj),
                                             Bp<double>(w.fr), Bp<double>(w.mu), Bp<double>(w.phi));
  k_face_contacts<<<gridn(S), kT, 0, st>>>(S, g.n_o, ng, g.surf, g.tris, Bp<int>(w.btri), Bp<double>(w.best),
                                           Bp<int>(w.gflag), Bp<int>(w.fpos), Bp<int>(w.vpos), Bp<int>(w.jpos), v,
                                           g.mu, g.neg_beta_dt, g.e_rest, g.rest_threshold, Bp<int>(w.ci),
                                           Bp<int>(w.cj), Bp<double>(w.fr), Bp<double>(w.mu), Bp<double>(w.phi),
                                           Bp<int>(w.jrp), Bp<int>(w.jci), Bp<double>(w.jcx));
  k_set_int<<<1, 1, 0, st>>>(Bp<int>(w.jrp) + 3 * nv, nj);
  PK(cudaGetLastError());
  launches += 16;
  out.n_ground = ng;
  out.n_face = nf;
  out.n_virtual = nv;
  out.jv_nnz = nj;
  out.col_i = Bp<int>(w.ci);
  out.col_j = Bp<int>(w.cj);
  out.frames = Bp<double>(w.fr);
  out.mu = Bp<double>(w.mu);
  out.phi = Bp<double>(w.phi);
  out.jv_indptr = Bp<int>(w.jrp);
  out.jv_indices = Bp<int>(w.jci);
  out.jv_data = Bp<double>(w.jcx);
  return VFPI_OK;
}

}  // namespace vfpi
