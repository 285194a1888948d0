// Device step pipeline of the FEM scene batches (configs[0]/[2]; SURVEY
// §8(f) item 1): right-hand side assembly, node-plane contact detection,
// contact parameters and midpoint integration, so a batch steps without host
// round trips of the state. Every expression follows the host restatement
// (scenes.FemCube.system / contacts / advance) operation for operation, so
// the device pipeline and the host pipeline produce identical bits.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

// b = ((2/dt) m) v - K (x - X) + m g   (FemCube.system; K @ u in scipy's
// per-row column order, FMA-free, explicit zeros included)
__global__ void k_fem_rhs(int64_t n, const int64_t* __restrict__ krp, const int* __restrict__ kc,
                          const double* __restrict__ kv, const double* __restrict__ x, const double* __restrict__ X,
                          const double* __restrict__ v, const double* __restrict__ m, const double* __restrict__ g,
                          double twodt, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ku = 0.0;
  for (int64_t e = krp[i]; e < krp[i + 1]; ++e) {
    const int j = kc[e];
    ku = dadd(ku, dmul(kv[e], dsub(x[j], X[j])));
  }
  const double t1 = dmul(dmul(twodt, m[i]), v[i]);
  b[i] = dadd(dsub(t1, ku), dmul(m[i], g[i]));
}

// K in SELL-32 (slices of 32 consecutive rows, entry k of row r at
// off[slice] + 32 k + (r & 31); padding column -1), so the per-row
// sequential sums of the right-hand side read K coalesced
__global__ void k_fem_sell_width(int64_t n, const int64_t* __restrict__ krp, int64_t* __restrict__ width) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nsl = (n + 31) / 32;
  if (s > nsl) return;
  if (s == nsl) { width[s] = 0; return; }
  int64_t w = 0;
  for (int64_t r = 32 * s; r < n && r < 32 * s + 32; ++r) w = max(w, krp[r + 1] - krp[r]);
  width[s] = 32 * w;
}

__global__ void k_fem_sell_pack(int64_t n, const int64_t* __restrict__ krp, const int* __restrict__ kc,
                                const double* __restrict__ kv, const int64_t* __restrict__ off,
                                double* __restrict__ sv, int* __restrict__ sc) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t s = r >> 5, o = off[s];
  const int W = (int)((off[s + 1] - o) >> 5);
  const int64_t e0 = krp[r], len = krp[r + 1] - e0;
  for (int k = 0; k < W; ++k) {
    const int64_t dst = o + 32 * (int64_t)k + (r & 31);
    sv[dst] = k < len ? kv[e0 + k] : 0.0;
    sc[dst] = k < len ? kc[e0 + k] : -1;
  }
}

__global__ void k_fem_rhs_sell(int64_t n, const int64_t* __restrict__ off, const double* __restrict__ sv,
                               const int* __restrict__ sc, const double* __restrict__ x,
                               const double* __restrict__ X, const double* __restrict__ v,
                               const double* __restrict__ m, const double* __restrict__ g, double twodt,
                               double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = off[i >> 5] + (i & 31);
  const int W = (int)((off[(i >> 5) + 1] - off[i >> 5]) >> 5);
  // row operands first, then the K row in batches of 8 independent loads
  // (same sequential accumulation order)
  const double mi = m[i], vi = v[i], gi = g[i];
  double ku = 0.0;
  int k = 0;
  for (; k + 8 <= W; k += 8) {
    int j[8];
    double a[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      j[u] = __ldcs(sc + o + 32 * (int64_t)(k + u));
      a[u] = __ldcs(sv + o + 32 * (int64_t)(k + u));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = j[u] >= 0 ? dsub(x[j[u]], X[j[u]]) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j[u] >= 0) ku = dadd(ku, dmul(a[u], xv[u]));
  }
  for (; k < W; ++k) {
    const int jj = __ldcs(sc + o + 32 * (int64_t)k);
    if (jj >= 0) ku = dadd(ku, dmul(__ldcs(sv + o + 32 * (int64_t)k), dsub(x[jj], X[jj])));
  }
  const double t1 = dmul(dmul(twodt, mi), vi);
  b[i] = dadd(dsub(t1, ku), dmul(mi, gi));
}

// The same right-hand side with K in the node-block layout of the batch (one
// warp per node slice, one lane per node: 3 row sums per lane, blocks in
// increasing block column, entries of a block in increasing column -- each
// row's sequence of k_fem_rhs; the masks keep K's explicit zeros)
__global__ void __launch_bounds__(256) k_fem_rhs_nodes(int64_t nslices, int nn, int nsl,
                                                       const int64_t* __restrict__ slice_off,
                                                       const int* __restrict__ node_list,
                                                       const unsigned* __restrict__ kdesc,
                                                       const double* __restrict__ kval, const double* __restrict__ x,
                                                       const double* __restrict__ X, const double* __restrict__ v,
                                                       const double* __restrict__ m, const double* __restrict__ g,
                                                       double twodt, double* __restrict__ b) {
  const int64_t gs = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gs >= nslices) return;
  const int scene = (int)(gs / nsl), sl = (int)(gs % nsl);
  const int p = sl * 32 + lane;
  const int64_t off = slice_off[gs];
  const int W = (int)(slice_off[gs + 1] - off);
  const bool live = p < nn;
  const int node = live ? node_list[(int64_t)scene * nn + p] : 0;
  double k0 = 0.0, k1 = 0.0, k2 = 0.0;
  // two blocks per step with every load issued first (the 9 value slots of a
  // block share its 2304-byte line set, so loading absent slots costs no DRAM
  // traffic); absent entries are still skipped, not added as zeros
  constexpr int U = 2;
  for (int k = 0; k < W; k += U) {
    unsigned mk[U];
    double kv[U][9], u[U][3];
#pragma unroll
    for (int e = 0; e < U; ++e) {
      const bool in = k + e < W;
      const unsigned d = in ? __ldcs(kdesc + (off + k + e) * 32 + lane) : 0u;
      mk[e] = d >> 23;
      const int c = mk[e] ? 3 * (int)(d & ((1u << 23) - 1u)) : 0;
      const double* vp = kval + (off + (in ? k + e : k)) * (9 * 32) + lane;
#pragma unroll
      for (int t = 0; t < 9; ++t) kv[e][t] = __ldcs(vp + 32 * t);
#pragma unroll
      for (int q = 0; q < 3; ++q) u[e][q] = dsub(x[c + q], X[c + q]);
    }
#pragma unroll
    for (int e = 0; e < U; ++e) {
      const unsigned m = mk[e];
      if (m & 0x001) k0 = dadd(k0, dmul(kv[e][0], u[e][0]));
      if (m & 0x002) k0 = dadd(k0, dmul(kv[e][1], u[e][1]));
      if (m & 0x004) k0 = dadd(k0, dmul(kv[e][2], u[e][2]));
      if (m & 0x008) k1 = dadd(k1, dmul(kv[e][3], u[e][0]));
      if (m & 0x010) k1 = dadd(k1, dmul(kv[e][4], u[e][1]));
      if (m & 0x020) k1 = dadd(k1, dmul(kv[e][5], u[e][2]));
      if (m & 0x040) k2 = dadd(k2, dmul(kv[e][6], u[e][0]));
      if (m & 0x080) k2 = dadd(k2, dmul(kv[e][7], u[e][1]));
      if (m & 0x100) k2 = dadd(k2, dmul(kv[e][8], u[e][2]));
    }
  }
  if (!live) return;
  const double ku[3] = {k0, k1, k2};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int64_t i = 3 * (int64_t)node + q;
    const double mi = m[i];
    const double t1 = dmul(dmul(twodt, mi), v[i]);
    b[i] = dadd(dsub(t1, ku[q]), dmul(mi, g[i]));
  }
}

// Node-plane contacts (FemCube.contacts): a node is in contact when it lies
// below the margin of the plane z = 0. After the exclusive scan of that
// predicate over all nodes (scene-ordered compaction), one pass writes the
// scene pointers cts and every contact's parameters; optionally it zeroes
// both impulse parities of every contact (the run loop's solve start).
__global__ void k_fem_detect(int64_t nodes, int S, int nodes_per_scene, const int* __restrict__ pos,
                             const double* __restrict__ x, const double* __restrict__ v, double margin,
                             const double* __restrict__ frame, double mu, double neg_beta_dt, double e_rest,
                             double thr, int* __restrict__ cts, int* __restrict__ ci, int* __restrict__ cj,
                             double* __restrict__ frames, double* __restrict__ muv, double* __restrict__ mu2v,
                             double* __restrict__ phi, double* __restrict__ lam0, double* __restrict__ lam1) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nodes) return;
  const double z = x[3 * k + 2];
  const bool in = z < margin;
  const int c = pos[k];
  if (k % nodes_per_scene == 0) cts[k / nodes_per_scene] = c;
  if (k == nodes - 1) cts[S] = c + (in ? 1 : 0);
  if (!in) return;
  const double depth = np_max(0.0, -z);        // np.maximum(0.0, -z[nodes])
  double ph = dmul(neg_beta_dt, depth);        // -(beta / dt) * depth
  const double vn = v[3 * k + 2];
  if (fabs(vn) > thr) ph = dadd(ph, dmul(e_rest, np_min(0.0, vn)));  // np.where(rest, ...)
  ci[c] = (int)(3 * k);
  cj[c] = -1;
  if (lam0) {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      lam0[3 * (size_t)c + t] = 0.0;
      lam1[3 * (size_t)c + t] = 0.0;
    }
  }
#pragma unroll
  for (int t = 0; t < 9; ++t) frames[9 * (size_t)c + t] = frame[t];
  muv[c] = mu;
  mu2v[c] = mu;
  phi[c] = ph;
}

struct BelowMargin {  // the contact predicate as a scan input
  const double* x;
  double margin;
  __host__ __device__ int operator()(int64_t k) const { return x[3 * k + 2] < margin ? 1 : 0; }
};
using FlagIter = thrust::transform_iterator<BelowMargin, thrust::counting_iterator<int64_t>>;

// midpoint integration (FemCube.advance): x += dt v_hat; v = 2 v_hat - v;
// the solution also warm-starts the next step
__global__ void k_fem_advance(int64_t n, double dt, const double* __restrict__ vh, double* __restrict__ x,
                              double* __restrict__ v, double* __restrict__ warm) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double h = vh[i];
  x[i] = dadd(x[i], dmul(dt, h));
  v[i] = dsub(dmul(2.0, h), v[i]);
  if (warm) warm[i] = h;
}

// y = J x with J in CSR, each row summed from 0 in stored order (scipy's
// csr_matvec; explicit zeros included): the warm-start extension
// v0[n_o:] = J_v v0[:n_o] of harness._warm_velocity (harness.py:502-512)
__global__ void k_csr_matvec(int64_t rows, const int* __restrict__ rp, const int* __restrict__ ci,
                             const double* __restrict__ cx, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int e = rp[r]; e < rp[r + 1]; ++e) s = dadd(s, dmul(cx[e], x[ci[e]]));
  y[r] = s;
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_fem_rhs(int64_t n, const int64_t* krp, const int* kc, const double* kv, const double* x, const double* X,
                    const double* v, const double* m, const double* g, double twodt, double* b, cudaStream_t st) {
  if (n > 0) k_fem_rhs<<<nb(n), 256, 0, st>>>(n, krp, kc, kv, x, X, v, m, g, twodt, b);
}

void launch_fem_sell_width(int64_t n, const int64_t* krp, int64_t* width, cudaStream_t st) {
  k_fem_sell_width<<<nb((n + 31) / 32 + 1), 256, 0, st>>>(n, krp, width);
}

void launch_fem_sell_pack(int64_t n, const int64_t* krp, const int* kc, const double* kv, const int64_t* off,
                          double* sv, int* sc, cudaStream_t st) {
  if (n > 0) k_fem_sell_pack<<<nb(n), 256, 0, st>>>(n, krp, kc, kv, off, sv, sc);
}

void launch_fem_rhs_sell(int64_t n, const int64_t* off, const double* sv, const int* sc, const double* x,
                         const double* X, const double* v, const double* m, const double* g, double twodt, double* b,
                         cudaStream_t st) {
  if (n > 0) k_fem_rhs_sell<<<nb(n), 256, 0, st>>>(n, off, sv, sc, x, X, v, m, g, twodt, b);
}

size_t fem_detect_tmp_bytes(int64_t nodes) {
  size_t tb = 0;
  FlagIter it(thrust::counting_iterator<int64_t>(0), BelowMargin{nullptr, 0.0});
  cub::DeviceScan::ExclusiveSum(nullptr, tb, it, (int*)nullptr, (int)nodes);
  return tb;
}

int launch_fem_detect(int64_t nodes, int S, int nodes_per_scene, const double* x, const double* v, double margin,
                      void* tmp, size_t tmp_bytes, int* pos, int* cts, const double* frame, double mu,
                      double neg_beta_dt, double e_rest, double thr, int* ci, int* cj, double* frames, double* muv,
                      double* mu2v, double* phi, double* lam0, double* lam1, cudaStream_t st) {
  if (nodes <= 0) return 0;
  FlagIter it(thrust::counting_iterator<int64_t>(0), BelowMargin{x, margin});
  if (cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, it, pos, (int)nodes, st) != cudaSuccess) return 1;
  k_fem_detect<<<nb(nodes), 256, 0, st>>>(nodes, S, nodes_per_scene, pos, x, v, margin, frame, mu, neg_beta_dt,
                                          e_rest, thr, cts, ci, cj, frames, muv, mu2v, phi, lam0, lam1);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

void launch_fem_advance(int64_t n, double dt, const double* vh, double* x, double* v, double* warm, cudaStream_t st) {
  if (n > 0) k_fem_advance<<<nb(n), 256, 0, st>>>(n, dt, vh, x, v, warm);
}

// scenes by decreasing iteration count of their last solve, ties by index,
// into perm (one CTA of 1024 threads; S <= kMaxOrderedScenes): one block radix
// sort of the unique keys (inverted count | scene index)
__device__ __forceinline__ void scene_order_block(int S, const SolveStatus* __restrict__ st, int* __restrict__ perm) {
  constexpr int IPT = kMaxOrderedScenes / 1024;
  using Sort = cub::BlockRadixSort<unsigned, 1024, IPT>;
  __shared__ typename Sort::TempStorage tmp;
  unsigned key[IPT];
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const int sc = threadIdx.x * IPT + u;
    const unsigned it = (unsigned)min(max(sc < S ? st[sc].iterations : 0, 0), (1 << 20) - 1);
    key[u] = sc < S ? ((((1u << 20) - 1u - it) << 11) | (unsigned)sc) : 0xffffffffu;
  }
  Sort(tmp).Sort(key, 0, 32);
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const int r = threadIdx.x * IPT + u;  // blocked arrangement: thread t holds ranks t*IPT ..
    if (r < S) perm[r] = (int)(key[u] & 0x7ffu);
  }
}

// per-step counters of a device-driven run (vfpi_fem_run): integer sums, so
// the atomics give exact, order-independent totals
__global__ void __launch_bounds__(1024) k_fem_run_stats(int S, const SolveStatus* __restrict__ st, const int* __restrict__ cts, int step,
                                unsigned long long* __restrict__ acc, int* __restrict__ its_out,
                                int* __restrict__ cts_out, int* __restrict__ perm) {
  unsigned long long ci = 0, it = 0, dv = 0;
  int mx = 0;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int i = st[s].iterations;
    const int nc = cts[s + 1] - cts[s];
    ci += (unsigned long long)nc * (unsigned long long)i;
    it += (unsigned long long)i;
    dv += st[s].diverged ? 1ull : 0ull;
    mx = max(mx, i);
    if (its_out) its_out[(size_t)step * S + s] = i;
  }
  atomicAdd(acc + 0, ci);
  atomicAdd(acc + 1, it);
  atomicAdd(acc + 2, dv);
  atomicMax(acc + 3, (unsigned long long)mx);
  if (threadIdx.x == 0) {
    atomicAdd(acc + 4, (unsigned long long)cts[S]);
    if (cts_out) cts_out[step] = cts[S];
  }
  if (perm) scene_order_block(S, st, perm);  // the next step's longest-first scene order
}

__global__ void __launch_bounds__(1024) k_scene_order(int S, const SolveStatus* __restrict__ st, int* __restrict__ perm) {
  scene_order_block(S, st, perm);
}

void launch_fem_rhs_nodes(int S, int nn, int nsl, const int64_t* slice_off, const int* node_list,
                          const unsigned* kdesc, const double* kval, const double* x, const double* X,
                          const double* v, const double* m, const double* g, double twodt, double* b,
                          cudaStream_t st) {
  const int64_t ns = (int64_t)S * nsl;
  if (ns > 0)
    k_fem_rhs_nodes<<<(unsigned)((ns + 7) / 8), 256, 0, st>>>(ns, nn, nsl, slice_off, node_list, kdesc, kval, x, X, v,
                                                            m, g, twodt, b);
}

void launch_scene_order(int S, const SolveStatus* st, int* perm, cudaStream_t stream) {
  if (S > 0 && S <= kMaxOrderedScenes) k_scene_order<<<1, 1024, 0, stream>>>(S, st, perm);
}

__global__ void k_iota_int(int n, int* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

void launch_fem_run_stats(int S, const SolveStatus* st, const int* cts, int step, unsigned long long* acc,
                          int* its_out, int* cts_out, cudaStream_t stream, int* perm) {
  k_fem_run_stats<<<1, 1024, 0, stream>>>(S, st, cts, step, acc, its_out, cts_out,
                                          S <= kMaxOrderedScenes ? perm : nullptr);
}

void launch_iota_int(int n, int* v, cudaStream_t st) {
  if (n > 0) k_iota_int<<<nb(n), 256, 0, st>>>(n, v);
}

void launch_csr_matvec(int64_t rows, const int* rp, const int* ci, const double* cx, const double* x, double* y,
                       cudaStream_t st) {
  if (rows > 0) k_csr_matvec<<<nb(rows), 256, 0, st>>>(rows, rp, ci, cx, x, y);
}

}  // namespace vfpi
