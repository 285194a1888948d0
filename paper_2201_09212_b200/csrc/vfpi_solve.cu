// The V-FPI iteration as ONE persistent cooperative kernel.
//
// Reference loop: solver.py:388-446 (post-loop :448-460). Per iteration l:
//   (1) surrogate-dynamics sweep  r = A v - b ; v* = v - w∘r          (:402-403)
//   (2) gather eta = J_c v*                                           (:405, contacts.py:402-411)
//   (3) one-shot projection per contact                               (:407, :262-281)
//   (2') scatter v_new = v* + w∘J_c^T lam                             (:411, contacts.py:414-423)
//   [Chebyshev blend]                                                 (:415-420, :429-430)
//   (4) theta = ||v_next - v||, finiteness, convergence test          (:422-446)
//
// B200 mapping. Each CTA owns a fixed slice of the row list in which every
// contact's 3 or 6 rows are co-located with the contact itself (built in
// vfpi_setup.cu), so steps (1)-(2')-(4) for a CTA need only its own rows:
//   * (1) is a SELL-32 sweep: a warp reads 32 rows' k-th entries as one
//     coalesced 256 B value + 128 B column load, each lane accumulating its
//     row sequentially (bit-exact to scipy's CSC matvec), v* of contact rows
//     staged in shared memory, free rows finished in registers;
//   * (2)(3)(2') run one thread per contact out of shared memory;
//   * (4) is a fixed-order CTA reduction -> per-CTA partial -> one grid
//     barrier -> every CTA reduces the partials in the same order, so all CTAs
//     take identical convergence decisions without a host round trip.
// The consistency check ||A v - b - J_c^T lam|| the reference runs when
// theta < tol (:434-444) reuses the NEXT iteration's sweep (r of the next
// iterate is exactly A v - b), so it costs no extra pass; the decision for
// iteration l is taken one barrier later, and v^(l), lam^(l) are kept in a
// 3-deep / 2-deep ring until then.
#include <cooperative_groups.h>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace cg = cooperative_groups;

#ifndef VFPI_SWEEP_RING
#define VFPI_SWEEP_RING 1  // scene batches: SELL stream through a TMA-fed shared-memory ring (see SellRing)
#endif

namespace vfpi {

namespace {

// fixed-order CTA sum of up to 3 doubles; result valid in sm_out[0..2] after return
__device__ __forceinline__ void cta_reduce3(double a, double b, double c, double* sm_warp, double* sm_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = dadd(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = dadd(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = dadd(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  if (lane == 0) {
    sm_warp[3 * warp + 0] = a;
    sm_warp[3 * warp + 1] = b;
    sm_warp[3 * warp + 2] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0, z = 0.0;
    for (int w = 0; w < nw; ++w) {
      x = dadd(x, sm_warp[3 * w + 0]);
      y = dadd(y, sm_warp[3 * w + 1]);
      z = dadd(z, sm_warp[3 * w + 2]);
    }
    sm_out[0] = x;
    sm_out[1] = y;
    sm_out[2] = z;
  }
  __syncthreads();
}

// every CTA reduces all G partials in the same fixed order (warp 0), result
// broadcast through shared memory
__device__ __forceinline__ void grid_totals(const double* __restrict__ part, int G, int off, double* sm_tot) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int g0 = lane; g0 < G; g0 += 32 * 4) {  // four partials per lane in flight
      double x[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int g = g0 + 32 * u;
        const double* q = part + (size_t)g * kPartialStride + off;
        x[u][0] = g < G ? __ldcg(q + 0) : 0.0;
        x[u][1] = g < G ? __ldcg(q + 1) : 0.0;
        x[u][2] = g < G ? __ldcg(q + 2) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (g0 + 32 * u < G) {
          a = dadd(a, x[u][0]);
          b = dadd(b, x[u][1]);
          c = dadd(c, x[u][2]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = dadd(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = dadd(b, __shfl_xor_sync(0xffffffffu, b, o));
      c = dadd(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
    if (lane == 0) {
      sm_tot[0] = a;
      sm_tot[1] = b;
      sm_tot[2] = c;
    }
  }
  __syncthreads();
}

// sequential SELL-32 row sum of one slice: acc = sum_k val[k] * x(col[k]),
// in increasing column order, FMA-free, starting from 0 (sparse.py:97-102).
#ifndef VFPI_SELL_UNROLL
#define VFPI_SELL_UNROLL 8
#endif
#ifndef VFPI_SC_MIN_BLOCKS
#define VFPI_SC_MIN_BLOCKS 4  // single-system kernel: 4 CTAs/SM (64 registers)
#endif
#ifndef VFPI_RING_MIN_BLOCKS
#define VFPI_RING_MIN_BLOCKS 3  // scene-batch kernel with the SELL ring: 3 CTAs/SM
#endif

template <class X>
__device__ __forceinline__ double sell_row(const double* __restrict__ sv, const int* __restrict__ sc, int64_t off,
                                           int W, int lane, X x) {
  constexpr int U = VFPI_SELL_UNROLL;
  double acc = 0.0;
  const double* vp = sv + off + lane;
  const int* cp = sc + off + lane;
  int k = 0;
  for (; k + U <= W; k += U) {
    int c[U];
    double a[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldcs(cp + 32 * (k + u));  // streamed once per iteration: evict-first,
      a[u] = __ldcs(vp + 32 * (k + u));  // so the gathered vectors stay in L2
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? x(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) acc = dadd(acc, dmul(a[u], xv[u]));
  }
  for (; k < W; ++k) {
    const int c = __ldcs(cp + 32 * k);
    if (c >= 0) acc = dadd(acc, dmul(__ldcs(vp + 32 * k), x(c)));
  }
  return acc;
}

// ---- SELL stream through a per-warp shared-memory ring (TMA bulk copies) ----
// Scene-batch kernels (SC; VFPI_SWEEP_RING): every warp streams its own SELL slices, in a fixed
// cyclic order that repeats every iteration (A does not change during a
// solve), as chunks of kRingChunk k-steps (32 rows x kRingChunk entries:
// 2 KB of values + 1 KB of columns) into kRingStages shared-memory stages
// with cp.async.bulk + mbarrier complete_tx. The copy engine keeps
// kRingStages chunks per warp in flight while the lanes gather x for the
// chunk they consume, so HBM streaming no longer waits on the gather
// latency, and the in-flight bytes cost no registers. Lane 0 refills a stage
// as soon as the warp has consumed it, including across the contact phase
// and the barrier (the next iteration's first chunks arrive early).
// Measured (B200): configs[2]-shaped batch 0.69 -> 0.74 of HBM peak with 2
// stages of 8 k-steps at 3 CTAs/SM; the single-system kernel keeps 4 CTAs/SM
// of register-fed loads, which the ring's smem cost would halve (configs[3]
// 0.65 -> 0.52-0.55, configs[4] 0.57 -> 0.54-0.58), so it streams directly.
#ifndef VFPI_RING_CHUNK
#define VFPI_RING_CHUNK 8
#endif
#ifndef VFPI_RING_STAGES
#define VFPI_RING_STAGES 2
#endif
constexpr int kRingChunk = VFPI_RING_CHUNK;
constexpr int kRingStages = VFPI_RING_STAGES;
constexpr int kRingChunkElems = kRingChunk * 32;
constexpr int kRingStageBytes = kRingChunkElems * 12;
constexpr int kRingBytes = VFPI_SWEEP_RING ? (kThreads / 32) * kRingStages * kRingStageBytes + 128 : 0;

__device__ __forceinline__ bool mbar_try_wait(unsigned addr, unsigned parity) {
  unsigned done;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done)
               : "r"(addr), "r"(parity)
               : "memory");
  return done != 0;
}

struct SellRing {
  double* val;     // [kRingStages][kRingChunkElems]
  int* col;        // [kRingStages][kRingChunkElems]
  unsigned bar0;   // shared address of this warp's first stage barrier
  int s_first;     // first slice of the warp (s0 + warp)
  int ps, pc;      // producer cursor: slice, chunk within the slice
  unsigned issued, consumed;
  bool work;       // the warp owns at least one non-empty slice
};

// lane 0: issue the chunk at the producer cursor into stage issued % kRingStages
// (every lane then advances its copy of `issued`)
__device__ __forceinline__ void ring_issue(SellRing& r, const IterParams& p, int s1, int nw, uint64_t pol) {
  int64_t off;
  int W;
  for (;;) {  // skip empty slices (r.work guarantees termination)
    off = p.slice_off[r.ps];
    W = (int)((p.slice_off[r.ps + 1] - off) >> 5);
    if (W > 0) break;
    r.ps += nw;
    if (r.ps >= s1) r.ps = r.s_first;
  }
  const int k0 = r.pc * kRingChunk;
  const int kk = min(kRingChunk, W - k0);
  const int stage = (int)(r.issued % kRingStages);
  const unsigned bar = r.bar0 + 8u * (unsigned)stage;
  const unsigned dv = (unsigned)__cvta_generic_to_shared(r.val + (size_t)stage * kRingChunkElems);
  const unsigned dc = (unsigned)__cvta_generic_to_shared(r.col + (size_t)stage * kRingChunkElems);
  const unsigned bv = (unsigned)kk * 32u * 8u, bc = (unsigned)kk * 32u * 4u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bv + bc) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dv), "l"(p.sell_val + off + 32 * (int64_t)k0), "r"(bv), "r"(bar), "l"(pol)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dc), "l"(p.sell_col + off + 32 * (int64_t)k0), "r"(bc), "r"(bar), "l"(pol)
      : "memory");
  ++r.pc;
  if (r.pc * kRingChunk >= W) {
    r.pc = 0;
    r.ps += nw;
    if (r.ps >= s1) r.ps = r.s_first;
  }
}

// sequential row sum of the warp's next slice (width W) out of the ring,
// same order and operations as sell_row
template <class X>
__device__ __forceinline__ double ring_row(SellRing& r, const IterParams& p, int W, int lane, int s1, int nw,
                                           uint64_t pol, X x) {
  double acc = 0.0;
  for (int k0 = 0; k0 < W; k0 += kRingChunk) {
    const int kk = min(kRingChunk, W - k0);
    const int stage = (int)(r.consumed % kRingStages);
    const unsigned bar = r.bar0 + 8u * (unsigned)stage;
    const unsigned par = (r.consumed / kRingStages) & 1u;
    while (!mbar_try_wait(bar, par)) {
    }
    const double* vs = r.val + (size_t)stage * kRingChunkElems + lane;
    const int* cs = r.col + (size_t)stage * kRingChunkElems + lane;
    if (kk == kRingChunk) {
      int c[kRingChunk];
      double a[kRingChunk], xv[kRingChunk];
#pragma unroll
      for (int u = 0; u < kRingChunk; ++u) {
        c[u] = cs[32 * u];
        a[u] = vs[32 * u];
      }
#pragma unroll
      for (int u = 0; u < kRingChunk; ++u) xv[u] = c[u] >= 0 ? x(c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kRingChunk; ++u)
        if (c[u] >= 0) acc = dadd(acc, dmul(a[u], xv[u]));
    } else {
      for (int u = 0; u < kk; ++u) {
        const int c = cs[32 * u];
        if (c >= 0) acc = dadd(acc, dmul(vs[32 * u], x(c)));
      }
    }
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ring_issue(r, p, s1, nw, pol);
    }
    ++r.issued;
    ++r.consumed;
  }
  return acc;
}

// SC = false: one system over a cooperative grid (grid barrier per iteration).
// SC = true : a batch of independent scenes, one CTA per scene (CTA b owns
//             scene b's rows and contacts); every CTA runs its own iteration
//             loop, reductions and termination with CTA barriers only.
template <bool SC>
constexpr bool kUseRing = SC && VFPI_SWEEP_RING;
template <bool SC>
constexpr int kRingSmem = kUseRing<SC> ? kRingBytes : 0;

template <int OP, bool CHEB, bool BB, bool HASC, bool SC>
__global__ void __launch_bounds__(kThreads, kUseRing<SC> ? VFPI_RING_MIN_BLOCKS : VFPI_SC_MIN_BLOCKS)
    k_iterate(IterParams p) {
  extern __shared__ double smem[];
  __shared__ double sm_warp[3 * (kThreads / 32)];
  __shared__ double sm_tot[4];

  const int b = blockIdx.x;
  const int G = p.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int p0 = p.blk_row[b], p1 = p.blk_row[b + 1];
  const int s0 = p.blk_slice[b], s1 = p.blk_slice[b + 1];
  const int c0 = p.blk_ct[b], c1 = p.blk_ct[b + 1];
  const int nct = c1 - c0;
  double* vs_s = smem;                         // v* of contact rows     [6*nct]
  double* jt_s = smem + kSlotsPerContact * nct;  // J_c^T lam_{l-1} rows   [6*nct]

  for (int t = threadIdx.x; t < kSlotsPerContact * nct; t += blockDim.x) jt_s[t] = 0.0;
  __shared__ __align__(8) uint64_t ring_bar[kUseRing<SC> ? kThreads / 32 : 1][kRingStages];
  uint64_t pol = 0;
  SellRing ring{};
  if constexpr (kUseRing<SC>) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const size_t cbytes = (size_t)2 * kSlotsPerContact * nct * sizeof(double);
    unsigned char* base = reinterpret_cast<unsigned char*>(smem) + ((cbytes + 127) & ~(size_t)127);
    unsigned char* mine = base + (size_t)warp * kRingStages * kRingStageBytes;
    ring.val = reinterpret_cast<double*>(mine);
    ring.col = reinterpret_cast<int*>(mine + (size_t)kRingStages * kRingChunkElems * sizeof(double));
    ring.bar0 = (unsigned)__cvta_generic_to_shared(&ring_bar[warp][0]);
    ring.s_first = s0 + warp;
    ring.ps = ring.s_first;
    ring.pc = 0;
    ring.issued = ring.consumed = 0;
    bool w = false;
    for (int s = s0 + warp; s < s1 && !w; s += nwarps) w = p.slice_off[s + 1] > p.slice_off[s];
    ring.work = w;
    if (lane == 0) {
      for (int st = 0; st < kRingStages; ++st)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ring.bar0 + 8u * (unsigned)st) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (w)
        for (int st = 0; st < kRingStages; ++st) {
          ring_issue(ring, p, s1, nwarps, pol);
          ++ring.issued;
        }
    }
    __syncwarp();
    ring.issued = w ? kRingStages : 0;  // lane 0's count, for every lane
  }
  __syncthreads();

  const double u = p.under_relax;
  const double omu = dsub(1.0, u);
  double rho = 0.0, nu = 1.0, theta_prev = 0.0;
  double alpha_prev = (BB && !SC) ? *p.w_mean : 0.0;
  double alpha = 0.0;
  bool fixed_scene_alpha = false;  // SC: fixed-alpha default 1/max|diag| of this scene
  if constexpr (SC) {
    // per-scene quantities the single-system setup computes globally:
    // BB fallback alpha = mean(w) (solver.py:381), fixed-alpha default (:368)
    double sw = 0.0, mx = -INFINITY, nanf = 0.0;
    for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
      const int row = __ldg(p.row_list + pos);
      sw = dadd(sw, __ldg(p.w + row));
      const double a = fabs(__ldg(p.diag + row));
      if (isnan(a)) nanf = 1.0;
      mx = a > mx ? a : mx;
    }
    // max |diag| over the scene: warp shuffles then warps in fixed order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = t > mx ? t : mx;
    }
    cta_reduce3(sw, 0.0, nanf, sm_warp, sm_tot);
    const double wsum = sm_tot[0], anynan = sm_tot[2];
    __syncthreads();
    if (lane == 0) sm_warp[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = -INFINITY;
      for (int w2 = 0; w2 < nwarps; ++w2) m = sm_warp[w2] > m ? sm_warp[w2] : m;
      sm_tot[3] = m;
    }
    __syncthreads();
    const double dmax = anynan > 0.0 ? NAN : sm_tot[3];
    const int nrows = p1 - p0;
    if (BB) alpha_prev = nrows > 0 ? ddiv(wsum, (double)nrows) : 0.0;
    if (p.step == VFPI_STEP_FIXED_ALPHA && p.fixed_alpha_default) {
      fixed_scene_alpha = true;
      alpha = ddiv(1.0, dmax);
    }
    __syncthreads();
  }
  double* trace = SC ? p.trace + (size_t)b * p.trace_stride : p.trace;
  SolveStatus* status = SC ? p.status + b : p.status;
  bool pending = false;       // theta_{l-1} < tol: consistency check due
  int final_buf = 0, final_lam = 0, iters = 0, conv = 0, div = 0;
  double consistency = NAN;

  for (int l = 1;; ++l) {
    const bool check_only = (l == p.max_iters + 1);
    // iterate buffers are written by other CTAs during the launch: plain
    // (coherent) loads only, never the read-only/nc path
    const double* vcur = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l - 1) % 3);
    const double* vprev = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l + 1) % 3);  // == v^(l-2)
    double* vnext = ring3(p.vbuf0, p.vbuf1, p.vbuf2, l % 3);
    double* __restrict__ lam_out = ring2(p.lam0, p.lam1, l & 1);
    double* part = p.partials + (size_t)(l & 1) * G * kPartialStride;

    // ---- Barzilai-Borwein scalar step (solver.py:389-400) ----------------
    bool use_alpha = fixed_scene_alpha;
    if (BB && l >= 2 && !check_only) {
      double sz = 0.0, ss = 0.0, zz = 0.0;
      for (int s = s0 + warp; s < s1; s += nwarps) {
        const int pos = p0 + (s - s0) * 32 + lane;
        const int64_t off = p.slice_off[s];
        const int W = (int)((p.slice_off[s + 1] - off) >> 5);
        const double z = sell_row(p.sell_val, p.sell_col, off, W, lane,
                                  [&](int c) { return dsub(vcur[c], vprev[c]); });
        if (pos < p1) {
          const int row = __ldg(p.row_list + pos);
          const double sv = dsub(vcur[row], vprev[row]);
          sz = dadd(sz, dmul(sv, z));
          ss = dadd(ss, dmul(sv, sv));
          zz = dadd(zz, dmul(z, z));
        }
      }
      cta_reduce3(sz, ss, zz, sm_warp, sm_tot);
      if constexpr (!SC) {
        if (threadIdx.x == 0) {
          part[(size_t)b * kPartialStride + 4] = sm_tot[0];
          part[(size_t)b * kPartialStride + 5] = sm_tot[1];
          part[(size_t)b * kPartialStride + 6] = sm_tot[2];
        }
        cg::this_grid().sync();
        grid_totals(part, G, 4, sm_tot);
      }
      const double tsz = sm_tot[0], tss = sm_tot[1], tzz = sm_tot[2];
      const bool bb1 = (p.step == VFPI_STEP_BB1) || (p.step == VFPI_STEP_BB_ALTERNATING && (l % 2 == 0));
      if (tsz <= 0.0) alpha = alpha_prev;
      else alpha = bb1 ? ddiv(tss, tsz) : ddiv(tsz, tzz);
      alpha_prev = alpha;
      use_alpha = true;
    }

    // ---- Chebyshev weight for this iteration (solver.py:284-290, :417) ----
    if (CHEB && !check_only) {
      if (l < p.cheby_start) nu = 1.0;
      else if (l == p.cheby_start) nu = ddiv(2.0, dsub(2.0, dmul(rho, rho)));
      else nu = ddiv(4.0, dsub(4.0, dmul(dmul(rho, rho), nu)));
    }

    double th = 0.0, fr = 0.0, nf = 0.0;
    auto finish_row = [&](int row, double vnew, double vc) {
      double vn = vnew;
      if (CHEB) {
        const double vss = dadd(dmul(u, vnew), dmul(omu, vc));
        if (l > 1) {
          const double vp = vprev[row];
          vn = dadd(dmul(nu, dsub(vss, vp)), vp);
        } else {
          vn = vss;
        }
      }
      const double d = dsub(vn, vc);
      th = dadd(th, dmul(d, d));
      if (!isfinite(vn)) nf = dadd(nf, 1.0);
      vnext[row] = vn;
    };

    // ---- (1) surrogate-dynamics sweep ------------------------------------
    for (int s = s0 + warp; s < s1; s += nwarps) {
      const int pos = p0 + (s - s0) * 32 + lane;
      const int64_t off = p.slice_off[s];
      const int W = (int)((p.slice_off[s + 1] - off) >> 5);
      // the row's own operands are independent of the row sum. The ring
      // kernels (registers to spare) issue their two levels of dependent
      // loads before the sweep so they land while the SELL stream is in
      // flight (configs[2] batch 0.74 -> 0.77 of HBM peak); the 64-register
      // single-system kernel loads them afterwards (early loads spill there:
      // configs[3] 0.65 -> 0.55)
      const bool live = pos < p1;
      int row = 0, slot = -1;
      double bv = 0.0, wv = 0.0, vc = 0.0;
      auto row_operands = [&] {
        if (live) {
          row = __ldg(p.row_list + pos);
          if (HASC) slot = __ldg(p.row_slot + pos);
          bv = __ldg(p.b + row);
          if (!use_alpha) wv = __ldg(p.w + row);
          vc = vcur[row];
        }
      };
      double y;
      if constexpr (kUseRing<SC>) {
        row_operands();
        y = ring_row(ring, p, W, lane, s1, nwarps, pol, [&](int c) { return vcur[c]; });
      } else {
        y = sell_row(p.sell_val, p.sell_col, off, W, lane, [&](int c) { return vcur[c]; });
        row_operands();
      }
      if (live) {
        const double r = dsub(y, bv);
        // force residual of the previous iterate (solver.py:437-439)
        const double f = (slot >= 0) ? dsub(r, jt_s[slot]) : dsub(r, 0.0);
        fr = dadd(fr, dmul(f, f));
        if (!check_only) {
          const double wr = use_alpha ? alpha : wv;
          const double vstar = dsub(vc, dmul(wr, r));
          if (slot >= 0) {
            vs_s[slot] = vstar;
          } else {
            const double vnew = HASC ? dadd(vstar, dmul(wr, 0.0)) : vstar;
            finish_row(row, vnew, vc);
          }
        }
      }
    }

    // ---- (2)(3)(2') contacts: gather, one-shot projection, scatter -------
    if (HASC && !check_only) {
      __syncthreads();
      for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
        const int m = __ldg(p.cont_list + k);
        const int loc = (k - c0) * kSlotsPerContact;
        const int ci = __ldg(p.col_i + m), cj = __ldg(p.col_j + m);
        double R[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) R[t] = __ldg(p.frames + 9 * (size_t)m + t);
        double vi[3], vj[3] = {0.0, 0.0, 0.0}, rel[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) vi[t] = vs_s[loc + t];
        if (cj >= 0) {
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            vj[t] = vs_s[loc + 3 + t];
            rel[t] = dsub(vi[t], vj[t]);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 3; ++t) rel[t] = vi[t];
        }
        double eta[3], lam[3], world[3];
        frame_apply(R, rel, eta);
        double g;
        if (use_alpha) g = (cj >= 0) ? dadd(dadd(alpha, alpha), p.omega) : dadd(alpha, p.omega);
        else g = __ldg(p.gamma + m);
        trial_impulse(eta, __ldg(p.phi + m), g, lam);
        project(OP, lam, __ldg(p.mu + m), __ldg(p.mu2 + m));
#pragma unroll
        for (int t = 0; t < 3; ++t) lam_out[3 * (size_t)m + t] = lam[t];
        frame_apply_t(R, lam, world);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int row = ci + t;
          const double oi = dadd(0.0, world[t]);
          jt_s[loc + t] = oi;
          const double wr = use_alpha ? alpha : __ldg(p.w + row);
          finish_row(row, dadd(vi[t], dmul(wr, oi)), vcur[row]);
        }
        if (cj >= 0) {
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int row = cj + t;
            const double oj = dsub(0.0, world[t]);
            jt_s[loc + 3 + t] = oj;
            const double wr = use_alpha ? alpha : __ldg(p.w + row);
            finish_row(row, dadd(vj[t], dmul(wr, oj)), vcur[row]);
          }
        }
      }
    }

    // ---- (4) residual reduction + grid-wide decision --------------------
    cta_reduce3(th, fr, nf, sm_warp, sm_tot);
    if constexpr (!SC) {
      if (threadIdx.x == 0) {
        part[(size_t)b * kPartialStride + 0] = sm_tot[0];
        part[(size_t)b * kPartialStride + 1] = sm_tot[1];
        part[(size_t)b * kPartialStride + 2] = sm_tot[2];
      }
      cg::this_grid().sync();
      grid_totals(part, G, 0, sm_tot);
    }
    const double theta = dsqrt(sm_tot[0]);
    const double fres = dsqrt(sm_tot[1]);  // ||A v^(l-1) - b - J_c^T lam^(l-1)||
    const bool nonfinite = sm_tot[2] > 0.0;

    if (pending) {  // decision for iterate l-1 (solver.py:434-444)
      consistency = fres;
      if (fres <= dmul(p.cfactor, p.tol)) {
        iters = l - 1; conv = 1;
        final_buf = (l - 1) % 3; final_lam = (l - 1) & 1;
        break;
      }
    }
    if (check_only) {  // l == max_iters + 1 (or max_iters == 0)
      iters = p.max_iters;
      consistency = fres;
      final_buf = (l - 1) % 3; final_lam = (l - 1) & 1;
      break;
    }
    if ((SC || b == 0) && threadIdx.x == 0) trace[l - 1] = theta;
    if (nonfinite) {  // DivergenceError (solver.py:424-427)
      iters = l; div = 1;
      final_buf = l % 3; final_lam = l & 1;
      break;
    }
    pending = theta < p.tol;
    if (CHEB) {
      rho = (theta_prev <= 0.0) ? rho : py_min(ddiv(theta, theta_prev), 1.0);
    }
    theta_prev = theta;
  }

  if constexpr (kUseRing<SC>) {  // drain the chunks in flight before the shared memory is released
    for (unsigned n = ring.consumed; n < ring.issued; ++n) {
      const unsigned bar = ring.bar0 + 8u * (n % kRingStages);
      while (!mbar_try_wait(bar, (n / kRingStages) & 1u)) {
      }
    }
  }
  // ---- outputs: each CTA copies its own rows / contacts -------------------
  const double* vfin = ring3(p.vbuf0, p.vbuf1, p.vbuf2, final_buf);
  for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
    const int row = __ldg(p.row_list + pos);
    p.out_v[row] = vfin[row];
  }
  const double* lfin = ring2(p.lam0, p.lam1, final_lam);
  for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
    const int m = __ldg(p.cont_list + k);
#pragma unroll
    for (int t = 0; t < 3; ++t) p.out_lam[3 * (size_t)m + t] = lfin[3 * (size_t)m + t];
  }
  if ((SC || b == 0) && threadIdx.x == 0) {
    status->iterations = iters;
    status->converged = conv;
    status->diverged = div;
    status->final_vbuf = final_buf;
    status->consistency = consistency;
  }
}

// post-loop SCC residuals (solver.py:453-455): eta = J_c v_final
__global__ void k_scc_final(int n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                            const double* __restrict__ frames, const double* __restrict__ v,
                            const double* __restrict__ lam, const double* __restrict__ phi,
                            const double* __restrict__ mu, double* scc) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  const int i = ci[m], j = cj[m];
  double rel[3], eta[3], l[3];
  for (int t = 0; t < 3; ++t) rel[t] = (j >= 0) ? dsub(v[i + t], v[j + t]) : v[i + t];
  frame_apply(frames + 9 * (size_t)m, rel, eta);
  for (int t = 0; t < 3; ++t) l[t] = lam[3 * (size_t)m + t];
  scc[m] = scc_one(eta, l, phi[m], mu[m]);
}

using KernelFn = void (*)(IterParams);

template <int OP, bool SC>
KernelFn pick3(bool cheb, bool bb, bool hasc) {
  if (cheb) {
    if (bb) return hasc ? k_iterate<OP, true, true, true, SC> : k_iterate<OP, true, true, false, SC>;
    return hasc ? k_iterate<OP, true, false, true, SC> : k_iterate<OP, true, false, false, SC>;
  }
  if (bb) return hasc ? k_iterate<OP, false, true, true, SC> : k_iterate<OP, false, true, false, SC>;
  return hasc ? k_iterate<OP, false, false, true, SC> : k_iterate<OP, false, false, false, SC>;
}

KernelFn pick(int op, bool cheb, bool bb, bool hasc, bool sc = false) {
  if (sc) {
    if (op == OP_PROXIMAL) return pick3<OP_PROXIMAL, true>(cheb, bb, hasc);
    if (op == OP_ANISO) return pick3<OP_ANISO, true>(cheb, bb, hasc);
    return pick3<OP_STRICT, true>(cheb, bb, hasc);
  }
  if (op == OP_PROXIMAL) return pick3<OP_PROXIMAL, false>(cheb, bb, hasc);
  if (op == OP_ANISO) return pick3<OP_ANISO, false>(cheb, bb, hasc);
  return pick3<OP_STRICT, false>(cheb, bb, hasc);
}

}  // namespace

int iterate_max_blocks_per_sm(int op, bool cheb, bool bb, int smem_bytes, bool scenes) {
  KernelFn f = pick(op, cheb, bb, true, scenes);
  if (ensure_max_dynamic_smem((const void*)f) != cudaSuccess) return 0;
  int nb = 0;
  const int ring = scenes ? kRingSmem<true> : kRingSmem<false>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kThreads, smem_bytes + ring) != cudaSuccess) return 0;
  return nb;
}

int launch_iterate(const IterParams& p, int op, bool cheb, bool bb, int smem_bytes, cudaStream_t st,
                   std::string& err) {
  KernelFn f = pick(op, cheb, bb, p.n_c > 0);
  {
    cudaError_t e = ensure_max_dynamic_smem((const void*)f);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return VFPI_CUDA_ERROR; }
  }
  IterParams local = p;
  void* args[] = {&local};
  cudaError_t e =
      cudaLaunchCooperativeKernel((const void*)f, dim3(p.G), dim3(kThreads), args, smem_bytes + kRingSmem<false>, st);
  if (e != cudaSuccess) {
    err = std::string("cooperative launch: ") + cudaGetErrorString(e);
    return VFPI_CUDA_ERROR;
  }
  return VFPI_OK;
}

int launch_iterate_scenes(const IterParams& p, int op, bool cheb, bool bb, int smem_bytes, cudaStream_t st,
                          std::string& err) {
  KernelFn f = pick(op, cheb, bb, p.n_c > 0, true);
  cudaError_t e = ensure_max_dynamic_smem((const void*)f);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return VFPI_CUDA_ERROR; }
  f<<<p.G, kThreads, smem_bytes + kRingSmem<true>, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("scene-batch launch: ") + cudaGetErrorString(e);
    return VFPI_CUDA_ERROR;
  }
  return VFPI_OK;
}

int launch_scc_final(const IterParams& p, double* scc, cudaStream_t st) {
  if (p.n_c <= 0) return VFPI_OK;
  k_scc_final<<<(p.n_c + 255) / 256, 256, 0, st>>>(p.n_c, p.col_i, p.col_j, p.frames, p.out_v, p.out_lam, p.phi,
                                                   p.mu, scc);
  return cudaGetLastError() == cudaSuccess ? VFPI_OK : VFPI_CUDA_ERROR;
}

}  // namespace vfpi
