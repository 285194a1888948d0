// V-FPI iteration, shared-memory-resident variant (the configs[1] path).
//
// Same algorithm and decision pipeline as vfpi_solve.cu (reference loop
// solver.py:388-446), but each CTA (one per SM) keeps its whole partition on
// chip for the lifetime of the launch:
//   * its rows' numeric entries (values + columns, CTA-contiguous CSR),
//     b, w, the contact frames and parameters, lam (both parities), J_c^T lam
//     and v* of contact rows -> only the x-gathers of the SpMV and the
//     v_next stores touch L2 per iteration;
//   * the SpMV is split in two passes so the gathers are fully parallel while
//     the row sums keep scipy's sequential order bit for bit:
//       pass A  prod[e] = a[e] * x[col[e]]   (all entries, 8 gathers in flight / thread)
//       pass B  acc(row) = (((0 + prod[k0]) + prod[k0+1]) + ...)   (one thread per row)
//   * the grid barrier is a flag barrier fused with the deterministic
//     residual reduction: every CTA publishes (theta^2, force^2, #nonfinite)
//     and an epoch flag; every CTA waits for all flags and sums the G partials
//     in the same fixed order, so decisions are identical everywhere.
#include <climits>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// fixed-order CTA sum of three doubles -> sm_out[0..2] (visible after the trailing barrier)
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
  if (warp == 0) {
    double x = lane < nw ? sm_warp[3 * lane + 0] : 0.0;
    double y = lane < nw ? sm_warp[3 * lane + 1] : 0.0;
    double z = lane < nw ? sm_warp[3 * lane + 2] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x = dadd(x, __shfl_xor_sync(0xffffffffu, x, o));
      y = dadd(y, __shfl_xor_sync(0xffffffffu, y, o));
      z = dadd(z, __shfl_xor_sync(0xffffffffu, z, o));
    }
    if (lane == 0) {
      sm_out[0] = x;
      sm_out[1] = y;
      sm_out[2] = z;
    }
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier fused with the deterministic reduction of three partial sums.
// Arrive: thread 0 stores the CTA's partials, then one release reduction on a
// monotonic counter (target epoch*G: no reset between barriers). Wait: thread
// 0 spins with acquire loads on that single word. Collect: warp 0 reads the G
// partials (<= 8 independent loads per lane) and reduces them in a fixed order
// that is identical in every CTA, so every CTA gets bit-identical totals.
constexpr int kMaxPartialsPerLane = 8;  // G <= 256
constexpr int kLPC = 4;                 // lanes per contact in the one-shot phase

__device__ __forceinline__ void grid_reduce3(double a, double b, double c, double* part, int off, unsigned* counter,
                                             int G, int epoch, double* sm_warp, double* sm_tot) {
  cta_reduce3(a, b, c, sm_warp, sm_tot);
  if (threadIdx.x == 0) {
    double* q = part + (size_t)blockIdx.x * kPartialStride + off;
    q[0] = sm_tot[0];
    q[1] = sm_tot[1];
    q[2] = sm_tot[2];
    red_release_add(counter, 1u);
    const unsigned target = (unsigned)epoch * (unsigned)G;
    const long long t0 = clock64();
    while (ld_acquire_u32(counter) < target) {
      if (clock64() - t0 > (1ll << 36)) __trap();  // ~30 s: never in a healthy run
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxPartialsPerLane; ++k) {
      const int g = lane + 32 * k;
      if (g < G) {
        const double* q = part + (size_t)g * kPartialStride + off;
        x = dadd(x, __ldcg(q + 0));
        y = dadd(y, __ldcg(q + 1));
        z = dadd(z, __ldcg(q + 2));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x = dadd(x, __shfl_xor_sync(0xffffffffu, x, o));
      y = dadd(y, __shfl_xor_sync(0xffffffffu, y, o));
      z = dadd(z, __shfl_xor_sync(0xffffffffu, z, o));
    }
    if (lane == 0) {
      sm_tot[0] = x;
      sm_tot[1] = y;
      sm_tot[2] = z;
    }
  }
  __syncthreads();
}

// pass A: prod[dst[i]] = a[i] * x(col[i]) over the CTA's column-sorted entries
// (neighbouring lanes gather neighbouring columns), UN gathers per thread in flight
template <class X>
__device__ __forceinline__ void products(const double* __restrict__ sv, const int* __restrict__ sc,
                                         const int* __restrict__ sd, double* __restrict__ prod, int E, X x) {
  constexpr int UN = 8;
  const int T = blockDim.x;
  for (int base = threadIdx.x; base < E; base += UN * T) {
    int c[UN];
    double xv[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = base + u * T;
      c[u] = i < E ? sc[i] : INT_MIN;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) xv[u] = c[u] != INT_MIN ? x(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = base + u * T;
      if (i < E) prod[sd[i]] = dmul(sv[i], xv[u]);
    }
  }
}

// pass B: sequential (scipy-order) sum of one row's products, loads batched by 4
__device__ __forceinline__ double row_sum(const double* __restrict__ prod, int k, int k1) {
  double acc = 0.0;
  for (; k + 4 <= k1; k += 4) {
    const double t0 = prod[k], t1 = prod[k + 1], t2 = prod[k + 2], t3 = prod[k + 3];
    acc = dadd(dadd(dadd(dadd(acc, t0), t1), t2), t3);
  }
  for (; k < k1; ++k) acc = dadd(acc, prod[k]);
  return acc;
}

template <int OP, bool CHEB, bool BB, bool HASC>
__global__ void __launch_bounds__(kResThreads, 1) k_iterate_res(IterParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double sm_warp[3 * (kResThreads / 32)];
  __shared__ double sm_tot[4];
  __shared__ unsigned long long sm_role_end[2];
  const int b = blockIdx.x, G = p.G, T = blockDim.x, tid = threadIdx.x;
  if (tid < 2) sm_role_end[tid] = 0;
  const int p0 = p.blk_row[b], p1 = p.blk_row[b + 1], R = p1 - p0;
  const int64_t e0 = p.pos_ptr[p0];
  const int E = (int)(p.pos_ptr[p1] - e0);
  const int c0 = p.blk_ct[b], c1 = p.blk_ct[b + 1], C = c1 - c0;
  const int CR = HASC ? p.blk_cr[b] : 0;  // rows [0, CR) belong to the CTA's contacts
  const ResLayout Lo(E, R, C, CR);        // this CTA's own footprint (launch size = max over CTAs)
  double* sv = reinterpret_cast<double*>(smraw + Lo.o_sv);
  double* prod = reinterpret_cast<double*>(smraw + Lo.o_prod);
  int* sc = reinterpret_cast<int*>(smraw + Lo.o_sc);
  int* sd = reinterpret_cast<int*>(smraw + Lo.o_sd);
  int* rp = reinterpret_cast<int*>(smraw + Lo.o_rp);
  int* rw = reinterpret_cast<int*>(smraw + Lo.o_row);
  double* bs = reinterpret_cast<double*>(smraw + Lo.o_b);
  double* ws = reinterpret_cast<double*>(smraw + Lo.o_w);
  double* vown = reinterpret_cast<double*>(smraw + Lo.o_v0);   // own rows of v^(l-1)
  double* vown2 = reinterpret_cast<double*>(smraw + Lo.o_v1);  // own rows of v^(l)
  int* cm = reinterpret_cast<int*>(smraw + Lo.o_cm);
  int* cq = reinterpret_cast<int*>(smraw + Lo.o_cq);
  double* cfr = reinterpret_cast<double*>(smraw + Lo.o_fr);
  double* cpar = reinterpret_cast<double*>(smraw + Lo.o_par);  // mu, mu2, phi, gamma
  double* lam_s = reinterpret_cast<double*>(smraw + Lo.o_lam); // [2][3C]
  double* vs_s = reinterpret_cast<double*>(smraw + Lo.o_vs);   // [CR]
  double* jt_s = reinterpret_cast<double*>(smraw + Lo.o_jt);   // [CR]

  // ---- stage the partition on chip (once per launch) --------------------
  for (int i = tid; i < E; i += T) {
    const int src = __ldg(p.ps_src + e0 + i);
    const int c = __ldg(p.ps_col + e0 + i);
    sc[i] = c;
    sd[i] = (int)(src - e0);
    sv[i] = __ldg(p.pk_val + src);
  }
  for (int q = tid; q < R; q += T) {
    const int row = __ldg(p.row_list + p0 + q);
    rp[q] = (int)(__ldg(p.pos_ptr + p0 + q) - e0);
    rw[q] = row;
    bs[q] = __ldg(p.b + row);
    ws[q] = __ldg(p.w + row);
    vown[q] = p.vbuf0[row];
  }
  if (tid == 0) rp[R] = E;
  for (int k = tid; k < C; k += T) {
    const int m = __ldg(p.cont_list + c0 + k);
    cm[k] = m;
    cq[k] = __ldg(p.cont_q + c0 + k) | (__ldg(p.col_j + m) >= 0 ? (1 << 30) : 0);
#pragma unroll
    for (int t = 0; t < 9; ++t) cfr[9 * k + t] = __ldg(p.frames + 9 * (size_t)m + t);
    cpar[4 * k + 0] = __ldg(p.mu + m);
    cpar[4 * k + 1] = __ldg(p.mu2 + m);
    cpar[4 * k + 2] = __ldg(p.phi + m);
    cpar[4 * k + 3] = __ldg(p.gamma + m);
  }
  for (int t = tid; t < 6 * C; t += T) lam_s[t] = 0.0;
  for (int t = tid; t < CR; t += T) jt_s[t] = 0.0;
  __syncthreads();

  // warps [0, WC) run the contact one-shots while warps [WC, nw) finish the free rows
  const int nw = T >> 5, warp = tid >> 5;
  // split the warps between the contact quads (kLPC lanes per contact) and the
  // free rows so both finish together: cost ~ rounds x per-round latency
  int WC = 0;
  if (C > 0) {
    const int FR = R - CR;
    if (FR == 0) {
      WC = nw;
    } else {
      const int efree = E - rp[CR];
      const long long kf = 8LL * (efree / FR + 1) + 200;  // cycles per free-row round
      long long best = LLONG_MAX;
      for (int w = 1; w < nw; ++w) {
        const long long tc = (long long)((C + (32 / kLPC) * w - 1) / ((32 / kLPC) * w)) * 1000;
        const long long tf = (long long)((FR + 32 * (nw - w) - 1) / (32 * (nw - w))) * kf;
        const long long c2 = tc > tf ? tc : tf;
        if (c2 < best) { best = c2; WC = w; }
      }
    }
  }

  double* vb[3] = {p.vbuf0, p.vbuf1, p.vbuf2};
  const double u = p.under_relax;
  const double omu = dsub(1.0, u);
  double rho = 0.0, nu = 1.0, theta_prev = 0.0;
  double alpha_prev = BB ? *p.w_mean : 0.0;
  double alpha = 0.0;
  bool pending = false;
  int final_buf = 0, final_lam = 0, iters = 0, conv = 0, div = 0;
  double consistency = NAN;
  int epoch = 0;

  for (int l = 1;; ++l) {
    const bool check_only = (l == p.max_iters + 1);
    const bool profl = p.prof != nullptr && l >= p.prof_iter0 && l < p.prof_iter0 + 4;
    auto stamp = [&](int k) {  // phase timestamps for tuning (off unless p.prof is set)
      if (profl) {
        __syncthreads();
        if (tid == 0) {
          long long g;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
          p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 8 + k] = k == 7 ? g : clock64();
        }
      }
    };
    stamp(0);
    const double* vcur = vb[(l - 1) % 3];   // written by other CTAs: coherent loads only
    const double* vprev = vb[(l + 1) % 3];  // v^(l-2)
    double* vnext = vb[l % 3];
    double* lam_out = lam_s + (l & 1) * 3 * C;
    double* part = p.partials + (size_t)(l & 1) * G * kPartialStride;

    // ---- Barzilai-Borwein scalar step (solver.py:389-400) ----------------
    bool use_alpha = false;
    if (BB && l >= 2 && !check_only) {
      products(sv, sc, sd, prod, E, [&](int c) { return dsub(vcur[c], vprev[c]); });
      __syncthreads();
      double sz = 0.0, ss = 0.0, zz = 0.0;
      for (int q = tid; q < R; q += T) {
        const double z = row_sum(prod, rp[q], rp[q + 1]);
        const int row = rw[q];
        const double s = dsub(vown[q], vprev[row]);
        sz = dadd(sz, dmul(s, z));
        ss = dadd(ss, dmul(s, s));
        zz = dadd(zz, dmul(z, z));
      }
      grid_reduce3(sz, ss, zz, part, 4, reinterpret_cast<unsigned*>(p.bar_flags), G, ++epoch, sm_warp, sm_tot);
      const double tsz = sm_tot[0], tss = sm_tot[1], tzz = sm_tot[2];
      const bool bb1 = (p.step == VFPI_STEP_BB1) || (p.step == VFPI_STEP_BB_ALTERNATING && (l % 2 == 0));
      if (tsz <= 0.0) alpha = alpha_prev;
      else alpha = bb1 ? ddiv(tss, tsz) : ddiv(tsz, tzz);
      alpha_prev = alpha;
      use_alpha = true;
      __syncthreads();  // prod and sm_tot are reused below
    }

    if (CHEB && !check_only) {  // solver.py:284-290, :417
      if (l < p.cheby_start) nu = 1.0;
      else if (l == p.cheby_start) nu = ddiv(2.0, dsub(2.0, dmul(rho, rho)));
      else nu = ddiv(4.0, dsub(4.0, dmul(dmul(rho, rho), nu)));
    }

    double th = 0.0, fr = 0.0, nf = 0.0;
    // v_new -> (Chebyshev) -> v_next of own row q; theta / finiteness partials
    auto finish_row = [&](int q, double vnew) {
      const double vc = vown[q];
      const int row = rw[q];
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
      vown2[q] = vn;
    };
    // r = A v - b of own row q; force residual of the previous iterate (solver.py:437-439)
    auto residual = [&](int q) {
      const double r = dsub(row_sum(prod, rp[q], rp[q + 1]), bs[q]);
      const double f = (q < CR) ? dsub(r, jt_s[q]) : dsub(r, 0.0);
      fr = dadd(fr, dmul(f, f));
      return r;
    };

    // ---- (1) surrogate-dynamics sweep: pass A gathers, pass B ordered sums --
    products(sv, sc, sd, prod, E, [&](int c) { return vcur[c]; });
    __syncthreads();
    stamp(2);
    // contact rows first: their v* feeds the contact one-shots
    for (int q = tid; q < CR; q += T) {
      const double r = residual(q);
      if (!check_only) vs_s[q] = dsub(vown[q], dmul(use_alpha ? alpha : ws[q], r));
    }
    __syncthreads();
    stamp(3);

    if (warp < WC) {
      // ---- (2)(3)(2') contacts: gather, one-shot projection, scatter ------
      // kLPC lanes per contact: lane a < 3 owns frame row / component a; the
      // projection needs all three components and is evaluated redundantly.
      if (HASC && !check_only) {
        const int lane = tid & 31;
        const int a = (lane & (kLPC - 1)) < 3 ? (lane & (kLPC - 1)) : 2;
        const bool owner = (lane & (kLPC - 1)) < 3;
        const int qbase = lane & ~(kLPC - 1);  // first lane of this contact's group
        for (int k0 = warp * (32 / kLPC); k0 < C; k0 += WC * (32 / kLPC)) {
          const int k = k0 + lane / kLPC;
          const bool act = k < C;
          const int kk = act ? k : k0;
          const int code = cq[kk];
          const int qb = code & 0x3fffffff;
          const bool dj = (code >> 30) & 1;
          const double* R9 = cfr + 9 * kk;
          double rel[3], vi_a, vj_a = 0.0;
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const double xi = vs_s[qb + t];
            rel[t] = dj ? dsub(xi, vs_s[qb + 3 + t]) : xi;
          }
          vi_a = vs_s[qb + a];
          if (dj) vj_a = vs_s[qb + 3 + a];
          // eta_a = R[a,:] rel  ((p0+p2)+p1, einsum order) ; lam*_a
          const double eta_a = dadd(dadd(dmul(R9[3 * a + 0], rel[0]), dmul(R9[3 * a + 2], rel[2])),
                                    dmul(R9[3 * a + 1], rel[1]));
          double g;
          if (use_alpha) g = dj ? dadd(dadd(alpha, alpha), p.omega) : dadd(alpha, p.omega);
          else g = cpar[4 * kk + 3];
          const double ls_a = ddiv(-dadd(eta_a, a == 0 ? cpar[4 * kk + 2] : 0.0), g);
          double lam[3];
          lam[0] = __shfl_sync(0xffffffffu, ls_a, qbase + 0);
          lam[1] = __shfl_sync(0xffffffffu, ls_a, qbase + 1);
          lam[2] = __shfl_sync(0xffffffffu, ls_a, qbase + 2);
          if (act) {
            project(OP, lam, cpar[4 * kk + 0], cpar[4 * kk + 1]);
            if (owner) {
              lam_out[3 * k + a] = lam[a];
              // world_a = R[:,a] . lam  ((p0+p1)+p2)
              const double wa = dadd(dadd(dmul(R9[a], lam[0]), dmul(R9[3 + a], lam[1])), dmul(R9[6 + a], lam[2]));
              const double oi = dadd(0.0, wa);  // np.add.at onto zeros
              jt_s[qb + a] = oi;
              finish_row(qb + a, dadd(vi_a, dmul(use_alpha ? alpha : ws[qb + a], oi)));
              if (dj) {
                const double oj = dsub(0.0, wa);  // np.subtract.at onto zeros
                jt_s[qb + 3 + a] = oj;
                finish_row(qb + 3 + a, dadd(vj_a, dmul(use_alpha ? alpha : ws[qb + 3 + a], oj)));
              }
            }
          }
        }
      }
    }
    if (profl && (tid & 31) == 0 && warp < WC) atomicMax(&sm_role_end[0], (unsigned long long)clock64());
    if (warp >= WC || WC == nw) {
      // ---- free rows: v_new = v* (+ w * 0 when contacts exist) ------------
      const int t0 = (WC == nw) ? tid : tid - WC * 32;
      const int TT = (WC == nw) ? T : T - WC * 32;
      for (int q = CR + t0; q < R; q += TT) {
        const double r = residual(q);
        if (!check_only) {
          const double wr = use_alpha ? alpha : ws[q];
          const double vstar = dsub(vown[q], dmul(wr, r));
          finish_row(q, HASC ? dadd(vstar, dmul(wr, 0.0)) : vstar);
        }
      }
    }

    if (profl && (tid & 31) == 0 && (warp >= WC || WC == nw)) atomicMax(&sm_role_end[1], (unsigned long long)clock64());
    // ---- (4) residual reduction + grid-wide decision --------------------
    stamp(4);
    if (profl && tid == 0) {
      p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 8 + 6] = (long long)sm_role_end[0];
      p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 8 + 1] = (long long)sm_role_end[1];
      sm_role_end[0] = 0;
      sm_role_end[1] = 0;
    }
    stamp(7);
    grid_reduce3(th, fr, nf, part, 0, reinterpret_cast<unsigned*>(p.bar_flags), G, ++epoch, sm_warp, sm_tot);
    stamp(5);
    const double theta = dsqrt(sm_tot[0]);
    const double fres = dsqrt(sm_tot[1]);
    const bool nonfinite = sm_tot[2] > 0.0;
    if (pending) {
      consistency = fres;
      if (fres <= dmul(p.cfactor, p.tol)) {
        iters = l - 1; conv = 1;
        final_buf = (l - 1) % 3; final_lam = (l - 1) & 1;
        break;
      }
    }
    if (check_only) {
      iters = p.max_iters;
      consistency = fres;
      final_buf = (l - 1) % 3; final_lam = (l - 1) & 1;
      break;
    }
    if (b == 0 && tid == 0) p.trace[l - 1] = theta;
    if (nonfinite) {
      iters = l; div = 1;
      final_buf = l % 3; final_lam = l & 1;
      break;
    }
    pending = theta < p.tol;
    if (CHEB) rho = (theta_prev <= 0.0) ? rho : py_min(ddiv(theta, theta_prev), 1.0);
    theta_prev = theta;
    double* tmp = vown;  // own rows of v^(l) become the current iterate
    vown = vown2;
    vown2 = tmp;
  }

  const double* vfin = vb[final_buf];
  for (int q = tid; q < R; q += T) p.out_v[rw[q]] = vfin[rw[q]];
  const double* lfin = lam_s + final_lam * 3 * C;
  for (int k = tid; k < C; k += T) {
    const int m = cm[k];
#pragma unroll
    for (int t = 0; t < 3; ++t) p.out_lam[3 * (size_t)m + t] = lfin[3 * k + t];
  }
  if (b == 0 && tid == 0) {
    p.status->iterations = iters;
    p.status->converged = conv;
    p.status->diverged = div;
    p.status->final_vbuf = final_buf;
    p.status->consistency = consistency;
  }
}

using KernelFn = void (*)(IterParams);

template <int OP>
KernelFn pick3(bool cheb, bool bb, bool hasc) {
  if (cheb) {
    if (bb) return hasc ? k_iterate_res<OP, true, true, true> : k_iterate_res<OP, true, true, false>;
    return hasc ? k_iterate_res<OP, true, false, true> : k_iterate_res<OP, true, false, false>;
  }
  if (bb) return hasc ? k_iterate_res<OP, false, true, true> : k_iterate_res<OP, false, true, false>;
  return hasc ? k_iterate_res<OP, false, false, true> : k_iterate_res<OP, false, false, false>;
}

KernelFn pick(int op, bool cheb, bool bb, bool hasc) {
  if (op == OP_PROXIMAL) return pick3<OP_PROXIMAL>(cheb, bb, hasc);
  if (op == OP_ANISO) return pick3<OP_ANISO>(cheb, bb, hasc);
  return pick3<OP_STRICT>(cheb, bb, hasc);
}

}  // namespace


int launch_iterate_resident(const IterParams& p, int op, bool cheb, bool bb, size_t smem_bytes, cudaStream_t st,
                            std::string& err) {
  KernelFn f = pick(op, cheb, bb, p.n_c > 0);
  cudaError_t e = ensure_max_dynamic_smem((const void*)f);
  if (e != cudaSuccess) { err = std::string("smem attribute: ") + cudaGetErrorString(e); return VFPI_CUDA_ERROR; }
  int nb = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kResThreads, smem_bytes);
  if (e != cudaSuccess || nb < 1) { err = "resident kernel does not fit on an SM"; return VFPI_UNSUPPORTED; }
  IterParams local = p;
  void* args[] = {&local};
  e = cudaLaunchCooperativeKernel((const void*)f, dim3(p.G), dim3(kResThreads), args, smem_bytes, st);
  if (e != cudaSuccess) {
    err = std::string("cooperative launch (resident): ") + cudaGetErrorString(e);
    return VFPI_CUDA_ERROR;
  }
  return VFPI_OK;
}

}  // namespace vfpi
