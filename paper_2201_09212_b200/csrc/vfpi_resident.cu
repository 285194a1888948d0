// V-FPI iteration, shared-memory-resident variant (the configs[1] path).
//
// Same algorithm as vfpi_solve.cu (reference loop solver.py:388-446), but each
// CTA (one per SM) keeps its whole partition on chip for the lifetime of the
// launch: its rows' SELL-32 entries, b, w, its own rows of v, the contact
// frames / parameters, lam (both parities), J_c^T lam and v* of contact rows.
// Per iteration only two things cross L2:
//   * phase 1 stages, as whole 32-byte sectors, the entries of v^(l-1) the CTA
//     reads from other CTAs' rows (the sector list is fixed per solve, so the
//     ~5 scattered 8-byte gathers per entry become ~1 coalesced 32-byte load
//     per distinct sector, all in flight at once);
//   * v_next of its own rows is stored for the other CTAs.
// Row sums then run out of shared memory in scipy's sequential order (bit for
// bit), contacts run as lane quads beside the free rows, and one release
// reduction on a monotonic counter is the grid barrier. The residual partials
// of iteration l are reduced (in the same fixed order by every CTA) while the
// sectors of iteration l+1 are in flight, and the convergence decision for l
// is taken at the top of l+1.
#include <climits>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

constexpr int kMaxPartialsPerLane = 8;  // G <= 256

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// fixed-order CTA sum of three doubles -> sm_out[0..2] (visible after the next barrier)
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

// Arrive (publish this CTA's partials, release-add the counter) and wait until
// all G CTAs arrived at `epoch` (counter target epoch*G, never reset).
__device__ __forceinline__ void grid_arrive_wait(const double* sm_tot, double* part, int off, unsigned* counter,
                                                 int G, int epoch) {
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
}

// warp 0: fixed-order sum of the G published partials -> sm_tot[0..2]
// (roots: sm_tot[0..1] = square roots, the residual norms of the decision)
__device__ __forceinline__ void warp0_collect(const double* part, int off, int G, double* sm_tot, bool roots) {
  const int lane = threadIdx.x & 31;
  double px[kMaxPartialsPerLane], py[kMaxPartialsPerLane], pz[kMaxPartialsPerLane];
#pragma unroll
  for (int k = 0; k < kMaxPartialsPerLane; ++k) {  // all loads in flight first
    const int g = lane + 32 * k;
    const double* q = part + (size_t)g * kPartialStride + off;
    px[k] = g < G ? __ldcg(q + 0) : 0.0;
    py[k] = g < G ? __ldcg(q + 1) : 0.0;
    pz[k] = g < G ? __ldcg(q + 2) : 0.0;
  }
  double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
  for (int k = 0; k < kMaxPartialsPerLane; ++k) {
    if (lane + 32 * k < G) {
      x = dadd(x, px[k]);
      y = dadd(y, py[k]);
      z = dadd(z, pz[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x = dadd(x, __shfl_xor_sync(0xffffffffu, x, o));
    y = dadd(y, __shfl_xor_sync(0xffffffffu, y, o));
    z = dadd(z, __shfl_xor_sync(0xffffffffu, z, o));
  }
  if (lane == 0) {
    sm_tot[0] = roots ? dsqrt(x) : x;
    sm_tot[1] = roots ? dsqrt(y) : y;
    sm_tot[2] = z;
  }
}

// sequential (scipy-order) dot of one row with x: SELL element i = base + 32k,
// x from the staged sectors or from the CTA's own rows
#ifndef VFPI_ROW_UNROLL
#define VFPI_ROW_UNROLL 8  // free rows: 8 entries' loads in flight (measured best of 2/4/8/16)
#endif
#ifndef VFPI_ROW3_UNROLL
#define VFPI_ROW3_UNROLL 4
#endif
#ifndef VFPI_RES_FREE_START
#define VFPI_RES_FREE_START 1  // free-row warps start: 0 at once, 1 after the contact-row sweep
#endif
// x operand at a byte offset of the CTA's shared memory (the gather maps
// hold byte offsets, so a gather is one load with no index arithmetic)
__device__ __forceinline__ double xs_at(const unsigned char* sm, unsigned off) {
  return *reinterpret_cast<const double*>(sm + off);
}

__device__ __forceinline__ double row_dot(const double* __restrict__ sv, const unsigned* __restrict__ mp, int base,
                                          int len, const unsigned char* sm) {
  constexpr int U = VFPI_ROW_UNROLL;
  double acc = 0.0;
  int k = 0;
  for (; k + U <= len; k += U) {
    double a[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * (k + u);
      a[u] = sv[i];
      x[u] = xs_at(sm, mp[i]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = dadd(acc, dmul(a[u], x[u]));
  }
  for (; k < len; ++k) {
    const int i = base + 32 * k;
    acc = dadd(acc, dmul(sv[i], xs_at(sm, mp[i])));
  }
  return acc;
}

// three independent row sums at once (one contact side), each in scipy order
__device__ __forceinline__ void row_dot3(const double* __restrict__ sv, const unsigned* __restrict__ mp,
                                         const int* __restrict__ sb, const int* __restrict__ rlen,
                                         const unsigned char* sm, int q0, int q1, int q2, double* out) {
  const int qq[3] = {q0, q1, q2};
  int base[3], len[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    base[a] = sb[qq[a] >> 5] + (qq[a] & 31);
    len[a] = rlen[qq[a]];
  }
  const int L = max(len[0], max(len[1], len[2]));
  double acc[3] = {0.0, 0.0, 0.0};
  // branch-free: every lane loads (a row past its end re-reads its last
  // element) and only adds while k < len, so the three chains interleave
  for (int k = 0; k < L; k += VFPI_ROW3_UNROLL) {  // 12 independent loads per step (rows of <= 4 entries: one step)
    double pr[VFPI_ROW3_UNROLL][3];
    bool ok[VFPI_ROW3_UNROLL][3];
#pragma unroll
    for (int u = 0; u < VFPI_ROW3_UNROLL; ++u)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int kk = k + u;
        ok[u][a] = kk < len[a];
        const int i = base[a] + 32 * (ok[u][a] ? kk : 0);
        pr[u][a] = dmul(sv[i], xs_at(sm, mp[i]));
      }
#pragma unroll
    for (int u = 0; u < VFPI_ROW3_UNROLL; ++u)
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[a] = ok[u][a] ? dadd(acc[a], pr[u][a]) : acc[a];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) out[a] = acc[a];
}

// PROF: phase timestamps (tuning aid, scripts/prof_phases.py); compiled only
// into the configs[1] instantiation so the production kernels carry no checks
template <int OP, bool CHEB, bool BB, bool HASC, bool PROF = false>
__global__ void __launch_bounds__(kResThreads, 1) k_iterate_res(IterParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double sm_warp[3 * (kResThreads / 32)];
  __shared__ double sm_tot[4];
  __shared__ unsigned long long sm_role_end[8];
  const int b = blockIdx.x, G = p.G, T = blockDim.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  if (tid < 8) sm_role_end[tid] = 0;
  const int p0 = p.blk_row[b], p1 = p.blk_row[b + 1], R = p1 - p0;
  const int s0 = p.blk_slice[b], s1 = p.blk_slice[b + 1];
  const int64_t ep0 = p.slice_off[s0];
  const int EP = (int)(p.slice_off[s1] - ep0);
  const int c0 = p.blk_ct[b], c1 = p.blk_ct[b + 1], C = c1 - c0;
  const int CR = HASC ? p.blk_cr[b] : 0;  // rows [0, CR) belong to the CTA's contacts
  const int sec0 = p.sec_ptr[b];
  const int NS = p.sec_ptr[b + 1] - sec0;
  const ResLayout Lo(EP, R, C, CR, NS);  // this CTA's own footprint (launch size = max over CTAs)
  double* sv = reinterpret_cast<double*>(smraw + Lo.o_sv);
  unsigned* mp = reinterpret_cast<unsigned*>(smraw + Lo.o_map);
  double* xs = reinterpret_cast<double*>(smraw + Lo.o_xs);
  unsigned* sec = reinterpret_cast<unsigned*>(smraw + Lo.o_sec);
  int* sb = reinterpret_cast<int*>(smraw + Lo.o_sb);
  int* rlen = reinterpret_cast<int*>(smraw + Lo.o_len);
  int* rw = reinterpret_cast<int*>(smraw + Lo.o_row);
  double* bs = reinterpret_cast<double*>(smraw + Lo.o_b);
  double* ws = reinterpret_cast<double*>(smraw + Lo.o_w);
  double* vown = reinterpret_cast<double*>(smraw + Lo.o_v0);   // own rows of v^(l-1) (= xs + 4 NS)
  double* vown2 = reinterpret_cast<double*>(smraw + Lo.o_v1);  // own rows of v^(l)
  int* cm = reinterpret_cast<int*>(smraw + Lo.o_cm);
  int* cq = reinterpret_cast<int*>(smraw + Lo.o_cq);
  // contact data component-major ([t][C]): the lane that owns contact k reads
  // consecutive words with its neighbours (no bank conflicts; a [k][t] layout
  // strides 72 B / 32 B / 24 B across lanes)
  double* cfr = reinterpret_cast<double*>(smraw + Lo.o_fr);    // [9][C]
  double* cpar = reinterpret_cast<double*>(smraw + Lo.o_par);  // [4][C]: mu, mu2, phi, gamma
  double* lam_s = reinterpret_cast<double*>(smraw + Lo.o_lam); // [2][3][C]
  double* jt_s = reinterpret_cast<double*>(smraw + Lo.o_jt);   // [CR]
  unsigned* counter = reinterpret_cast<unsigned*>(p.bar_flags);

  // ---- stage the partition on chip (once per launch) --------------------
  for (int i = tid; i < EP; i += T) {
    sv[i] = __ldg(p.sell_val + ep0 + i);
    mp[i] = __ldg(p.sell_map + ep0 + i);
  }
  for (int j = tid; j < NS; j += T) sec[j] = __ldg(p.secs + sec0 + j);
  for (int s = tid; s <= s1 - s0; s += T) sb[s] = (int)(__ldg(p.slice_off + s0 + s) - ep0);
  for (int q = tid; q < R; q += T) {
    const int row = __ldg(p.row_list + p0 + q);
    rlen[q] = (int)(__ldg(p.pos_ptr + p0 + q + 1) - __ldg(p.pos_ptr + p0 + q));
    rw[q] = row;
    bs[q] = __ldg(p.b + row);
    ws[q] = __ldg(p.w + row);
    vown[q] = p.vbuf0[row];
  }
  for (int k = tid; k < C; k += T) {
    const int m = __ldg(p.cont_list + c0 + k);
    cm[k] = m;
    cq[k] = __ldg(p.cont_q + c0 + k) | (__ldg(p.col_j + m) >= 0 ? (1 << 30) : 0);
#pragma unroll
    for (int t = 0; t < 9; ++t) cfr[t * C + k] = __ldg(p.frames + 9 * (size_t)m + t);
    cpar[0 * C + k] = __ldg(p.mu + m);
    cpar[1 * C + k] = __ldg(p.mu2 + m);
    cpar[2 * C + k] = __ldg(p.phi + m);
    cpar[3 * C + k] = __ldg(p.gamma + m);
  }
  for (int t = tid; t < 6 * C; t += T) lam_s[t] = 0.0;
  for (int t = tid; t < CR; t += T) jt_s[t] = 0.0;
  __syncthreads();
  // gather map -> byte offsets of the x operands
  for (int i = tid; i < EP; i += T) mp[i] = (unsigned)Lo.o_xs + 8u * mp[i];
  __syncthreads();

  // split the warps: [0, WC) run one contact per lane (its rows, the one-shot
  // projection and the scatter), [WC, nw) sweep the free rows
  int WC = 0;
  if (C > 0) {
    WC = (C + 31) / 32;
    if (WC > nw - 1 && R > CR) WC = nw - 1;
    if (WC > nw) WC = nw;
  }
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
    const bool profl = PROF && p.prof != nullptr && l >= p.prof_iter0 && l < p.prof_iter0 + 4;
    auto stamp = [&](int k) {  // phase timestamps for tuning (off unless p.prof is set)
      if (profl) {
        __syncthreads();
        if (tid == 0) {
          long long g;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
          p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 16 + k] = k == 7 ? g : clock64();
        }
      }
    };
    stamp(0);
    const double* vcur = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l - 1) % 3);   // written by other CTAs: coherent loads only
    const double* vprev = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l + 1) % 3);  // v^(l-2)
    double* vnext = ring3(p.vbuf0, p.vbuf1, p.vbuf2, l % 3);
    double* lam_out = lam_s + (l & 1) * 3 * C;

    // ---- phase 1: stage the remote sectors of v^(l-1); reduce partials of l-1
    {
      // warps 1.. stage with asynchronous global->shared copies (two 16-byte
      // cp.async per sector, no register round trip); warp 0 reduces the
      // partials and takes the roots meanwhile
      const int TS = T - 32;
      if (warp > 0) {
        const unsigned xs_sh = (unsigned)__cvta_generic_to_shared(xs);
        for (int j = tid - 32; j < NS; j += TS) {
          // only the 16-byte halves the CTA's entries read (marks from k_sell_map)
          const unsigned sj = sec[j];
          const double* src = vcur + 4 * (size_t)(sj & kSecIdMask);
          const unsigned d = xs_sh + 32u * (unsigned)j;
          if (sj & (1u << 30))
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
          if (sj & (1u << 31))
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16u), "l"(src + 2) : "memory");
        }
        // own rows of v^(l-1) (written last iteration) join the x array
        if (l > 1)
          for (int q = tid - 32; q < R; q += TS) vown[q] = vown2[q];
        asm volatile("cp.async.wait_all;" ::: "memory");
      } else if (l > 1) {
        warp0_collect(p.partials + (size_t)((l - 1) & 1) * G * kPartialStride, 0, G, sm_tot, true);
      }
    }
    __syncthreads();
    stamp(2);

    // ---- decision for iteration l-1 (solver.py:422-446) -------------------
    if (l > 1) {
      const int lp = l - 1;
      const double theta = sm_tot[0];  // theta_{l-1} (square roots taken by warp 0)
      const double fres = sm_tot[1];   // ||A v^(l-2) - b - J_c^T lam^(l-2)||
      const bool nonfinite = sm_tot[2] > 0.0;
      if (pending) {
        consistency = fres;
        if (fres <= dmul(p.cfactor, p.tol)) {
          iters = lp - 1; conv = 1;
          final_buf = (lp - 1) % 3; final_lam = (lp - 1) & 1;
          break;
        }
      }
      if (lp == p.max_iters + 1) {
        iters = p.max_iters;
        consistency = fres;
        final_buf = (lp - 1) % 3; final_lam = (lp - 1) & 1;
        break;
      }
      if (b == 0 && tid == 0) p.trace[lp - 1] = theta;
      if (nonfinite) {
        iters = lp; div = 1;
        final_buf = lp % 3; final_lam = lp & 1;
        break;
      }
      pending = theta < p.tol;
      if (CHEB) rho = (theta_prev <= 0.0) ? rho : py_min(ddiv(theta, theta_prev), 1.0);
      theta_prev = theta;
    }
    double* part = p.partials + (size_t)(l & 1) * G * kPartialStride;

    // ---- Barzilai-Borwein scalar step (solver.py:389-400) ----------------
    bool use_alpha = false;
    if (BB && l >= 2 && !check_only) {
      double sz = 0.0, ss = 0.0, zz = 0.0;
      for (int q = tid; q < R; q += T) {
        // z = A s with s = v - v_prev gathered from global (BB is not a hot configuration)
        const int base = sb[q >> 5] + (q & 31);
        double z = 0.0;
        for (int k = 0; k < rlen[q]; ++k) {
          const int i = base + 32 * k;
          const unsigned m = (mp[i] - (unsigned)Lo.o_xs) >> 3;
          const int g = (m >= 4u * (unsigned)NS) ? rw[m - 4u * (unsigned)NS]
                                                 : (int)(4u * (sec[m >> 2] & kSecIdMask) + (m & 3u));
          z = dadd(z, dmul(sv[i], dsub(vcur[g], vprev[g])));
        }
        const double s = dsub(vown[q], vprev[rw[q]]);
        sz = dadd(sz, dmul(s, z));
        ss = dadd(ss, dmul(s, s));
        zz = dadd(zz, dmul(z, z));
      }
      cta_reduce3(sz, ss, zz, sm_warp, sm_tot);
      __syncthreads();
      grid_arrive_wait(sm_tot, part, 4, counter, G, ++epoch);
      if (warp == 0) warp0_collect(part, 4, G, sm_tot, false);
      __syncthreads();
      const double tsz = sm_tot[0], tss = sm_tot[1], tzz = sm_tot[2];
      const bool bb1 = (p.step == VFPI_STEP_BB1) || (p.step == VFPI_STEP_BB_ALTERNATING && (l % 2 == 0));
      if (tsz <= 0.0) alpha = alpha_prev;
      else alpha = bb1 ? ddiv(tss, tsz) : ddiv(tsz, tzz);
      alpha_prev = alpha;
      use_alpha = true;
      __syncthreads();  // sm_tot is reused below
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
          const double vpv = vprev[row];
          vn = dadd(dmul(nu, dsub(vss, vpv)), vpv);
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
      const double r = dsub(row_dot(sv, mp, sb[q >> 5] + (q & 31), rlen[q], smraw), bs[q]);
      const double f = (q < CR) ? dsub(r, jt_s[q]) : dsub(r, 0.0);
      fr = dadd(fr, dmul(f, f));
      return r;
    };

    // ---- (1)-(3): contact lanes -- sweep of the contact's rows, one-shot
    // projection, scatter -- beside the free-row warps ----------------------
    stamp(3);
    if (warp < WC) {
      const int CD = CR / 3 - C;  // two-sided contacts of the CTA
      for (int k0 = warp * 32; k0 < C; k0 += WC * 32) {  // warp-uniform trip count
        const int k = k0 + lane;
        const bool act = k < C;
        const int kc = act ? k : 0;
        const int code = cq[kc];
        const bool dj = (code >> 30) & 1;
        const int kd = code & 0x3fffffff;
        int qs[6];
        qs[0] = kc;
        qs[1] = C + kc;
        qs[2] = 2 * C + kc;
        qs[3] = 3 * C + kd;
        qs[4] = qs[3] + CD;
        qs[5] = qs[4] + CD;
        // (1) surrogate-dynamics sweep of the contact's rows (3 chains at a time)
        double vsr[6];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !dj) break;
          double dot[3];
          row_dot3(sv, mp, sb, rlen, smraw, qs[3 * h], qs[3 * h + 1], qs[3 * h + 2], dot);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int q = qs[3 * h + a];
            const double r = dsub(dot[a], bs[q]);
            const double f = dsub(r, jt_s[q]);
            if (act) fr = dadd(fr, dmul(f, f));
            vsr[3 * h + a] = dsub(vown[q], dmul(use_alpha ? alpha : ws[q], r));
          }
        }
        // the free-row warps start once every contact's rows are swept (they
        // would otherwise take the issue slots the contact lanes' chains need)
        if (VFPI_RES_FREE_START == 1 && k0 == warp * 32 && WC < nw) asm volatile("bar.arrive 2, %0;" ::"r"(T) : "memory");
        if (profl) { __syncwarp(); if (lane == 0) atomicMax(&sm_role_end[2], (unsigned long long)clock64()); }
        if (!act || !HASC || check_only) continue;
        // (2) gather + (3) one-shot projection (solver.py:262-281)
        double R9[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) R9[t] = cfr[t * C + k];
        double rel[3], eta[3], lam[3], wv[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) rel[t] = dj ? dsub(vsr[t], vsr[3 + t]) : vsr[t];
        frame_apply(R9, rel, eta);
        double g;
        if (use_alpha) g = dj ? dadd(dadd(alpha, alpha), p.omega) : dadd(alpha, p.omega);
        else g = cpar[3 * C + k];
        trial_impulse(eta, cpar[2 * C + k], g, lam);
        project(OP, lam, cpar[0 * C + k], cpar[1 * C + k]);
#pragma unroll
        for (int t = 0; t < 3; ++t) lam_out[t * C + k] = lam[t];
        // (2') scatter J_c^T lam and v_new = v* + w J_c^T lam
        frame_apply_t(R9, lam, wv);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int q = qs[a];
          const double oi = dadd(0.0, wv[a]);  // np.add.at onto zeros
          jt_s[q] = oi;
          finish_row(q, dadd(vsr[a], dmul(use_alpha ? alpha : ws[q], oi)));
        }
        if (dj) {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int q = qs[3 + a];
            const double oj = dsub(0.0, wv[a]);  // np.subtract.at onto zeros
            jt_s[q] = oj;
            finish_row(q, dadd(vsr[3 + a], dmul(use_alpha ? alpha : ws[q], oj)));
          }
        }
        if (profl) { __syncwarp(__activemask()); if ((tid & 31) == __ffs(__activemask()) - 1) atomicMax(&sm_role_end[4], (unsigned long long)clock64()); }
      }
      if (profl && lane == 0) atomicMax(&sm_role_end[0], (unsigned long long)clock64());
    }
    if (VFPI_RES_FREE_START == 1 && warp >= WC && WC > 0 && WC < nw) asm volatile("bar.sync 2, %0;" ::"r"(T) : "memory");
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
      if (profl && lane == 0) atomicMax(&sm_role_end[1], (unsigned long long)clock64());
    }

    // ---- (4) residual partials + grid barrier (reduction at the top of l+1)
    stamp(4);
    if (profl && tid == 0) {
      p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 16 + 6] = (long long)sm_role_end[0];
      p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 16 + 1] = (long long)sm_role_end[1];
      for (int t = 2; t < 5; ++t) p.prof[((size_t)b * 4 + (l - p.prof_iter0)) * 16 + 6 + t] = (long long)sm_role_end[t];
      for (int t = 0; t < 8; ++t) sm_role_end[t] = 0;
    }
    stamp(7);
    {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        th = dadd(th, __shfl_xor_sync(0xffffffffu, th, o));
        fr = dadd(fr, __shfl_xor_sync(0xffffffffu, fr, o));
        nf = dadd(nf, __shfl_xor_sync(0xffffffffu, nf, o));
      }
      if (lane == 0) {
        sm_warp[3 * warp + 0] = th;
        sm_warp[3 * warp + 1] = fr;
        sm_warp[3 * warp + 2] = nf;
      }
      __syncthreads();
      if (warp == 0) {  // fixed-order tree over the warps' partials
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
          sm_tot[0] = x;
          sm_tot[1] = y;
          sm_tot[2] = z;
        }
      }
    }
    grid_arrive_wait(sm_tot, part, 0, counter, G, ++epoch);
    stamp(5);
  }

  const double* vfin = ring3(p.vbuf0, p.vbuf1, p.vbuf2, final_buf);
  for (int q = tid; q < R; q += T) p.out_v[rw[q]] = vfin[rw[q]];
  const double* lfin = lam_s + final_lam * 3 * C;
  for (int k = tid; k < C; k += T) {
    const int m = cm[k];
#pragma unroll
    for (int t = 0; t < 3; ++t) p.out_lam[3 * (size_t)m + t] = lfin[t * C + k];
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
  if (p.prof != nullptr && op == OP_STRICT && !cheb && !bb && p.n_c > 0)
    f = k_iterate_res<OP_STRICT, false, false, true, true>;
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
