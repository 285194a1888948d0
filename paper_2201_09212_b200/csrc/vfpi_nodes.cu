// Scene-batch V-FPI iteration over a NODE-BLOCK SELL layout (FEM batches).
//
// Same iteration as k_iterate<..., SC=true> (vfpi_solve.cu; reference loop
// solver.py:388-446): one CTA per scene, the scene's own loop, reductions and
// termination with CTA barriers only. What changes is how the surrogate sweep
// r = A v - b (sparse.py:97-102, solver.py:402-403) streams A:
//
//   * one lane per FEM NODE (its 3 rows), 32 nodes per slice, nodes of a scene
//     ordered by decreasing block count so slices are dense;
//   * the k-th entry of a lane is a 3x3 BLOCK: one 32-bit descriptor (global
//     block column | 9-bit mask of the entries A actually stores) and the 9
//     values row-major (zeros where absent), stored [k][lane] and
//     [k][9][lane] per slice, so a warp's k-step is one 128 B + nine 256 B
//     coalesced lines;
//   * the slice stream goes through a per-warp shared-memory ring fed by TMA
//     bulk copies (cp.async.bulk + mbarrier complete_tx, evict-first), as in
//     the row-SELL ring of the scene kernel.
//
// Row p of node i sums its present entries block by block in increasing block
// column and, inside a block, in increasing column: exactly increasing column
// order, sequential, FMA-free from 0 -- the same bits as scipy's CSC matvec.
// A block moves 4 + 72 B for up to 9 stored entries (8.4 B per entry when
// full) instead of 12 B per entry of the row layout, the three x values of a
// block column are gathered once for three rows, and three row sums per lane
// are independent chains. Contacts (S-contacts on node rows, FEM) are handled
// exactly as in k_iterate: v* of a contact node's rows is staged in shared
// memory, then one thread per contact gathers, projects and scatters.
//
// Only the fixed-order reductions of theta and the force residual visit rows
// in a different order than the row kernel (both are the GPU's own fixed
// order; the reference's are OpenBLAS dots), so v and lam are bit-identical
// to the row kernel's for the same iteration count.
#include <cooperative_groups.h>

#include <climits>
#include <vector>

#include <cub/cub.cuh>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace cg = cooperative_groups;

#ifndef VFPI_NB_CHUNK
#define VFPI_NB_CHUNK 2  // k-steps (node blocks) per ring stage
#endif
#ifndef VFPI_NB_STAGES
#define VFPI_NB_STAGES 2
#endif
#ifndef VFPI_NB_WARPS
#define VFPI_NB_WARPS 8
#endif
#ifndef VFPI_NB_MIN_BLOCKS
#define VFPI_NB_MIN_BLOCKS 2
#endif

#ifdef VFPI_NB_DEBUG
#define NB_CHECK(cond, fmt, ...)                                                             \
  do {                                                                                       \
    if (!(cond)) printf("NB_CHECK %s:%d b=%d t=%d " fmt "\n", __FILE__, __LINE__, (int)blockIdx.x, \
                        (int)threadIdx.x, __VA_ARGS__);                                      \
  } while (0)
#else
#define NB_CHECK(cond, fmt, ...) \
  do {                           \
  } while (0)
#endif

namespace vfpi {

namespace {

constexpr int kNbThreads = 32 * VFPI_NB_WARPS;
constexpr int kNbChunk = VFPI_NB_CHUNK;
constexpr int kNbStages = VFPI_NB_STAGES;
constexpr int kDescBytes = 32 * 4;          // one k-step of descriptors
constexpr int kValBytes = 9 * 32 * 8;       // one k-step of block values
constexpr int kNbStageBytes = kNbChunk * (kDescBytes + kValBytes);
// packed block values (single-system grid layouts): a stage takes as many
// k-steps (<= kNbPackMax) as its kNbChunk k-steps of value space hold, so
// sparse blocks put more x gathers in flight per stage wait
#ifndef VFPI_NB_PACKMAX
#define VFPI_NB_PACKMAX 3
#endif
constexpr int kNbPackMax = VFPI_NB_PACKMAX;
constexpr int kNbGridStageBytes = kNbPackMax * kDescBytes + kNbChunk * kValBytes;
template <bool GRID>
__host__ __device__ constexpr int nb_stage_bytes() { return GRID ? kNbGridStageBytes : kNbStageBytes; }
template <bool GRID>
__host__ __device__ constexpr int nb_desc_area() { return GRID ? kNbPackMax * kDescBytes : kNbChunk * kDescBytes; }
constexpr int kNbRingBytes = VFPI_NB_WARPS * kNbStages * kNbStageBytes + 128;
constexpr unsigned kMaskShift = 23;
constexpr unsigned kColMask = (1u << kMaskShift) - 1u;

__device__ __forceinline__ bool nb_try_wait(unsigned addr, unsigned parity) {
  unsigned done;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done)
               : "r"(addr), "r"(parity)
               : "memory");
  return done != 0;
}

__device__ __forceinline__ void cta_sum3(double a, double b, double c, double* sm_warp, double* sm_out) {
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

struct NbRing {
  unsigned char* base;  // this warp's stages
  unsigned short* e1;   // packed layouts: per stage [kNbPackMax]: k-steps in the stage, then the value
                        // offset (doubles) of its k-steps 1.. in the stage
  bool nodesc;          // block columns come from the FEM template (no descriptor stream)
  unsigned bar0;
  int s0, s_end, nw, w;    // the CTA's slices [s0, s_end); this warp w takes one per round of nw (serpentine)
  int pr, pc;              // producer cursor: round, chunk within the slice
  int64_t p_off;           // the producer slice's k-step offset and width
  int p_W;
  unsigned vo_sa;          // packed grids: shared address of the prefetched value offsets [kNbPackMax + 1]
  unsigned issued, consumed;
  bool work;
};

// the warp's slice of round k: rounds alternate direction (serpentine), so
// with slices sorted by decreasing width every warp gets a wide and a narrow
// one in turn (a CTA barrier waits for its busiest warp)
__device__ __forceinline__ int nb_slice(int s0, int nw, int w, int k) {
  return s0 + k * nw + ((k & 1) ? nw - 1 - w : w);
}

template <bool GRID>
__device__ __forceinline__ void nb_issue(NbRing& r, const NodeLayoutDev& L, uint64_t pol) {
  int64_t off = GRID ? r.p_off : 0;
  int W = GRID ? r.p_W : 0;
  if (!GRID || r.pc == 0) {  // grids: only a new slice is looked up (mid-slice stages reuse its offset and width)
    for (;;) {
      const int ps = nb_slice(r.s0, r.nw, r.w, r.pr);
      if (ps >= r.s_end) {  // past the warp's last slice: wrap to the next iteration's first
        r.pr = 0;
        continue;
      }
      off = L.slice_off[ps];
      W = (int)(L.slice_off[ps + 1] - off);
      if (W > 0) break;
      ++r.pr;
    }
    if (GRID) {
      r.p_off = off;
      r.p_W = W;
    }
  }
  const int k0 = r.pc;  // k-step of the slice the stage starts at
  int kk = min(kNbChunk, W - k0);
  const int stage = (int)(r.issued % kNbStages);
  const unsigned bar = r.bar0 + 8u * (unsigned)stage;
  unsigned char* sb = r.base + (size_t)stage * nb_stage_bytes<GRID>();
  const unsigned dd = (unsigned)__cvta_generic_to_shared(sb);
  const unsigned dv = (unsigned)__cvta_generic_to_shared(sb + nb_desc_area<GRID>());
  unsigned bv;
  const double* vsrc;
  if (GRID && L.voff) {  // packed: k-step k holds E_k (<= 9) value slots per lane
    // the value offsets of the stage's candidate k-steps, loaded together (one
    // latency on the issuing lane's path instead of one per k-step)
    int64_t vo[kNbPackMax + 1];
    if (k0 != 0) {  // mid-slice: the previous issue prefetched them into shared memory
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int j = 0; j <= kNbPackMax; ++j)
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(vo[j]) : "r"(r.vo_sa + 8u * (unsigned)j) : "memory");
    } else {
#pragma unroll
      for (int j = 0; j <= kNbPackMax; ++j) vo[j] = L.voff[off + min(k0 + j, W)];
    }
    const int64_t v0 = vo[0];
    kk = 1;
#pragma unroll
    for (int j = 1; j < kNbPackMax; ++j)
      if (kk == j && k0 + j < W && 8 * (vo[j + 1] - v0) <= kNbChunk * kValBytes) {
        r.e1[kNbPackMax * stage + j] = (unsigned short)(vo[j] - v0);
        kk = j + 1;
      }
    r.e1[kNbPackMax * stage] = (unsigned short)kk;
    int64_t vend = vo[1];
#pragma unroll
    for (int j = 2; j <= kNbPackMax; ++j) vend = kk == j ? vo[j] : vend;
    bv = (unsigned)(8 * (vend - v0));
    vsrc = L.val + v0;
  } else {
    bv = (unsigned)kk * kValBytes;
    vsrc = L.val + (off + k0) * (9 * 32);
  }
  const unsigned bd = r.nodesc ? 0u : (unsigned)kk * kDescBytes;  // FEM batches: template columns
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bd + bv) : "memory");
  if (bd > 0)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dd), "l"(L.desc + (off + k0) * 32), "r"(bd), "r"(bar), "l"(pol)
        : "memory");
  if (bv > 0)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dv), "l"(vsrc), "r"(bv), "r"(bar), "l"(pol)
        : "memory");
  r.pc += kk;
  if (r.pc >= W) {
    r.pc = 0;
    ++r.pr;
  }
  else if (GRID && L.voff) {
    // packed: the next issue's value offsets (same slice) on their way to
    // shared memory now, so that issue does not wait for them
#pragma unroll
    for (int j = 0; j <= kNbPackMax; ++j)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(r.vo_sa + 8u * (unsigned)j),
                   "l"(L.voff + off + min(r.pc + j, W))
                   : "memory");
  }
}

// the three row sums of this lane's node over its slice (width W) out of the ring
// (PACKED: a block's present entries sit at consecutive value slots, rank order)
// tcs (FEM batches): the template block columns of this lane's slice (+ lane),
// node0 the scene's first global node. Every one of the 9 slots of a block is
// then added: slots A does not store hold +0, and +0 * x (x finite: every
// iterate the sweep reads is finite, a non-finite one ends the solve first)
// is a signed zero that leaves a row sum unchanged -- a sum that starts at +0
// is never -0 under round-to-nearest -- so the bits equal the masked sum.
template <bool MAYPACK, class X>
__device__ __forceinline__ void nb_rows(NbRing& r, const NodeLayoutDev& L, int W, int lane, uint64_t pol, X x,
                                        double& y0, double& y1, double& y2, int nrows_dbg,
                                        const int* __restrict__ tcs = nullptr, int node0 = 0,
                                        const double* xv = nullptr) {
  // MAYPACK = grid mode (its stage layout; packed values when L.voff is set)
  const bool packed = MAYPACK && L.voff != nullptr;
  constexpr int CHM = MAYPACK ? kNbPackMax : kNbChunk;  // k-steps a stage may hold
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  // template columns: the block columns of a stage are loaded a stage ahead,
  // and its x gathers are issued before the wait for its values (neither
  // depends on the stream); a k-step past the slice repeats the last one's
  int bcn[kNbChunk];
  if (!MAYPACK && tcs) {
#pragma unroll
    for (int u = 0; u < kNbChunk; ++u) bcn[u] = __ldg(tcs + 32 * min(u, W - 1));
  }
  for (int k0 = 0, kk = 0; k0 < W; k0 += kk) {
    double xt[kNbChunk][3];
    if (!MAYPACK && tcs) {
#pragma unroll
      for (int u = 0; u < kNbChunk; ++u) {
        const int c = 3 * (node0 + (bcn[u] < 0 ? 0 : bcn[u]));
        xt[u][0] = x(c);
        xt[u][1] = x(c + 1);
        xt[u][2] = x(c + 2);
      }
#pragma unroll
      for (int u = 0; u < kNbChunk; ++u) bcn[u] = __ldg(tcs + 32 * min(k0 + kNbChunk + u, W - 1));
    }
    const int stage = (int)(r.consumed % kNbStages);
    const unsigned bar = r.bar0 + 8u * (unsigned)stage;
    const unsigned par = (r.consumed / kNbStages) & 1u;
    while (!nb_try_wait(bar, par)) {
    }
    kk = packed ? (int)r.e1[kNbPackMax * stage] : min(kNbChunk, W - k0);
    const unsigned char* sb = r.base + (size_t)stage * nb_stage_bytes<MAYPACK>();
    const unsigned* ds = reinterpret_cast<const unsigned*>(sb) + lane;
    const double* vs = reinterpret_cast<const double*>(sb + nb_desc_area<MAYPACK>()) + lane;
    if (tcs) {
#pragma unroll
      for (int u = 0; u < kNbChunk; ++u) {
        if (u < kk) {
          const double x0 = xt[u][0], x1 = xt[u][1], x2 = xt[u][2];
          const double* v = vs + 9 * 32 * u;
          a0 = dadd(a0, dmul(v[32 * 0], x0));
          a0 = dadd(a0, dmul(v[32 * 1], x1));
          a0 = dadd(a0, dmul(v[32 * 2], x2));
          a1 = dadd(a1, dmul(v[32 * 3], x0));
          a1 = dadd(a1, dmul(v[32 * 4], x1));
          a1 = dadd(a1, dmul(v[32 * 5], x2));
          a2 = dadd(a2, dmul(v[32 * 6], x0));
          a2 = dadd(a2, dmul(v[32 * 7], x1));
          a2 = dadd(a2, dmul(v[32 * 8], x2));
        }
      }
    } else {
    // the stage's x gathers first (all of its k-steps' loads in flight at once:
    // absent blocks and k-steps past kk gather column 0 and are masked out),
    // then the sums
    unsigned dsc[CHM];
    double xg[CHM][3];
#pragma unroll
    for (int u = 0; u < CHM; ++u) {
      dsc[u] = u < kk ? ds[32 * u] : 0u;
      const int c = (dsc[u] >> kMaskShift) ? 3 * (int)(dsc[u] & kColMask) : 0;
      NB_CHECK(c + 2 < nrows_dbg, "gather c=%d n=%d d=%u", c, nrows_dbg, dsc[u]);
      // the node's three x values as two aligned 16-byte loads (two LSU
      // requests per block instead of three): doubles [c & ~1, +4) hold
      // c .. c+2 whatever c's parity; the iterate buffers are 32-byte aligned
      // and padded past n (vfpi_api.cu npad), so the fourth double exists
      {
        const double* xa = xv + (c & ~1);
        const double2 q0 = *reinterpret_cast<const double2*>(xa);
        const double2 q1 = *reinterpret_cast<const double2*>(xa + 2);
        const bool odd = c & 1;
        xg[u][0] = odd ? q0.y : q0.x;
        xg[u][1] = odd ? q1.x : q0.y;
        xg[u][2] = odd ? q1.y : q1.x;
      }
    }
#pragma unroll
    for (int u = 0; u < CHM; ++u) {
      if (u < kk) {
        const unsigned m = dsc[u] >> kMaskShift;
        if (m) {
          const double x0 = xg[u][0], x1 = xg[u][1], x2 = xg[u][2];
          if (packed) {
            const double* v = vs + (u == 0 ? 0 : (int)r.e1[kNbPackMax * stage + u]);
            int q = 0;  // rank of the entry among the block's present entries
            if (m & 0x001) { a0 = dadd(a0, dmul(v[32 * q], x0)); ++q; }
            if (m & 0x002) { a0 = dadd(a0, dmul(v[32 * q], x1)); ++q; }
            if (m & 0x004) { a0 = dadd(a0, dmul(v[32 * q], x2)); ++q; }
            if (m & 0x008) { a1 = dadd(a1, dmul(v[32 * q], x0)); ++q; }
            if (m & 0x010) { a1 = dadd(a1, dmul(v[32 * q], x1)); ++q; }
            if (m & 0x020) { a1 = dadd(a1, dmul(v[32 * q], x2)); ++q; }
            if (m & 0x040) { a2 = dadd(a2, dmul(v[32 * q], x0)); ++q; }
            if (m & 0x080) { a2 = dadd(a2, dmul(v[32 * q], x1)); ++q; }
            if (m & 0x100) a2 = dadd(a2, dmul(v[32 * q], x2));
          } else {
            const double* v = vs + 9 * 32 * u;
            if (m & 0x001) a0 = dadd(a0, dmul(v[32 * 0], x0));
            if (m & 0x002) a0 = dadd(a0, dmul(v[32 * 1], x1));
            if (m & 0x004) a0 = dadd(a0, dmul(v[32 * 2], x2));
            if (m & 0x008) a1 = dadd(a1, dmul(v[32 * 3], x0));
            if (m & 0x010) a1 = dadd(a1, dmul(v[32 * 4], x1));
            if (m & 0x020) a1 = dadd(a1, dmul(v[32 * 5], x2));
            if (m & 0x040) a2 = dadd(a2, dmul(v[32 * 6], x0));
            if (m & 0x080) a2 = dadd(a2, dmul(v[32 * 7], x1));
            if (m & 0x100) a2 = dadd(a2, dmul(v[32 * 8], x2));
          }
        }
      }
    }
    }
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      nb_issue<MAYPACK>(r, L, pol);
    }
    ++r.issued;
    ++r.consumed;
  }
  y0 = a0;
  y1 = a1;
  y2 = a2;
}

// every CTA reduces all G partials in the same fixed order (warp 0)
__device__ __forceinline__ void nb_grid_totals(const double* __restrict__ part, int G, double* sm_tot) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int g0 = lane; g0 < G; g0 += 32 * 4) {
      double x[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int g = g0 + 32 * u;
        const double* q = part + (size_t)g * kPartialStride;
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

// MODE kScene  : a batch of independent scenes, CTA b = scene b (its own loop,
//                contacts staged in shared memory, CTA barriers only);
// MODE kGrid   : one system over a cooperative grid, CTA b owns a range of node
//                slices; v* / J_c^T lam of contact rows go through global
//                arrays, so an iteration is sweep | grid barrier | contacts |
//                grid barrier (reductions), and every CTA takes the same
//                decision from the same fixed-order totals;
// MODE kCluster: a batch of scenes, one thread-block CLUSTER per scene (when
//                the batch is too small to fill the GPU, e.g. a rank's shard
//                at 8 GPUs): the scene's node slices split over the cluster's
//                CTAs, contacts through global slots, cluster barriers, and the
//                partials summed over distributed shared memory in rank order.
constexpr int kScene = 0, kGrid = 1, kCluster = 2;

template <int OP, bool CHEB, bool HASC, int MODE>
__global__ void __launch_bounds__(kNbThreads, VFPI_NB_MIN_BLOCKS) k_iterate_nodes(IterParams p, NodeLayoutDev L) {
  extern __shared__ double smem[];
  __shared__ double sm_warp[3 * (kNbThreads / 32)];
  __shared__ double sm_tot[4];
  __shared__ __align__(8) uint64_t ring_bar[kNbThreads / 32][kNbStages];
  __shared__ unsigned short ring_e1[kNbThreads / 32][kNbStages * kNbPackMax];
  __shared__ __align__(16) long long ring_vo[kNbThreads / 32][kNbPackMax + 1];

  // contact slots (v* / J_c^T lam of contact rows, 6 per contact, global index)
  // live in global memory in every mode: single-node contacts are solved inline
  // by the node's lane, so the slots see a few doubles per contact and iteration,
  // and the kernel's shared memory does not depend on the contact count
  constexpr bool GRID = MODE == kGrid, CLUSTER = MODE == kCluster, SHARED_C = false;
  __shared__ double sm_cpart[2][4];  // cluster mode: this CTA's partials, by iteration parity
  const int crank = CLUSTER ? (int)cg::this_cluster().block_rank() : 0;
  const int csize = CLUSTER ? (int)cg::this_cluster().num_blocks() : 1;
  // scene batches: CTA / cluster c runs scene scene_perm[c] (longest predicted
  // first); b = the layout's CTA index of this CTA's share of that scene
  const int cid = CLUSTER ? (int)blockIdx.x / csize : (int)blockIdx.x;
  const int scene = (!GRID && L.scene_perm) ? __ldg(L.scene_perm + cid) : cid;
  const int b = CLUSTER ? scene * csize + crank : (GRID ? (int)blockIdx.x : scene);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int np0 = L.blk_pos[b], np1 = L.blk_pos[b + 1];      // node positions of the CTA
  const int s0 = L.blk_slice[b], s1 = L.blk_slice[b + 1];    // node slices of the CTA
  const int c0 = GRID ? 0 : p.blk_ct[scene], c1 = GRID ? p.n_c : p.blk_ct[scene + 1];
  const int nct = SHARED_C ? c1 - c0 : 0;
  double* vs_s = SHARED_C ? smem : L.vs_g;                       // v* of contact rows    [6*contacts]
  double* jt_s = SHARED_C ? smem + kSlotsPerContact * nct : L.jt_g;  // J_c^T lam_{l-1} rows
  if (SHARED_C)
    for (int t = threadIdx.x; t < kSlotsPerContact * nct; t += blockDim.x) jt_s[t] = 0.0;

  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  NbRing ring{};
  {
    const size_t cbytes = (size_t)2 * kSlotsPerContact * nct * sizeof(double);
    unsigned char* base = reinterpret_cast<unsigned char*>(smem) + ((cbytes + 127) & ~(size_t)127);
    ring.base = base + (size_t)warp * kNbStages * nb_stage_bytes<GRID>();
    ring.bar0 = (unsigned)__cvta_generic_to_shared(&ring_bar[warp][0]);
    ring.e1 = &ring_e1[warp][0];
    ring.vo_sa = (unsigned)__cvta_generic_to_shared(&ring_vo[warp][0]);
    // FEM batches (one CTA or one cluster per scene): block columns from the batch's
    // template, loaded a stage ahead, instead of a streamed descriptor
    ring.nodesc = !GRID && L.tcol != nullptr;
    ring.s0 = s0;
    ring.s_end = s1;
    ring.nw = nwarps;
    ring.w = warp;
    ring.pr = 0;
    bool w = false;
    for (int k = 0, s = nb_slice(s0, nwarps, warp, 0); s < s1 && !w; s = nb_slice(s0, nwarps, warp, ++k))
      w = L.slice_off[s + 1] > L.slice_off[s];
    ring.work = w;
    if (lane == 0) {
      for (int st = 0; st < kNbStages; ++st)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ring.bar0 + 8u * (unsigned)st) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (w)
        for (int st = 0; st < kNbStages; ++st) {
          nb_issue<GRID>(ring, L, pol);
          ++ring.issued;
        }
    }
    __syncwarp();
    ring.issued = w ? kNbStages : 0;
  }
  __syncthreads();

  const double u = p.under_relax;
  const double omu = dsub(1.0, u);
  double rho = 0.0, nu = 1.0, theta_prev = 0.0;
  double alpha = 0.0;
  bool use_alpha = false;
  if (!GRID && p.step == VFPI_STEP_FIXED_ALPHA && p.fixed_alpha_default) {
    // scene batches: fixed-alpha default 1 / max|diag| of the scene (solver.py:368),
    // over the CTA's nodes and, for a cluster, over the cluster's CTAs;
    // a single system gets it from the setup (w filled with alpha)
    double mx = -INFINITY, nanf = 0.0;
    for (int pos = np0 + threadIdx.x; pos < np1; pos += blockDim.x) {
      const int node = __ldg(L.node_list + pos);
      for (int q = 0; q < 3; ++q) {
        const double a = fabs(__ldg(p.diag + 3 * node + q));
        if (isnan(a)) nanf = 1.0;
        mx = a > mx ? a : mx;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = t > mx ? t : mx;
    }
    cta_sum3(0.0, 0.0, nanf, sm_warp, sm_tot);
    const double anynan_cta = sm_tot[2];
    __syncthreads();
    if (lane == 0) sm_warp[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = -INFINITY;
      for (int w2 = 0; w2 < nwarps; ++w2) m = sm_warp[w2] > m ? sm_warp[w2] : m;
      sm_cpart[0][0] = m;
      sm_cpart[0][1] = anynan_cta;
    }
    __syncthreads();
    if constexpr (CLUSTER) cg::this_cluster().sync();
    double m = sm_cpart[0][0], anynan = sm_cpart[0][1];
    if constexpr (CLUSTER) {
      m = -INFINITY;
      anynan = 0.0;
      for (int r = 0; r < csize; ++r) {
        const double* q = cg::this_cluster().map_shared_rank(&sm_cpart[0][0], r);
        m = q[0] > m ? q[0] : m;
        anynan = q[1] > anynan ? q[1] : anynan;
      }
      cg::this_cluster().sync();  // sm_cpart is reused by the reductions below
    }
    alpha = ddiv(1.0, anynan > 0.0 ? NAN : m);
    use_alpha = true;
    __syncthreads();
  }
  double* trace = GRID ? p.trace : p.trace + (size_t)scene * p.trace_stride;
  SolveStatus* status = GRID ? p.status : p.status + scene;
  const bool writer = GRID ? (b == 0) : crank == 0;  // the CTA that writes trace / status
  bool pending = false;
  int final_buf = 0, final_lam = 0, iters = 0, conv = 0, div = 0;
  double consistency = NAN;

  for (int l = 1;; ++l) {
    const bool check_only = (l == p.max_iters + 1);
    const double* vcur = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l - 1) % 3);
    const double* vprev = ring3(p.vbuf0, p.vbuf1, p.vbuf2, (l + 1) % 3);
    double* vnext = ring3(p.vbuf0, p.vbuf1, p.vbuf2, l % 3);
    double* __restrict__ lam_out = ring2(p.lam0, p.lam1, l & 1);
    double* part = p.partials + (size_t)(l & 1) * p.G * kPartialStride;

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

    // ---- (1) surrogate sweep, one lane per node -------------------------
    // grids: the next slice's width is loaded a slice ahead (the sweep of a
    // slice starts with a wait on its width otherwise)
    // so is the lane's node of the next slice (its b, w, v and contact slot
    // loads start with a wait on it otherwise)
    int w_next = 0, node_next = 0;
    {
      const int sf = nb_slice(s0, nwarps, warp, 0);
      if (GRID && sf < s1) w_next = (int)(L.slice_off[sf + 1] - L.slice_off[sf]);
      const int pf = np0 + (sf - s0) * 32 + lane;
      if (sf < s1 && pf < np1) node_next = __ldg(L.node_list + pf);
    }
    for (int k = 0, s = nb_slice(s0, nwarps, warp, 0); s < s1; s = nb_slice(s0, nwarps, warp, ++k)) {
      const int pos = np0 + (s - s0) * 32 + lane;
      const int64_t off = GRID ? 0 : L.slice_off[s];
      const int W = GRID ? w_next : (int)(L.slice_off[s + 1] - off);
      const bool live = pos < np1;
      int node = 0, slot = -1;
      if (live) node = node_next;
      {
        const int sn = nb_slice(s0, nwarps, warp, k + 1);
        if (GRID) w_next = sn < s1 ? (int)(L.slice_off[sn + 1] - L.slice_off[sn]) : 0;
        const int pn = np0 + (sn - s0) * 32 + lane;
        if (sn < s1 && pn < np1) node_next = __ldg(L.node_list + pn);
      }
      double bv[3] = {0.0, 0.0, 0.0}, wv[3] = {0.0, 0.0, 0.0}, vc[3] = {0.0, 0.0, 0.0};
      if (live) {
        NB_CHECK(node >= 0 && 3 * node + 2 < p.n, "node=%d np0=%d np1=%d pos=%d", node, np0, np1, pos);
        if (HASC) slot = L.node_slot[node];
        NB_CHECK(slot < 0 || !SHARED_C || slot + 2 < kSlotsPerContact * nct, "slot=%d nct=%d node=%d", slot, nct,
                 node);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          bv[q] = __ldg(p.b + 3 * node + q);
          if (!use_alpha) wv[q] = __ldg(p.w + 3 * node + q);
          vc[q] = vcur[3 * node + q];
        }
      }
      double y[3];
      if (W > 0)
        nb_rows<GRID>(ring, L, W, lane, pol, [&](int c) { return vcur[c]; }, y[0], y[1], y[2], p.n,
                      (!GRID && L.tcol) ? L.tcol + (off - (int64_t)scene * L.k_scene) * 32 + lane : nullptr,
                      scene * L.nn, vcur);
      else y[0] = y[1] = y[2] = 0.0;
      if (live) {
        double vstar[3], wrq[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double r = dsub(y[q], bv[q]);
          const double f = (slot >= 0) ? dsub(r, jt_s[slot + q]) : dsub(r, 0.0);
          fr = dadd(fr, dmul(f, f));
          wrq[q] = use_alpha ? alpha : wv[q];
          vstar[q] = dsub(vc[q], dmul(wrq[q], r));
          if (!check_only && slot < 0) {
            const double vnew = HASC ? dadd(vstar[q], dmul(wrq[q], 0.0)) : vstar[q];
            finish_row(3 * node + q, vnew, vc[q]);
          }
        }
        if (HASC && !check_only && slot >= 0) {
          // an S-contact (single node) is solved right here by the node's lane:
          // its one-shot projection needs only this node's v* (contacts.py:402-423,
          // solver.py:405-411); two-node contacts are staged for the contact phase
          const int k = slot / kSlotsPerContact + (SHARED_C ? c0 : 0);
          const int m = GRID ? k : __ldg(p.cont_list + k);
          if (slot % kSlotsPerContact == 0 && __ldg(p.col_j + m) < 0) {
            double R[9];
#pragma unroll
            for (int t = 0; t < 9; ++t) R[t] = __ldg(p.frames + 9 * (size_t)m + t);
            double eta[3], lam[3], world[3];
            frame_apply(R, vstar, eta);
            const double g = use_alpha ? dadd(alpha, p.omega) : __ldg(p.gamma + m);
            trial_impulse(eta, __ldg(p.phi + m), g, lam);
            project(OP, lam, __ldg(p.mu + m), __ldg(p.mu2 + m));
#pragma unroll
            for (int t = 0; t < 3; ++t) lam_out[3 * (size_t)m + t] = lam[t];
            frame_apply_t(R, lam, world);
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              const double oi = dadd(0.0, world[t]);
              jt_s[slot + t] = oi;
              finish_row(3 * node + t, dadd(vstar[t], dmul(wrq[t], oi)), vc[t]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) vs_s[slot + q] = vstar[q];
          }
        }
      }
    }

    // ---- (2)(3)(2') two-node contacts: gather, one-shot projection, scatter
    if (HASC && L.has_d && !check_only) {
      if constexpr (GRID) cg::this_grid().sync();
      else if constexpr (CLUSTER) cg::this_cluster().sync();
      else __syncthreads();
      const int kstep = GRID ? (int)(gridDim.x * blockDim.x) : csize * (int)blockDim.x;
      const int kfirst = GRID ? (int)(b * blockDim.x) : crank * (int)blockDim.x;
      for (int k = c0 + kfirst + threadIdx.x; k < c1; k += kstep) {
        const int m = GRID ? k : __ldg(p.cont_list + k);
        const int loc = (SHARED_C ? k - c0 : k) * kSlotsPerContact;
        const int ci = __ldg(p.col_i + m), cj = __ldg(p.col_j + m);
        if (cj < 0) continue;  // S-contacts were solved in the sweep
        NB_CHECK(ci >= 0 && ci + 2 < p.n && m >= 0 && m < p.n_c, "contact m=%d ci=%d k=%d", m, ci, k);
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

    // ---- (4) residual reduction + decision -------------------------------
    cta_sum3(th, fr, nf, sm_warp, sm_tot);
    if constexpr (GRID) {
      if (threadIdx.x == 0) {
        part[(size_t)b * kPartialStride + 0] = sm_tot[0];
        part[(size_t)b * kPartialStride + 1] = sm_tot[1];
        part[(size_t)b * kPartialStride + 2] = sm_tot[2];
      }
      cg::this_grid().sync();
      nb_grid_totals(part, p.G, sm_tot);
    } else if constexpr (CLUSTER) {
      // cluster-wide totals: every CTA sums the cluster's partials in rank order
      if (threadIdx.x == 0)
        for (int t = 0; t < 3; ++t) sm_cpart[l & 1][t] = sm_tot[t];
      cg::this_cluster().sync();
      if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0, z = 0.0;
        for (int r = 0; r < csize; ++r) {
          const double* q = cg::this_cluster().map_shared_rank(&sm_cpart[l & 1][0], r);
          x = dadd(x, q[0]);
          y = dadd(y, q[1]);
          z = dadd(z, q[2]);
        }
        sm_tot[0] = x;
        sm_tot[1] = y;
        sm_tot[2] = z;
      }
      __syncthreads();
    }
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
    if (writer && threadIdx.x == 0) trace[l - 1] = theta;
    if (nonfinite) {
      iters = l; div = 1;
      final_buf = l % 3; final_lam = l & 1;
      break;
    }
    pending = theta < p.tol;
    if (CHEB) rho = (theta_prev <= 0.0) ? rho : py_min(ddiv(theta, theta_prev), 1.0);
    theta_prev = theta;
  }

  for (unsigned n = ring.consumed; n < ring.issued; ++n) {  // drain the chunks in flight
    const unsigned bar = ring.bar0 + 8u * (n % kNbStages);
    while (!nb_try_wait(bar, (n / kNbStages) & 1u)) {
    }
  }
  const double* vfin = ring3(p.vbuf0, p.vbuf1, p.vbuf2, final_buf);
  for (int pos = np0 + threadIdx.x; pos < np1; pos += blockDim.x) {
    const int node = __ldg(L.node_list + pos);
#pragma unroll
    for (int q = 0; q < 3; ++q) p.out_v[3 * node + q] = vfin[3 * node + q];
  }
  const double* lfin = ring2(p.lam0, p.lam1, final_lam);
  const int kstep = GRID ? (int)(gridDim.x * blockDim.x) : csize * (int)blockDim.x;
  const int kfirst = GRID ? (int)(b * blockDim.x) : crank * (int)blockDim.x;
  for (int k = c0 + kfirst + threadIdx.x; k < c1; k += kstep) {
    const int m = GRID ? k : __ldg(p.cont_list + k);
#pragma unroll
    for (int t = 0; t < 3; ++t) p.out_lam[3 * (size_t)m + t] = lfin[3 * (size_t)m + t];
  }
  if constexpr (CLUSTER) cg::this_cluster().sync();  // no CTA leaves while a peer may read its partials
  if (writer && threadIdx.x == 0) {
    status->iterations = iters;
    status->converged = conv;
    status->diverged = div;
    status->final_vbuf = final_buf;
    status->consistency = consistency;
  }
}

// ---- layout construction ---------------------------------------------------
__global__ void k_nb_iota(int n, int* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}


// per (scene, node position): gather the node's 3 rows (CSC columns of the
// symmetric A) into its template block slots: values + 9-bit masks
template <class PT>
__global__ void k_nb_fill(int S, int nn, int nsl, const int* __restrict__ t_order,
                          const int64_t* __restrict__ t_off, const int* __restrict__ t_bcol,
                          const PT* __restrict__ a_ptr, const int* __restrict__ a_idx, const double* __restrict__ a_val,
                          int64_t k_scene, unsigned* __restrict__ desc, double* __restrict__ val,
                          int* __restrict__ flags) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)S * nn) return;
  const int s = (int)(gid / nn), pos = (int)(gid % nn);
  const int sl = pos >> 5, lane = pos & 31;
  const int64_t toff = t_off[sl];
  const int W = (int)(t_off[sl + 1] - toff);
  const int64_t goff = (int64_t)s * k_scene + toff;  // global k-step offset of the slice
  const int lnode = t_order[pos];
  const int node = s * nn + lnode;
  unsigned mask[32];  // W <= 32 blocks per node (checked on the host)
  for (int k = 0; k < W; ++k) mask[k] = 0u;
  for (int p = 0; p < 3; ++p) {
    const int r = 3 * node + p;
    int k = 0;
    for (PT e = a_ptr[r]; e < a_ptr[r + 1]; ++e) {
      const int j = a_idx[e];
      const int lb = j / 3 - s * nn;
      while (k < W && t_bcol[toff * 32 + 32 * k + lane] != lb) ++k;
      if (k >= W) {  // an entry outside the template (A not on the K pattern)
        atomicOr(flags, 1);
        return;
      }
      const int t = 3 * p + (j % 3);
      val[(goff * 9 + 9 * k + t) * 32 + lane] = a_val[e];
      mask[k] |= 1u << t;
    }
  }
  for (int k = 0; k < W; ++k) {
    const int lb = t_bcol[toff * 32 + 32 * k + lane];
    desc[(goff + k) * 32 + lane] = (lb >= 0 && mask[k]) ? ((mask[k] << kMaskShift) | (unsigned)(s * nn + lb)) : 0u;
  }
}

__global__ void k_nb_slice_off(int S, int nsl, const int64_t* __restrict__ t_off, int64_t k_scene, int nn,
                               int64_t* __restrict__ off, int* __restrict__ node_list, const int* __restrict__ t_order,
                               int* __restrict__ blk_slice, int* __restrict__ blk_pos) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid < (int64_t)S * nsl) {
    const int s = (int)(gid / nsl), t = (int)(gid % nsl);
    off[gid] = (int64_t)s * k_scene + t_off[t];
  }
  if (gid == 0) off[(int64_t)S * nsl] = (int64_t)S * k_scene;
  if (gid < (int64_t)S * nn) node_list[gid] = (int)(gid / nn) * nn + t_order[gid % nn];
  if (gid <= S) {
    blk_slice[gid] = (int)gid * nsl;
    blk_pos[gid] = (int)gid * nn;
  }
}

// ---- single-system (grid) layout, built per solve from the row-sorted entries --
// (setup_pack: perm[row_ptr[r] + k] = CSC index of the k-th numeric entry of
// row r in increasing column order, colof = its column)

__device__ __forceinline__ int ng_owner(const int* __restrict__ blk_pos, int G, int pos) {
  int lo = 0, hi = G;  // blk_pos[lo] <= pos < blk_pos[lo + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (blk_pos[mid] <= pos) lo = mid;
    else hi = mid;
  }
  return lo;
}

// distinct block columns of a node's three rows (3-way merge); key sorts the
// CTA's nodes by decreasing count
// nodes carrying a single-node (S) contact: their lane also runs the contact's
// one-shot projection inline in the sweep
__global__ void k_ng_smark(int n_c, const int* __restrict__ ci, const int* __restrict__ cj, int* __restrict__ mark) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_c && cj[k] < 0) mark[ci[k] / 3] = 1;
}

// CTA split points of the weighted node sequence: CTA g owns the nodes whose
// exclusive weight prefix lies in [W g / G, W (g+1) / G)
__global__ void k_ng_split(int G, int nn, const int64_t* __restrict__ excl, int* __restrict__ bpos) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G) return;
  if (g == 0) { bpos[0] = 0; return; }
  if (g == G) { bpos[G] = nn; return; }
  const int64_t W = excl[nn];
  int lo = 0, hi = nn;  // first i with excl[i] * G >= W * g
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (excl[mid] * (int64_t)G < W * (int64_t)g) lo = mid + 1;
    else hi = mid;
  }
  bpos[g] = lo;
}

// sort key of a node: (owner CTA, decreasing block count, hash of its block
// mask sequence) -- nodes with the same masks share slices, so the packed
// k-steps' slot counts (max over the slice's lanes) waste little
__global__ void k_ng_key(int nn, int G, const int* __restrict__ blk_pos, const int* __restrict__ cnt,
                         const unsigned* __restrict__ hsh, unsigned* __restrict__ key, int* __restrict__ val) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const int g = ng_owner(blk_pos, G, i);
  key[i] = ((unsigned)g << 18) | ((unsigned)(127 - min(cnt[i], 127)) << 11) | (hsh ? (hsh[i] & 0x7ffu) : 0u);
  val[i] = i;
}

// block count of every node (its 3 rows' distinct block columns) and its
// partition weight: blocks + (single-node contact ? contact cost : 0)
__global__ void k_ng_count(int nn, const int64_t* __restrict__ row_ptr, const int* __restrict__ rowcnt,
                           const int* __restrict__ perm, const int* __restrict__ colof, const int* __restrict__ smark,
                           int contact_cost, int* __restrict__ cnt, int64_t* __restrict__ wt,
                           unsigned* __restrict__ hsh, int64_t* __restrict__ tot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  int64_t e[3], end[3];
  for (int q = 0; q < 3; ++q) {
    e[q] = row_ptr[3 * i + q];
    end[q] = e[q] + rowcnt[3 * i + q];
  }
  int c = 0;
  unsigned h = 2166136261u;
  for (;;) {
    int bc = INT_MAX;
    for (int q = 0; q < 3; ++q)
      if (e[q] < end[q]) bc = min(bc, colof[perm[e[q]]] / 3);
    if (bc == INT_MAX) break;
    ++c;
    unsigned mask = 0u;
    for (int q = 0; q < 3; ++q)
      while (e[q] < end[q]) {
        const int col = colof[perm[e[q]]];
        if (col / 3 != bc) break;
        mask |= 1u << (3 * q + col % 3);
        ++e[q];
      }
    h = (h ^ mask) * 16777619u;
  }
  hsh[i] = h ^ (h >> 11) ^ (h >> 22);
  // totals of blocks and stored entries (the packing decision)
  int ent = 0;
  for (int q = 0; q < 3; ++q) ent += rowcnt[3 * i + q];
  atomicAdd(reinterpret_cast<unsigned long long*>(tot), (unsigned long long)c);
  atomicAdd(reinterpret_cast<unsigned long long*>(tot) + 1, (unsigned long long)ent);
  cnt[i] = c;
  wt[i] = c + (smark[i] ? contact_cost : 0);
}

__global__ void k_ng_widths(int nsl, int G, const int* __restrict__ blk_slice, const int* __restrict__ blk_pos,
                            const int* __restrict__ node_list, const int* __restrict__ cnt, int64_t* __restrict__ w) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nsl) return;
  if (s == nsl) { w[s] = 0; return; }
  int lo = 0, hi = G;  // owner CTA of slice s
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (blk_slice[mid] <= s) lo = mid;
    else hi = mid;
  }
  const int pos = blk_pos[lo] + 32 * (s - blk_slice[lo]);  // its first (busiest) node
  w[s] = pos < blk_pos[lo + 1] ? cnt[node_list[pos]] : 0;
}

// packed values: VALS = false writes the descriptors (block column | mask);
// VALS = true writes each block's present entries, in entry order, to the
// value slots voff[k] + rank * 32 + lane of its k-step (slots past a lane's
// own count stay unwritten: no lane reads them)
template <bool VALS>
__global__ void k_ng_fill(int nn, int G, const int* __restrict__ blk_slice, const int* __restrict__ blk_pos,
                          const int* __restrict__ node_list, const int64_t* __restrict__ slice_off,
                          const int64_t* __restrict__ row_ptr, const int* __restrict__ rowcnt,
                          const int* __restrict__ perm, const int* __restrict__ colof, const double* __restrict__ data,
                          const int64_t* __restrict__ voff, unsigned* __restrict__ desc, double* __restrict__ val) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nn) return;
  const int g = ng_owner(blk_pos, G, pos);
  const int loc = pos - blk_pos[g];
  const int s = blk_slice[g] + (loc >> 5), lane = loc & 31;
  const int64_t off = slice_off[s];
  const int W = (int)(slice_off[s + 1] - off);
  const int i = node_list[pos];
  int64_t e[3], end[3];
  for (int q = 0; q < 3; ++q) {
    e[q] = row_ptr[3 * i + q];
    end[q] = e[q] + rowcnt[3 * i + q];
  }
  int k = 0;
  for (;;) {
    int bc = INT_MAX;
    for (int q = 0; q < 3; ++q)
      if (e[q] < end[q]) bc = min(bc, colof[perm[e[q]]] / 3);
    if (bc == INT_MAX || k >= W) break;
    unsigned mask = 0u;
    int64_t b0[3];
    for (int q = 0; q < 3; ++q) {
      b0[q] = e[q];
      while (e[q] < end[q]) {
        const int col = colof[perm[e[q]]];
        if (col / 3 != bc) break;
        mask |= 1u << (3 * q + col % 3);
        ++e[q];
      }
    }
    if constexpr (VALS) {
      // packed: rank of entry t among the block's present entries = its slot;
      // unpacked (voff == nullptr): slot t of the block's 9
      const int64_t v0 = voff ? voff[off + k] : (off + k) * (9 * 32);
      for (int q = 0; q < 3; ++q)
        for (int64_t f = b0[q]; f < e[q]; ++f) {
          const int ent = perm[f];
          const int t = 3 * q + colof[ent] % 3;
          val[v0 + 32 * (voff ? __popc(mask & ((1u << t) - 1u)) : t) + lane] = data[ent];
        }
    } else {
      desc[(off + k) * 32 + lane] = (mask << kMaskShift) | (unsigned)bc;
    }
    ++k;
  }
  if constexpr (!VALS)
    for (; k < W; ++k) desc[(off + k) * 32 + lane] = 0u;
}

// value slots of every k-step: 32 x (max stored entries of the 32 lanes' blocks)
__global__ void k_ng_ek(int64_t K, const unsigned* __restrict__ desc, int64_t* __restrict__ ek) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k > K) return;
  int e = k < K ? __popc(desc[k * 32 + lane] >> kMaskShift) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
  if (lane == 0) ek[k] = 32 * (int64_t)e;
}

__global__ void k_ng_contact_check(int n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                                   int* __restrict__ bad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_c && (ci[k] % 3 != 0 || (cj[k] >= 0 && cj[k] % 3 != 0))) atomicOr(bad, 1);
  if (k < n_c && cj[k] >= 0) atomicOr(bad + 1, 1);  // a two-node contact: the contact phase runs
}

__global__ void k_ng_node_slots(int n_c, const int* __restrict__ ci, const int* __restrict__ cj,
                                int* __restrict__ node_slot, const int* __restrict__ d_nc = nullptr,
                                double* __restrict__ jt = nullptr) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_c || (d_nc && k >= *d_nc)) return;
  node_slot[ci[k] / 3] = kSlotsPerContact * k;
  if (cj[k] >= 0) node_slot[cj[k] / 3] = kSlotsPerContact * k + 3;
  if (jt)  // J_c^T lam of the contact's slots starts at 0 (only live contacts' slots are read)
    for (int t = 0; t < kSlotsPerContact; ++t) jt[kSlotsPerContact * (size_t)k + t] = 0.0;
}

using NbFn = void (*)(IterParams, NodeLayoutDev);

template <int OP, int MODE>
NbFn nb_pick2(bool cheb, bool hasc) {
  if (cheb) return hasc ? k_iterate_nodes<OP, true, true, MODE> : k_iterate_nodes<OP, true, false, MODE>;
  return hasc ? k_iterate_nodes<OP, false, true, MODE> : k_iterate_nodes<OP, false, false, MODE>;
}

template <int MODE>
NbFn nb_pick_mode(int op, bool cheb, bool hasc) {
  if (op == OP_PROXIMAL) return nb_pick2<OP_PROXIMAL, MODE>(cheb, hasc);
  if (op == OP_ANISO) return nb_pick2<OP_ANISO, MODE>(cheb, hasc);
  return nb_pick2<OP_STRICT, MODE>(cheb, hasc);
}

NbFn nb_pick(int op, bool cheb, bool hasc, int mode) {
  if (mode == kGrid) return nb_pick_mode<kGrid>(op, cheb, hasc);
  if (mode == kCluster) return nb_pick_mode<kCluster>(op, cheb, hasc);
  return nb_pick_mode<kScene>(op, cheb, hasc);
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

int node_layout_build(NodeLayoutHost& h, int S, const int* d_a_ptr, const int* d_a_idx, const double* d_a_val,
                      NodeLayoutDev& out, int* d_flags, cudaStream_t st, int cluster,
                      const std::vector<int64_t>& t_off_host) {
  const int nn = h.nn, nsl = h.nsl;
  const int64_t ks = h.k_scene;
  const int CL = std::max(1, cluster);
  const size_t G = (size_t)S * CL;
  if (ensure(h.desc, 4 * 32 * (size_t)std::max<int64_t>(S * ks, 1)) ||
      ensure(h.val, 8 * 9 * 32 * (size_t)std::max<int64_t>(S * ks, 1)) ||
      ensure(h.slice_off, 8 * ((size_t)S * nsl + 1)) || ensure(h.node_list, 4 * (size_t)S * nn) ||
      ensure(h.node_slot, 4 * (size_t)S * nn) || ensure(h.blk_slice, 4 * (G + 1)) || ensure(h.blk_pos, 4 * (G + 1)))
    return 1;
  if (ensure(h.vs, 8 * kSlotsPerContact * (size_t)S * nn) || ensure(h.jt, 8 * kSlotsPerContact * (size_t)S * nn) ||
      ensure(h.perm, 4 * (size_t)std::max(S, 1)))
    return 1;
  // padding lanes (positions past the scene's last node) are never filled:
  // their descriptors must read as empty
  if (cudaMemsetAsync(h.val.p, 0, 8 * 9 * 32 * (size_t)S * ks, st) ||
      cudaMemsetAsync(h.desc.p, 0, 4 * 32 * (size_t)S * ks, st))
    return 1;
  const int64_t nt = std::max<int64_t>((int64_t)S * nsl, (int64_t)S * nn) + 1;
  k_nb_slice_off<<<nblk(nt), 256, 0, st>>>(S, nsl, (const int64_t*)h.t_off.p, ks, nn, (int64_t*)h.slice_off.p,
                                           (int*)h.node_list.p, (const int*)h.t_order.p, (int*)h.blk_slice.p,
                                           (int*)h.blk_pos.p);
  if (CL > 1) {
    // the scene's slices split over the cluster's CTAs by equal k-step shares
    std::vector<int> split((size_t)CL + 1, nsl);
    split[0] = 0;
    for (int r = 1; r < CL; ++r) {
      const int64_t want = ks * r / CL;
      int t = split[r - 1];
      while (t < nsl && t_off_host[t] < want) ++t;
      split[r] = std::max(t, split[r - 1] + 1 <= nsl ? split[r - 1] + 1 : nsl);
    }
    std::vector<int> bs(G + 1), bp(G + 1);
    for (int sc = 0; sc < S; ++sc)
      for (int r = 0; r < CL; ++r) {
        bs[(size_t)sc * CL + r] = sc * nsl + split[r];
        bp[(size_t)sc * CL + r] = sc * nn + std::min(nn, 32 * split[r]);
      }
    bs[G] = S * nsl;
    bp[G] = S * nn;
    if (cudaMemcpyAsync(h.blk_slice.p, bs.data(), 4 * (G + 1), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(h.blk_pos.p, bp.data(), 4 * (G + 1), cudaMemcpyHostToDevice, st) ||
        cudaStreamSynchronize(st))  // the host vectors die here
      return 1;
  }
  const int64_t nf = (int64_t)S * nn;
  k_nb_fill<int><<<nblk(nf, 128), 128, 0, st>>>(S, nn, nsl, (const int*)h.t_order.p, (const int64_t*)h.t_off.p,
                                           (const int*)h.t_bcol.p, d_a_ptr, d_a_idx, d_a_val, ks, (unsigned*)h.desc.p,
                                           (double*)h.val.p, d_flags);
  if (cudaGetLastError() != cudaSuccess) return 1;
  out.nn = nn;
  out.nsl = nsl;
  out.cluster = CL;
  out.tcol = (const int*)h.t_bcol.p;
  out.k_scene = ks;
  out.has_d = 0;  // FEM batches: node-plane contacts only (col_j = -1)
  out.blk_slice = (const int*)h.blk_slice.p;
  out.blk_pos = (const int*)h.blk_pos.p;
  out.node_list = (const int*)h.node_list.p;
  out.node_slot = (int*)h.node_slot.p;
  out.slice_off = (const int64_t*)h.slice_off.p;
  out.desc = (const unsigned*)h.desc.p;
  out.val = (const double*)h.val.p;
  out.vs_g = (double*)h.vs.p;
  out.jt_g = (double*)h.jt.p;
  // scene order: identity until the first solve's counts are known
  k_nb_iota<<<nblk(S), 256, 0, st>>>(S, (int*)h.perm.p);
  out.scene_perm = S <= kMaxOrderedScenes ? (const int*)h.perm.p : nullptr;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int node_fill_matrix(const NodeLayoutHost& h, int S, const int64_t* d_ptr, const int* d_idx, const double* d_val,
                     Workspace::Buf& desc, Workspace::Buf& val, int* d_flags, cudaStream_t st) {
  const int64_t ks = h.k_scene;
  if (ensure(desc, 4 * 32 * (size_t)std::max<int64_t>(S * ks, 1)) ||
      ensure(val, 8 * 9 * 32 * (size_t)std::max<int64_t>(S * ks, 1)))
    return 1;
  if (cudaMemsetAsync(val.p, 0, 8 * 9 * 32 * (size_t)S * ks, st) || cudaMemsetAsync(desc.p, 0, 4 * 32 * (size_t)S * ks, st))
    return 1;
  const int64_t nf = (int64_t)S * h.nn;
  k_nb_fill<int64_t><<<nblk(nf, 128), 128, 0, st>>>(S, h.nn, h.nsl, (const int*)h.t_order.p, (const int64_t*)h.t_off.p,
                                                    (const int*)h.t_bcol.p, d_ptr, d_idx, d_val, ks, (unsigned*)desc.p,
                                                    (double*)val.p, d_flags);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int node_slots_refresh(const NodeLayoutDev& L, int S, int n_c, const int* ci, const int* cj, const int* d_nc,
                       cudaStream_t st) {
  // global contact slots (6 k); J_c^T lam starts at 0. n_c is the exact count,
  // or with d_nc != nullptr an upper bound and *d_nc (device) the count
  if (cudaMemsetAsync(L.node_slot, 0xff, 4 * (size_t)S * L.nn, st) != cudaSuccess) return 1;
  if (d_nc) {  // n_c is an upper bound: zero the slots of the live contacts only
    if (n_c > 0) k_ng_node_slots<<<nblk(n_c), 256, 0, st>>>(n_c, ci, cj, L.node_slot, d_nc, L.jt_g);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
  }
  if (n_c > 0) k_ng_node_slots<<<nblk(n_c), 256, 0, st>>>(n_c, ci, cj, L.node_slot, d_nc);
  if (cudaMemsetAsync(L.jt_g, 0, 8 * kSlotsPerContact * (size_t)std::max(n_c, 1), st) != cudaSuccess) return 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int node_grid_build(NodeGridWork& w, const vfpi_system& d, int G, const int64_t* row_ptr, const int* rowcnt,
                    const int* perm, const int* colof, cudaStream_t st, NodeLayoutDev& out, std::string& err,
                    int64_t& launches, int contact_cost, int pack_mode) {
  auto fail = [&](const char* what) {
    err = std::string("node-block layout: ") + what;
    return VFPI_CUDA_ERROR;
  };
  const int n = (int)d.n, n_c = (int)d.n_c;
  if (n % 3 != 0 || n <= 0) return VFPI_UNSUPPORTED;
  const int nn = n / 3;
  if (nn >= (1 << 23)) return VFPI_UNSUPPORTED;
  // CTA g owns a contiguous range of node positions of equal weight (block
  // count + contact_cost per single-node contact: those lanes also run the
  // contact's one-shot) and their ceil(count / 32) slices
  if (ensure(w.blk_pos, 4 * ((size_t)G + 1)) || ensure(w.blk_slice, 4 * ((size_t)G + 1)) ||
      ensure(w.key, 4 * (size_t)nn) || ensure(w.key2, 4 * (size_t)nn) || ensure(w.val_i, 4 * (size_t)nn) ||
      ensure(w.node_list, 4 * (size_t)nn) || ensure(w.cnt, 4 * (size_t)nn) || ensure(w.node_slot, 4 * (size_t)nn) ||
      ensure(w.wt, 8 * ((size_t)nn + 1)) || ensure(w.wpre, 8 * ((size_t)nn + 1)) || ensure(w.flags, 16) ||
      ensure(w.hsh, 4 * (size_t)nn) ||
      ensure(w.vs, 8 * kSlotsPerContact * (size_t)std::max(n_c, 1)) ||
      ensure(w.jt, 8 * kSlotsPerContact * (size_t)std::max(n_c, 1)))
    return fail("allocation");
  if (!w.h_small && cudaMallocHost(&w.h_small, 16) != cudaSuccess) return fail("pinned allocation");
  if (!w.h_bpos.empty() && (int)w.h_bpos.size() != G + 1) w.h_bpos.clear();
  w.h_bpos.resize((size_t)G + 1);
  if (cudaMemsetAsync(w.flags.p, 0, 16, st) || cudaMemsetAsync(w.node_slot.p, 0, 4 * (size_t)nn, st) ||
      cudaMemsetAsync((int64_t*)w.wt.p + nn, 0, 8, st))
    return fail("memset");
  if (n_c > 0) k_ng_smark<<<nblk(n_c), 256, 0, st>>>(n_c, d.col_i, d.col_j, (int*)w.node_slot.p);
  if (ensure(w.tot, 16) || cudaMemsetAsync(w.tot.p, 0, 16, st)) return fail("allocation");
  k_ng_count<<<nblk(nn), 256, 0, st>>>(nn, row_ptr, rowcnt, perm, colof, (const int*)w.node_slot.p, contact_cost,
                                       (int*)w.cnt.p, (int64_t*)w.wt.p, (unsigned*)w.hsh.p, (int64_t*)w.tot.p);
  {
    size_t tw = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tw, (int64_t*)w.wt.p, (int64_t*)w.wpre.p, nn + 1, st);
    if (ensure(w.tmp, tw)) return fail("allocation");
    tw = w.tmp.cap;
    if (cub::DeviceScan::ExclusiveSum(w.tmp.p, tw, (int64_t*)w.wt.p, (int64_t*)w.wpre.p, nn + 1, st))
      return fail("scan");
  }
  k_ng_split<<<nblk(G + 1), 256, 0, st>>>(G, nn, (const int64_t*)w.wpre.p, (int*)w.blk_pos.p);
  if (cudaMemcpyAsync(w.h_bpos.data(), w.blk_pos.p, 4 * ((size_t)G + 1), cudaMemcpyDeviceToHost, st) ||
      cudaMemcpyAsync(w.h_small, w.tot.p, 16, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st))
    return fail("host read");
  // packed values pay where blocks store few of their 9 entries (axis-aligned
  // meshes: exact zeros); mode 2 also groups a CTA's nodes by block-mask
  // sequence so the slices' slot counts fit tighter (at some x locality)
  const bool want_pack = pack_mode == 3 || (pack_mode > 0 && (double)w.h_small[1] <= 7.0 * (double)w.h_small[0]);
  const bool by_masks = want_pack && pack_mode >= 2;
  std::vector<int> bsl((size_t)G + 1);
  bsl[0] = 0;
  for (int g = 0; g < G; ++g) bsl[g + 1] = bsl[g] + (w.h_bpos[g + 1] - w.h_bpos[g] + 31) / 32;
  const int nsl = bsl[G];
  if (ensure(w.width, 8 * ((size_t)nsl + 1)) || ensure(w.slice_off, 8 * ((size_t)nsl + 1)))
    return fail("allocation");
  if (cudaMemcpyAsync(w.blk_slice.p, bsl.data(), 4 * ((size_t)G + 1), cudaMemcpyHostToDevice, st)) return fail("upload");
  k_ng_key<<<nblk(nn), 256, 0, st>>>(nn, G, (const int*)w.blk_pos.p, (const int*)w.cnt.p,
                                     by_masks ? (const unsigned*)w.hsh.p : nullptr, (unsigned*)w.key.p,
                                     (int*)w.val_i.p);
  launches += 5 + (n_c > 0);
  if (n_c > 0) k_ng_contact_check<<<nblk(n_c), 256, 0, st>>>(n_c, d.col_i, d.col_j, (int*)w.flags.p);
  int eb = 18;
  while ((1 << (eb - 18)) <= G) ++eb;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned*)w.key.p, (unsigned*)w.key2.p, (int*)w.val_i.p,
                                  (int*)w.node_list.p, nn, 0, eb, st);
  size_t ts = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, ts, (int64_t*)w.width.p, (int64_t*)w.slice_off.p, nsl + 1, st);
  if (ensure(w.tmp, std::max(tb, ts))) return fail("allocation");
  tb = w.tmp.cap;
  if (cub::DeviceRadixSort::SortPairs(w.tmp.p, tb, (unsigned*)w.key.p, (unsigned*)w.key2.p, (int*)w.val_i.p,
                                      (int*)w.node_list.p, nn, 0, eb, st))
    return fail("sort");
  k_ng_widths<<<nblk(nsl + 1), 256, 0, st>>>(nsl, G, (const int*)w.blk_slice.p, (const int*)w.blk_pos.p,
                                             (const int*)w.node_list.p, (const int*)w.cnt.p, (int64_t*)w.width.p);
  ts = w.tmp.cap;
  if (cub::DeviceScan::ExclusiveSum(w.tmp.p, ts, (int64_t*)w.width.p, (int64_t*)w.slice_off.p, nsl + 1, st))
    return fail("scan");
  launches += 6 + (n_c > 0);
  if (cudaMemcpyAsync(w.h_small, (int64_t*)w.slice_off.p + nsl, 8, cudaMemcpyDeviceToHost, st) ||
      cudaMemcpyAsync((int*)(w.h_small + 1), w.flags.p, 8, cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st))
    return fail("host read");
  if (((int*)(w.h_small + 1))[0]) return VFPI_UNSUPPORTED;  // a contact column is not node aligned
  const int64_t K = w.h_small[0];
  // packed values: k-step k keeps 32 x E_k slots (E_k = the most entries any of
  // its lanes' blocks stores), no zeros for absent entries
  if (ensure(w.desc, 4 * 32 * (size_t)std::max<int64_t>(K, 1)) ||
      ensure(w.val, 8 * 9 * 32 * (size_t)std::max<int64_t>(K, 1)) || ensure(w.ek, 8 * ((size_t)K + 1)) ||
      ensure(w.voff, 8 * ((size_t)K + 1)))
    return fail("allocation");
  if (cudaMemsetAsync(w.desc.p, 0, 4 * 32 * (size_t)K, st))
    return fail("memset");  // padding lanes past a CTA's last node are never filled
  k_ng_fill<false><<<nblk(nn, 128), 128, 0, st>>>(nn, G, (const int*)w.blk_slice.p, (const int*)w.blk_pos.p,
                                                  (const int*)w.node_list.p, (const int64_t*)w.slice_off.p, row_ptr,
                                                  rowcnt, perm, colof, d.data, nullptr, (unsigned*)w.desc.p, nullptr);
  k_ng_ek<<<nblk(32 * (K + 1)), 256, 0, st>>>(K, (const unsigned*)w.desc.p, (int64_t*)w.ek.p);
  {
    size_t te = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, te, (int64_t*)w.ek.p, (int64_t*)w.voff.p, K + 1, st);
    if (ensure(w.tmp, te)) return fail("allocation");
    te = w.tmp.cap;
    if (cub::DeviceScan::ExclusiveSum(w.tmp.p, te, (int64_t*)w.ek.p, (int64_t*)w.voff.p, K + 1, st))
      return fail("scan");
  }
  // packed only where it saves a fifth of the value bytes (blocks with exact
  // zeros, e.g. unrotated meshes); full blocks stream faster unpacked
  if (cudaMemcpyAsync(w.h_small, (int64_t*)w.voff.p + K, 8, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st))
    return fail("host read");
  const bool packed = want_pack && (pack_mode == 3 || (double)w.h_small[0] <= 0.8 * 288.0 * (double)K);
  k_ng_fill<true><<<nblk(nn, 128), 128, 0, st>>>(nn, G, (const int*)w.blk_slice.p, (const int*)w.blk_pos.p,
                                                 (const int*)w.node_list.p, (const int64_t*)w.slice_off.p, row_ptr,
                                                 rowcnt, perm, colof, d.data,
                                                 packed ? (const int64_t*)w.voff.p : nullptr, nullptr,
                                                 (double*)w.val.p);
  launches += 4;
  if (cudaMemsetAsync(w.node_slot.p, 0xff, 4 * (size_t)nn, st)) return fail("memset");
  if (n_c > 0) k_ng_node_slots<<<nblk(n_c), 256, 0, st>>>(n_c, d.col_i, d.col_j, (int*)w.node_slot.p);
  if (cudaMemsetAsync(w.jt.p, 0, 8 * kSlotsPerContact * (size_t)std::max(n_c, 1), st)) return fail("memset");
  launches += 1 + (n_c > 0);
  if (cudaGetLastError() != cudaSuccess) return fail("launch");
  w.k_total = K;
  out.has_d = ((int*)(w.h_small + 1))[1] ? 1 : 0;
  out.nn = nn;
  out.nsl = nsl;
  out.blk_slice = (const int*)w.blk_slice.p;
  out.blk_pos = (const int*)w.blk_pos.p;
  out.node_list = (const int*)w.node_list.p;
  out.node_slot = (int*)w.node_slot.p;
  out.slice_off = (const int64_t*)w.slice_off.p;
  out.desc = (const unsigned*)w.desc.p;
  out.val = (const double*)w.val.p;
  out.voff = packed ? (const int64_t*)w.voff.p : nullptr;
  w.packed = packed;
  out.vs_g = (double*)w.vs.p;
  out.jt_g = (double*)w.jt.p;
  return VFPI_OK;
}

int node_kernel_smem(int max_ct, int mode) {
  (void)max_ct;  // contact slots are global: the ring is the only dynamic shared memory
  if (mode == kGrid) return VFPI_NB_WARPS * kNbStages * kNbGridStageBytes + 256;
  return kNbRingBytes + 128;
}

int node_kernel_blocks_per_sm(int op, bool cheb, int max_ct, int mode) {
  NbFn f = nb_pick(op, cheb, true, mode);
  if (ensure_max_dynamic_smem((const void*)f) != cudaSuccess) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kNbThreads, node_kernel_smem(mode == kScene ? max_ct : 0, mode)) !=
      cudaSuccess)
    return 0;
  return nb;
}

int launch_iterate_nodes(const IterParams& p, const NodeLayoutDev& L, int op, bool cheb, int max_ct, cudaStream_t st,
                         std::string& err, int mode) {
  NbFn f = nb_pick(op, cheb, p.n_c > 0, mode);
  cudaError_t e = ensure_max_dynamic_smem((const void*)f);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return VFPI_CUDA_ERROR; }
  if (mode == kGrid) {
    IterParams lp = p;
    NodeLayoutDev ll = L;
    void* args[] = {&lp, &ll};
    e = cudaLaunchCooperativeKernel((const void*)f, dim3(p.G), dim3(kNbThreads), args, node_kernel_smem(0, kGrid), st);
  } else if (mode == kCluster) {
    cudaLaunchConfig_t c{};
    c.gridDim = dim3((unsigned)(p.G * L.cluster));
    c.blockDim = dim3(kNbThreads);
    c.dynamicSmemBytes = (size_t)node_kernel_smem(0);
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)L.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    c.attrs = at;
    c.numAttrs = 1;
    e = cudaLaunchKernelEx(&c, f, p, L);
  } else {
    f<<<p.G, kNbThreads, node_kernel_smem(max_ct), st>>>(p, L);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    err = std::string("node-block launch: ") + cudaGetErrorString(e);
    return VFPI_CUDA_ERROR;
  }
  return VFPI_OK;
}

// CTAs per scene: the smallest power of two that gives the batch >= 1.5 waves
// of the GPU's 2 CTAs per SM (with the longest-first scene order the block
// scheduler then balances scenes of unequal iteration counts), at most 8 and
// at most one CTA per two node slices
int node_cluster_size(int S, int nsl, int num_sms) {
  int cl = 1;
  while (cl < 8 && (int64_t)S * cl < 3LL * num_sms && cl * 2 <= nsl) cl *= 2;
  return cl;
}

}  // namespace vfpi
