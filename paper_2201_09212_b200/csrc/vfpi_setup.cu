// Per-solve setup on the device: CSC -> row-sorted numeric entries, contact-
// aware CTA partition, SELL-32 packing, Frobenius step matrix and gamma.
//
// Reference semantics:
//   SparseSymmetric.diagonal     sparse.py:67-68
//   row_norms_sq                 sparse.py:105-108 (reduceat over pruned squares)
//   step_matrix_frobenius        solver.py:216-229 (tie groups solver.py:182-213)
//   surrogate_gamma / _check_tie solver.py:244-259
//   fixed-alpha default          solver.py:367-369
#include <cub/cub.cuh>
#include <atomic>
#include <map>
#include <mutex>
#include <unordered_map>
#include <climits>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

// Partition cost model, in bytes of per-CTA state (the resident kernel's
// shared-memory footprint, which also tracks per-iteration work): 24 B per
// numeric entry (value, column, destination, product), 40 B per row, 256 B
// per contact.
// (defaults in LayoutOptions: entry 24, row 40, contact 256)

#define VFPI_CK(x)                                                     \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      err = std::string(#x) + ": " + cudaGetErrorString(e_);           \
      return VFPI_CUDA_ERROR;                                          \
    }                                                                  \
  } while (0)

inline int nblk(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// column statistics: diagonal, squared norms, numeric row counts, sort keys
// ---------------------------------------------------------------------------
struct PrunedSquares {
  const double* data;
  int e0, e1;
  mutable int cur_e;
  mutable int64_t cur_k;
  __device__ double operator()(int64_t k) const {
    if (k < cur_k) { cur_k = -1; cur_e = e0 - 1; }
    while (cur_k < k) {
      ++cur_e;
      const double d = data[cur_e];
      if (dmul(d, d) != 0.0) ++cur_k;
    }
    const double d = data[cur_e];
    return dmul(d, d);
  }
};

__global__ void k_colstats(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                           const double* __restrict__ data, double* __restrict__ diag, double* __restrict__ rns,
                           int* __restrict__ rowcnt, int* __restrict__ keys, int* __restrict__ colof,
                           int* __restrict__ rowmin) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int e0 = indptr[j], e1 = indptr[j + 1];
  double dg = 0.0;
  int64_t npr = 0;
  for (int e = e0; e < e1; ++e) {
    const int i = indices[e];
    const double d = data[e];
    if (i == j) dg = dadd(dg, d);
    if (dmul(d, d) != 0.0) ++npr;
    const bool num = (d != 0.0);
    keys[e] = num ? i : n;
    colof[e] = j;
    if (num) {
      atomicAdd(&rowcnt[i], 1);
      atomicMin(&rowmin[i], j);
    }
  }
  diag[j] = dg;
  double r = 0.0;
  if (npr > 0) {
    PrunedSquares g{data, e0, e1, e0 - 1, -1};
    const double first = g(0);
    r = (npr == 1) ? first : dadd(first, np_pairwise(g, 1, npr - 1));
  }
  rns[j] = r;
}

__global__ void k_mark(int n, int n_c, const int* __restrict__ ci, const int* __restrict__ cj, int* mark,
                       int* flags) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_c) return;
  const int i = ci[m], j = cj[m];
  if (i < 0 || i > n - 3 || j < -1 || (j >= 0 && j > n - 3)) { atomicOr(flags, 2); return; }
  for (int t = 0; t < 3; ++t)
    if (atomicCAS(&mark[i + t], -1, m) != -1) atomicOr(flags, 1);
  if (j >= 0)
    for (int t = 0; t < 3; ++t)
      if (atomicCAS(&mark[j + t], -1, m) != -1) atomicOr(flags, 1);
}

// unit = one free row, or all (3 or 6) rows of one contact, anchored at col_i.
// Units are ordered by their anchor = the smallest column any of their rows
// touches (stable in row order): a unit then sits next to the rows it couples
// to (a rigid body's virtual nodes next to the body, FEM rows stay banded), so
// a CTA range reads few remote sectors of v.
__global__ void k_unit_keys(int n, const int* __restrict__ mark, const int* __restrict__ ci,
                            const int* __restrict__ cj, const int* __restrict__ rowmin, int* __restrict__ key,
                            int* __restrict__ val, int anchor) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int m = mark[r];
  int k = INT_MAX;
  if (m < 0) {
    k = min(r, rowmin[r]);
  } else if (r == ci[m]) {
    const int i = ci[m], j = cj[m];
    k = i;
    for (int t = 0; t < 3; ++t) k = min(k, rowmin[i + t]);
    if (j >= 0) {
      k = min(k, j);
      for (int t = 0; t < 3; ++t) k = min(k, rowmin[j + t]);
    }
  }
  key[r] = (k == INT_MAX) ? n : (anchor ? k : r);  // non-start rows: n; natural order: the start row itself
  val[r] = r;
}

// per sorted unit t (anchor order): cost / rows / contact indicators
__global__ void k_units(int n, const int* __restrict__ skey, const int* __restrict__ U, const int* __restrict__ mark,
                        const int* __restrict__ ci, const int* __restrict__ cj, const int* __restrict__ rowcnt,
                        int64_t* ucost, int* urows, int* ucont, int* ucr, int* ufr, int kEntryCost, int kRowCost,
                        int kContactCost) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n) return;
  int64_t cost = 0;
  int rows = 0, ct = 0;
  if (t < n && skey[t] < n) {
    const int r = U[t];
    const int m = mark[r];
    if (m < 0) {
      cost = (int64_t)kEntryCost * rowcnt[r] + kRowCost;
      rows = 1;
    } else {
      const int i = ci[m], j = cj[m];
      ct = 1;
      rows = (j >= 0) ? 6 : 3;
      cost = kContactCost;
      for (int q = 0; q < 3; ++q) cost += (int64_t)kEntryCost * rowcnt[i + q] + kRowCost;
      if (j >= 0)
        for (int q = 0; q < 3; ++q) cost += (int64_t)kEntryCost * rowcnt[j + q] + kRowCost;
    }
  }
  if (t < n) {
    ucost[t] = cost;
    urows[t] = rows;
    ucont[t] = ct;
  }
  ucr[t] = ct ? rows : 0;                // rows of a contact unit
  ufr[t] = (rows == 1 && !ct) ? 1 : 0;   // a free row
}

// CTA b starts at the unit whose cost range contains the first cost position
// of block b (blk_of(c) = floor(c*G/total)): that unit writes the starts of
// every CTA it opens (no atomics; a unit spanning several boundaries leaves the
// earlier ones empty).
__global__ void k_blocks(int n, int G, const int64_t* __restrict__ ucost, const int64_t* __restrict__ cpos,
                         const int* __restrict__ urows, const int* __restrict__ rpos, const int* __restrict__ kpos,
                         int* blk_row, int* blk_ct, int* blk_first) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || urows[t] == 0) return;
  const int64_t total = cpos[n - 1] + ucost[n - 1];
  if (total <= 0) return;
  auto blk_of = [&](int64_t c) -> int64_t {  // block of cost position c (floor, c >= 0)
    const int64_t b = (c * (int64_t)G) / total;
    return b > G - 1 ? G - 1 : b;
  };
  // blocks whose first cost position lies inside this unit's cost range
  const int64_t hi = blk_of(cpos[t] + ucost[t] - 1);
  const int64_t lo = (cpos[t] == 0) ? -1 : blk_of(cpos[t] - 1);
  for (int64_t b = lo + 1; b <= hi; ++b) {
    blk_row[b] = rpos[t];
    blk_ct[b] = kpos[t];
    blk_first[b] = t;
  }
}

// one CTA of kFixThreads threads, G <= kFixThreads: fill empty CTA ranges with
// the next non-empty start (suffix minimum), slice prefix, contact-row counts
constexpr int kFixThreads = 1024;

__global__ void __launch_bounds__(kFixThreads) k_blocks_fix(int n, int n_c, int G, int* blk_row, int* blk_ct,
                                                             int* blk_slice, int* blk_first, int* blk_cr,
                                                             const int* __restrict__ cposc, SetupSummary* sum) {
  __shared__ int s_row[kFixThreads + 1], s_ct[kFixThreads + 1], s_first[kFixThreads + 1], s_x[kFixThreads];
  const int b = threadIdx.x;
  s_row[b] = (b < G) ? blk_row[b] : n;
  s_ct[b] = (b < G) ? blk_ct[b] : n_c;
  s_first[b] = (b < G) ? blk_first[b] : n;
  if (b == 0) { s_row[kFixThreads] = n; s_ct[kFixThreads] = n_c; s_first[kFixThreads] = n; }
  __syncthreads();
  // suffix minimum (Hillis-Steele, log2 steps); INT_MAX marks empty ranges
  for (int o = 1; o < kFixThreads; o <<= 1) {
    const int r = (b + o <= kFixThreads) ? s_row[b + o] : n;
    const int c = (b + o <= kFixThreads) ? s_ct[b + o] : n_c;
    const int f = (b + o <= kFixThreads) ? s_first[b + o] : n;
    __syncthreads();
    s_row[b] = min(s_row[b], r);
    s_ct[b] = min(s_ct[b], c);
    s_first[b] = min(s_first[b], f);
    __syncthreads();
  }
  if (b == 0) { s_row[0] = 0; s_ct[0] = 0; s_first[0] = 0; }
  __syncthreads();
  const int nsl = (b < G) ? (s_row[b + 1] - s_row[b] + 31) / 32 : 0;
  const int nct = (b < G) ? (s_ct[b + 1] - s_ct[b]) : 0;
  // inclusive prefix of slice counts
  s_x[b] = nsl;
  __syncthreads();
  for (int o = 1; o < kFixThreads; o <<= 1) {
    const int t = (b >= o) ? s_x[b - o] : 0;
    __syncthreads();
    s_x[b] += t;
    __syncthreads();
  }
  if (b < G) {
    blk_row[b] = s_row[b];
    blk_ct[b] = s_ct[b];
    blk_first[b] = s_first[b];
    blk_slice[b] = s_x[b] - nsl;
    blk_cr[b] = cposc[s_first[b + 1]] - cposc[s_first[b]];
  }
  if (b == 0) {
    blk_row[G] = n;
    blk_ct[G] = n_c;
    blk_first[G] = n;
    blk_slice[G] = s_x[kFixThreads - 1];
    blk_cr[G] = 0;
    sum->n_slices = s_x[kFixThreads - 1];
  }
  // max contacts per CTA
  __syncthreads();
  s_x[b] = nct;
  __syncthreads();
  for (int o = kFixThreads / 2; o > 0; o >>= 1) {
    if (b < o) s_x[b] = max(s_x[b], s_x[b + o]);
    __syncthreads();
  }
  if (b == 0) sum->max_ct_per_blk = s_x[0];
}

__device__ __forceinline__ int owner(const int* __restrict__ starts, int G, int p) {
  // largest b with starts[b] <= p (starts has G+1 monotone entries)
  int lo = 0, hi = G;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (starts[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// Row list: within every CTA range, the rows of its contact units come first,
// then its free rows (unit order). cont_q = rank of a two-sided contact among
// the CTA's two-sided contacts. t = sorted unit index, U[t] = its start row.
__global__ void k_fill(int n, int G, const int* __restrict__ U, const int* __restrict__ mark,
                       const int* __restrict__ ci, const int* __restrict__ cj, const int* __restrict__ urows,
                       const int* __restrict__ rpos, const int* __restrict__ kpos, const int* __restrict__ cposc,
                       const int* __restrict__ cposf, const int* __restrict__ blk_row, const int* __restrict__ blk_ct,
                       const int* __restrict__ blk_first, const int* __restrict__ blk_cr, int* row_list, int* row_slot,
                       int* cont_list, int* cont_q) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || urows[t] == 0) return;
  const int r = U[t];
  const int b = owner(blk_row, G, rpos[t]);
  const int f = blk_first[b];
  const int m = mark[r];
  if (m < 0) {
    const int p = blk_row[b] + blk_cr[b] + (cposf[t] - cposf[f]);
    row_list[p] = r;
    row_slot[p] = -1;
    return;
  }
  // contact rows are component-major: row a of side i of local contact kl at
  // a*C + kl, row a of side j at 3C + a*CD + kd (kd = rank among the CTA's
  // two-sided contacts), so lane kl of the resident kernel reads its rows
  // from consecutive SELL lanes
  const int k = kpos[t];
  const int kl = k - blk_ct[b];
  const int Cb = blk_ct[b + 1] - blk_ct[b];
  const int CDb = blk_cr[b] / 3 - Cb;
  const int kd = (cposc[t] - cposc[f]) / 3 - kl;
  const int loc = kl * kSlotsPerContact;
  cont_list[k] = m;
  cont_q[k] = kd;
  const int i = ci[m], j = cj[m];
  for (int q = 0; q < 3; ++q) {
    const int p = blk_row[b] + q * Cb + kl;
    row_list[p] = i + q;
    row_slot[p] = loc + q;
  }
  if (j >= 0)
    for (int q = 0; q < 3; ++q) {
      const int p = blk_row[b] + 3 * Cb + q * CDb + kd;
      row_list[p] = j + q;
      row_slot[p] = loc + 3 + q;
    }
}

// Within every CTA, free rows are re-ordered by decreasing length (contact
// rows stay first and in place): SELL-32 slices then group rows of equal
// length, so padding and warp divergence of the row sums stay small.
__global__ void k_row_keys(int n, int G, const int* __restrict__ row_list, const int* __restrict__ row_slot,
                           const int* __restrict__ rowcnt, const int* __restrict__ blk_row, int* __restrict__ key,
                           int* __restrict__ val) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int b = owner(blk_row, G, p);
  const int len = min(rowcnt[row_list[p]], 255);
  key[p] = (b << 9) | (row_slot[p] < 0 ? (256 | (255 - len)) : 0);
  val[p] = p;
}

__global__ void k_row_permute(int n, const int* __restrict__ perm, const int* __restrict__ row_list,
                              const int* __restrict__ row_slot, int* __restrict__ row_list2,
                              int* __restrict__ row_slot2) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  row_list2[p] = row_list[perm[p]];
  row_slot2[p] = row_slot[perm[p]];
}

// warp per slice: width = longest row of its (up to) 32 rows
__global__ void k_slice_width(int S_max, int G, const SetupSummary* __restrict__ sum,
                              const int* __restrict__ blk_slice, const int* __restrict__ blk_row,
                              const int* __restrict__ row_list, const int* __restrict__ rowcnt, int64_t* width) {
  const int s = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (s > S_max) return;
  const int S = sum->n_slices;
  if (s >= S) {
    if (lane == 0) width[s] = 0;
    return;
  }
  const int b = owner(blk_slice, G, s);
  const int p = blk_row[b] + (s - blk_slice[b]) * 32 + lane;
  int W = p < blk_row[b + 1] ? rowcnt[row_list[p]] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) W = max(W, __shfl_xor_sync(0xffffffffu, W, o));
  if (lane == 0) width[s] = 32 * (int64_t)W;
}

__global__ void k_poslen(int n, const int* __restrict__ row_list, const int* __restrict__ rowcnt, int64_t* len) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  len[p] = (p < n) ? rowcnt[row_list[p]] : 0;
}

__global__ void __launch_bounds__(kFixThreads) k_summary(int n, int G, const int64_t* row_ptr,
                                                          const int64_t* slice_off, const int64_t* pos_ptr,
                                                          const int* blk_row, const int* blk_ct, const int* blk_cr,
                                                          const int* blk_slice, const int* sec_ptr, const int* flags,
                                                          SetupSummary* sum) {
  __shared__ long long s_e[kFixThreads], s_b[kFixThreads];
  __shared__ int s_r[kFixThreads];
  const int b = threadIdx.x;
  long long e = 0, by = 0;
  int r = 0;
  if (b < G) {
    e = pos_ptr[blk_row[b + 1]] - pos_ptr[blk_row[b]];
    r = blk_row[b + 1] - blk_row[b];
    const int64_t ep = slice_off[blk_slice[b + 1]] - slice_off[blk_slice[b]];
    by = (long long)ResLayout(ep, r, blk_ct[b + 1] - blk_ct[b], blk_cr[b], sec_ptr[b + 1] - sec_ptr[b]).total;
  }
  s_e[b] = e;
  s_b[b] = by;
  s_r[b] = r;
  __syncthreads();
  for (int o = kFixThreads / 2; o > 0; o >>= 1) {
    if (b < o) {
      s_e[b] = max(s_e[b], s_e[b + o]);
      s_b[b] = max(s_b[b], s_b[b + o]);
      s_r[b] = max(s_r[b], s_r[b + o]);
    }
    __syncthreads();
  }
  if (b == 0) {
    sum->nnz_num = row_ptr[n];
    sum->sell_elems = slice_off[sum->n_slices];
    sum->flags = *flags;
    sum->max_ent_per_blk = s_e[0];
    sum->max_rows_per_blk = s_r[0];
    sum->max_res_bytes = s_b[0];
  }
}

// ---- gather plan of the resident kernel -------------------------------------
// Every CTA stages, once per iteration, the 32-byte sectors of v its entries
// read from other CTAs' rows; columns that are its own rows read the on-chip
// copy. Built in phase 1 from the CSC entries (so the shared-memory size is
// known at the single host read): key = (cta << SB) | sector, radix sorted,
// first-of-run flags -> block-major unique sector list secs + per-CTA ranges.
// sell_map[i] (phase 2) is the index of SELL element i's x in the CTA's x
// array: 4*slot + (col & 3) for a staged sector, 4*NS + q for own row q.
constexpr unsigned kNoSector = 0xFFFFFFFFu;

__global__ void k_rowpos(int n, int G, const int* __restrict__ row_list, const int* __restrict__ blk_row,
                         int* __restrict__ rowpos, int* __restrict__ rowblk) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int r = row_list[q];
  rowpos[r] = q;
  rowblk[r] = owner(blk_row, G, q);
}

// per CSC entry (thread per column): sector key of a numeric entry whose row's
// CTA does not own its column
__global__ void k_sec_keys(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                           const double* __restrict__ data, const int* __restrict__ rowblk,
                           unsigned* __restrict__ key, int SB) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int bj = rowblk[j];
  for (int e = indptr[j]; e < indptr[j + 1]; ++e) {
    unsigned k = kNoSector;
    if (data[e] != 0.0) {
      const int b = rowblk[indices[e]];
      if (b != bj) k = ((unsigned)b << SB) | ((unsigned)j >> 2);
    }
    key[e] = k;
  }
}

__global__ void k_sec_flags(int64_t N, const unsigned* __restrict__ skey, int* __restrict__ flag) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  const unsigned k = skey[j];
  flag[j] = (k != kNoSector && (j == 0 || skey[j - 1] != k)) ? 1 : 0;
}

// unique sector list (sector ids) and the first unique index of every CTA
__global__ void k_sec_emit(int64_t N, const unsigned* __restrict__ skey, const int* __restrict__ flag,
                           const int* __restrict__ upos, unsigned* __restrict__ secs, int* __restrict__ sec_ptr, int SB) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N || !flag[j]) return;
  const unsigned k = skey[j];
  secs[upos[j]] = k & ((1u << SB) - 1u);
  const int b = (int)(k >> SB);
  if (j == 0 || (skey[j - 1] >> SB) != (unsigned)b || skey[j - 1] == kNoSector) sec_ptr[b] = upos[j];
}

// CTAs without remote sectors inherit the next start; sec_ptr[G] = total
// (one CTA, G < blockDim.x: suffix minimum)
__global__ void __launch_bounds__(1024) k_sec_ptr_fix(int G, int64_t N, const int* __restrict__ flag,
                                                      const int* __restrict__ upos, int* __restrict__ sec_ptr) {
  __shared__ int sp[1025];
  const int b = threadIdx.x;
  const int total = N > 0 ? upos[N - 1] + flag[N - 1] : 0;
  if (b <= G) {
    const int v = (b == G) ? total : sec_ptr[b];
    sp[b] = v < 0 ? INT_MAX : v;
  }
  __syncthreads();
  for (int o = 1; o <= G; o <<= 1) {
    const int v = (b <= G) ? ((b + o <= G) ? min(sp[b], sp[b + o]) : sp[b]) : 0;
    __syncthreads();
    if (b <= G) sp[b] = v;
    __syncthreads();
  }
  if (b <= G) sec_ptr[b] = sp[b];
}

// one CTA per partition: its sector list in shared memory, gather map of every
// SELL element of the partition (binary search on chip)
constexpr int kMapSmemSectors = 8192;

__global__ void __launch_bounds__(1024) k_sell_map(int G, const int* __restrict__ blk_slice,
                                                  const int* __restrict__ blk_row, const int64_t* __restrict__ slice_off,
                                                  const int* __restrict__ sell_col, const int* __restrict__ rowpos,
                                                  const unsigned* secs, const int* __restrict__ sec_ptr,
                                                  unsigned* __restrict__ map) {
  unsigned* secs_w = const_cast<unsigned*>(secs);
  __shared__ unsigned ssec[kMapSmemSectors];
  const int b = blockIdx.x;
  const int p0 = blk_row[b], p1 = blk_row[b + 1];
  const int u0 = sec_ptr[b], u1 = sec_ptr[b + 1];
  const int ns = u1 - u0;
  const bool on_chip = ns <= kMapSmemSectors;
  if (on_chip)
    for (int j = threadIdx.x; j < ns; j += blockDim.x) ssec[j] = secs[u0 + j];
  __syncthreads();
  const unsigned* sl = on_chip ? ssec : secs + u0;
  const int64_t e0 = slice_off[blk_slice[b]], e1 = slice_off[blk_slice[b + 1]];
  for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
    const int c = sell_col[i];
    unsigned m = 0u;
    if (c >= 0) {
      const int pc = rowpos[c];
      if (pc >= p0 && pc < p1) {
        m = 4u * (unsigned)ns + (unsigned)(pc - p0);  // own rows follow the staged sectors
      } else {
        const unsigned sec = (unsigned)c >> 2;
        int lo = 0, hi = ns;  // first sector >= sec (bits 30/31 are the half marks set below)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((sl[mid] & kSecIdMask) < sec) lo = mid + 1; else hi = mid;
        }
        m = 4u * (unsigned)lo + ((unsigned)c & 3u);
        // the kernel stages only the 16-byte halves of a sector its entries read
        atomicOr(secs_w + u0 + lo, 1u << (30 + (((unsigned)c & 3u) >> 1)));
      }
    }
    map[i] = m;
  }
}

__global__ void k_iota(int64_t n, int* v) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) v[e] = (int)e;
}

// one warp per slice: lane k-th entry of its row at off + k*32 + lane
__global__ void k_pack(int S, int G, const int* __restrict__ blk_slice, const int* __restrict__ blk_row,
                       const int* __restrict__ row_list, const int* __restrict__ rowcnt,
                       const int64_t* __restrict__ row_ptr, const int* __restrict__ perm,
                       const int* __restrict__ colof, const double* __restrict__ data,
                       const int64_t* __restrict__ slice_off, double* __restrict__ sv, int* __restrict__ sc) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  const int b = owner(blk_slice, G, s);
  const int p = blk_row[b] + (s - blk_slice[b]) * 32 + lane;
  const bool valid = p < blk_row[b + 1];
  const int row = valid ? row_list[p] : 0;
  const int len = valid ? rowcnt[row] : 0;
  const int64_t base = valid ? row_ptr[row] : 0;
  const int64_t off = slice_off[s];
  const int W = (int)((slice_off[s + 1] - off) >> 5);
  for (int k = 0; k < W; ++k) {
    const int64_t dst = off + (int64_t)k * 32 + lane;
    if (k < len) {
      const int e = perm[base + k];
      sv[dst] = data[e];
      sc[dst] = colof[e];
    } else {
      sv[dst] = 0.0;
      sc[dst] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// step matrix W and surrogate Delassus gamma
// ---------------------------------------------------------------------------
__global__ void k_w_frob(int n, const double* __restrict__ diag, const double* __restrict__ rns, double* w,
                         int* flags) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (rns[r] <= 0.0) atomicOr(flags, 4);
  w[r] = ddiv(diag[r], rns[r]);
}

// tie groups: strict ties each contacted node's triple; proximal also merges
// the two nodes of a D contact (solver.py:182-213, 366). Groups are disjoint
// because contact columns do not overlap (checked in k_mark).
__global__ void k_tie(int n_c, int pair_tie, const int* __restrict__ ci, const int* __restrict__ cj,
                      const double* __restrict__ diag, const double* __restrict__ rns, double* w,
                      const int* __restrict__ d_nc) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_c || (d_nc && m >= *d_nc)) return;
  const int i = ci[m], j = cj[m];
  if (pair_tie && j >= 0) {
    double sd = 0.0, sr = 0.0;
    for (int t = 0; t < 3; ++t) { sd = dadd(sd, diag[i + t]); sr = dadd(sr, rns[i + t]); }
    for (int t = 0; t < 3; ++t) { sd = dadd(sd, diag[j + t]); sr = dadd(sr, rns[j + t]); }
    const double v = ddiv(sd, sr);
    for (int t = 0; t < 3; ++t) { w[i + t] = v; w[j + t] = v; }
    return;
  }
  {
    double sd = 0.0, sr = 0.0;
    for (int t = 0; t < 3; ++t) { sd = dadd(sd, diag[i + t]); sr = dadd(sr, rns[i + t]); }
    const double v = ddiv(sd, sr);
    for (int t = 0; t < 3; ++t) w[i + t] = v;
  }
  if (j >= 0) {
    double sd = 0.0, sr = 0.0;
    for (int t = 0; t < 3; ++t) { sd = dadd(sd, diag[j + t]); sr = dadd(sr, rns[j + t]); }
    const double v = ddiv(sd, sr);
    for (int t = 0; t < 3; ++t) w[j + t] = v;
  }
}

__global__ void k_gamma(int n_c, const int* __restrict__ ci, const int* __restrict__ cj, const double* __restrict__ w,
                        double omega, double* gamma, int* flags, const int* __restrict__ d_nc) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_c || (d_nc && m >= *d_nc)) return;
  const int i = ci[m], j = cj[m];
  double g = w[i];
  if (!(w[i] == w[i + 1] && w[i] == w[i + 2])) atomicOr(flags, 8);
  if (j >= 0) {
    if (!(w[j] == w[j + 1] && w[j] == w[j + 2])) atomicOr(flags, 8);
    g = dadd(g, w[j]);
  }
  gamma[m] = dadd(g, omega);
}

// single-CTA deterministic reductions: max|diag| (NaN-propagating) and mean(w)
__global__ void k_absmax_alpha(int n, const double* __restrict__ diag, double* w_alpha_out) {
  __shared__ double sm[256];
  double mx = -INFINITY;
  bool nan = false;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const double a = fabs(diag[r]);
    if (isnan(a)) nan = true;
    mx = a > mx ? a : mx;
  }
  sm[threadIdx.x] = nan ? NAN : mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = -INFINITY;
    for (int t = 0; t < blockDim.x; ++t) m = np_max(sm[t], m);
    *w_alpha_out = ddiv(1.0, m);
  }
}

__global__ void k_fill_alpha(int n, const double* __restrict__ alpha, double* w) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) w[r] = *alpha;
}

__global__ void k_mean(int n, const double* __restrict__ w, double* out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) s = dadd(s, w[r]);
  sm[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < blockDim.x; ++k) t = dadd(t, sm[k]);
    *out = n > 0 ? ddiv(t, (double)n) : 0.0;
  }
}

__global__ void k_fill_int(int* p, int v, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}

}  // namespace

static std::atomic<uint64_t> g_alloc_gen{0};

uint64_t alloc_generation() { return g_alloc_gen.load(); }

// ---- device memory cache ------------------------------------------------------
// Every device buffer of the library comes from here: a freed buffer is kept
// (per device, by size) and handed to the next request of 1 to 1.5 times less
// size, so batches and handles created again and again (a serving loop, the
// bench's e2e leg) neither pay cudaMalloc/cudaFree -- cudaFree synchronises the
// device -- nor see their cost vary run to run. At most kPoolCap bytes stay
// cached; a failing cudaMalloc first returns the device's cached blocks.
namespace {
struct PoolBlock { void* p; size_t bytes; int dev; };
std::mutex g_pool_mu;
std::multimap<size_t, PoolBlock> g_pool;                       // cached (free) blocks by size
std::unordered_map<void*, std::pair<size_t, int>> g_live;    // blocks handed out: size, device
size_t g_pool_bytes = 0;
constexpr size_t kPoolCap = (size_t)48 << 30;

void pool_release_dev(int dev) {  // caller holds the lock
  for (auto it = g_pool.begin(); it != g_pool.end();) {
    if (it->second.dev == dev) {
      cudaFree(it->second.p);
      g_pool_bytes -= it->second.bytes;
      it = g_pool.erase(it);
    } else {
      ++it;
    }
  }
}
}  // namespace

cudaError_t dev_alloc(void** p, size_t bytes, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto it = g_pool.lower_bound(bytes); it != g_pool.end() && it->first <= bytes + bytes / 2; ++it)
    if (it->second.dev == dev) {
      *p = it->second.p;
      *got = it->second.bytes;
      g_pool_bytes -= it->second.bytes;
      g_live[*p] = {it->second.bytes, dev};
      g_pool.erase(it);
      return cudaSuccess;
    }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    pool_release_dev(dev);
    e = cudaMalloc(p, bytes);
  }
  if (e != cudaSuccess) {
    *p = nullptr;
    *got = 0;
    return e;
  }
  *got = bytes;
  g_live[*p] = {bytes, dev};
  return cudaSuccess;
}

void dev_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_live.find(p);
  if (it == g_live.end()) {  // not ours
    cudaFree(p);
    return;
  }
  const size_t bytes = it->second.first;
  const int dev = it->second.second;
  g_live.erase(it);
  {  // as cudaFree: work still in flight on the device may use the block
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev) cudaSetDevice(dev);
    cudaDeviceSynchronize();
    if (cur != dev) cudaSetDevice(cur);
  }
  g_pool.insert({bytes, PoolBlock{p, bytes, dev}});
  g_pool_bytes += bytes;
  while (g_pool_bytes > kPoolCap && !g_pool.empty()) {  // over the cap: drop the largest
    auto last = std::prev(g_pool.end());
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(last->second.dev);
    cudaFree(last->second.p);
    cudaSetDevice(cur);
    g_pool_bytes -= last->second.bytes;
    g_pool.erase(last);
  }
}

cudaError_t ensure(Workspace::Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (b.cap >= bytes) return cudaSuccess;
  g_alloc_gen.fetch_add(1);  // invalidates captured setup graphs
  dev_free(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t got = 0;
  cudaError_t e = dev_alloc(&b.p, bytes + bytes / 4, &got);
  if (e == cudaSuccess) b.cap = got;
  return e;
}

template <class T>
static T* P(Workspace::Buf& b) { return reinterpret_cast<T*>(b.p); }

static int end_bit_for(int64_t v) {
  int b = 1;
  while (b < 31 && (int64_t(1) << b) <= v) ++b;
  return b;
}

// Phase 1: column statistics, contact marks, partition into G CTAs, slice
// widths. Ends with ONE host read of the summary (sizes + flags).
int setup_layout_async(Workspace& ws, const vfpi_system& s, int G, cudaStream_t st, std::string& err,
                 int64_t& launches, const LayoutOptions& opt) {
  ++ws.layout_epoch;
  const int n = (int)s.n, n_c = (int)s.n_c;
  const int64_t nnz = s.nnz;
  if (G > 1024) { err = "more than 1024 CTA ranges per layout"; return VFPI_BAD_ARGUMENT; }
  if (opt.scene_row_ptr && opt.anchor_order) { err = "scene batches use the natural unit order"; return VFPI_BAD_ARGUMENT; }
  VFPI_CK(ensure(ws.diag, 8 * (size_t)n));
  VFPI_CK(ensure(ws.rns, 8 * (size_t)n));
  VFPI_CK(ensure(ws.rowcnt, 4 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.row_ptr, 8 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.keys, 4 * (size_t)nnz));
  VFPI_CK(ensure(ws.colof, 4 * (size_t)nnz));
  VFPI_CK(ensure(ws.mark, 4 * (size_t)n));
  VFPI_CK(ensure(ws.ucost, 8 * (size_t)n));
  VFPI_CK(ensure(ws.cpos, 8 * (size_t)n));
  VFPI_CK(ensure(ws.urows, 4 * (size_t)n));
  VFPI_CK(ensure(ws.rpos, 4 * (size_t)n));
  VFPI_CK(ensure(ws.ucont, 4 * (size_t)n));
  VFPI_CK(ensure(ws.kpos, 4 * (size_t)n));
  VFPI_CK(ensure(ws.ucr, 4 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.rowmin, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.ukey, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.ukey_s, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.uval, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.uorder, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.ufr, 4 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.cposc, 4 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.cposf, 4 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.blk_first, 4 * (size_t)(G + 1)));
  VFPI_CK(ensure(ws.blk_cr, 4 * (size_t)(G + 1)));
  VFPI_CK(ensure(ws.cont_q, 4 * (size_t)std::max(n_c, 1)));
  VFPI_CK(ensure(ws.blk_row, 4 * (size_t)(G + 1)));
  VFPI_CK(ensure(ws.blk_ct, 4 * (size_t)(G + 1)));
  VFPI_CK(ensure(ws.blk_slice, 4 * (size_t)(G + 1)));
  VFPI_CK(ensure(ws.row_list, 4 * (size_t)n));
  VFPI_CK(ensure(ws.row_slot, 4 * (size_t)n));
  VFPI_CK(ensure(ws.cont_list, 4 * (size_t)n_c));
  VFPI_CK(ensure(ws.flags, 16));
  VFPI_CK(ensure(ws.summary, sizeof(SetupSummary)));
  const int S_max = (n + 31) / 32 + G;  // each CTA rounds its row count up once
  VFPI_CK(ensure(ws.slice_w, 8 * (size_t)(S_max + 1)));
  VFPI_CK(ensure(ws.slice_off, 8 * (size_t)(S_max + 1)));
  VFPI_CK(ensure(ws.pos_len, 8 * (size_t)(n + 1)));
  VFPI_CK(ensure(ws.pos_ptr, 8 * (size_t)(n + 1)));

  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, P<int>(ws.rowcnt), P<int64_t>(ws.row_ptr), n + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, P<int64_t>(ws.ucost), P<int64_t>(ws.cpos), n, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, P<int>(ws.urows), P<int>(ws.rpos), n + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, P<int64_t>(ws.slice_w), P<int64_t>(ws.slice_off), S_max + 1, st);
  size_t t5 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t5, P<int64_t>(ws.pos_len), P<int64_t>(ws.pos_ptr), n + 1, st);
  VFPI_CK(ensure(ws.cub_tmp, std::max(std::max(std::max(t1, t2), std::max(t3, t4)), t5)));
  size_t tb = ws.cub_tmp.cap;

  VFPI_CK(cudaMemsetAsync(ws.rowcnt.p, 0, 4 * (size_t)(n + 1), st));
  VFPI_CK(cudaMemsetAsync(ws.rowmin.p, 0x7f, 4 * (size_t)std::max(n, 1), st));  // ~INT_MAX
  VFPI_CK(cudaMemsetAsync(ws.mark.p, 0xff, 4 * (size_t)n, st));
  VFPI_CK(cudaMemsetAsync(ws.flags.p, 0, 16, st));
  VFPI_CK(cudaMemsetAsync(ws.summary.p, 0, sizeof(SetupSummary), st));
  k_fill_int<<<nblk(G + 1), 256, 0, st>>>(P<int>(ws.blk_row), INT_MAX, G + 1);
  k_fill_int<<<nblk(G + 1), 256, 0, st>>>(P<int>(ws.blk_ct), INT_MAX, G + 1);
  k_fill_int<<<nblk(G + 1), 256, 0, st>>>(P<int>(ws.blk_first), INT_MAX, G + 1);
  launches += 3;
  if (n > 0) {
    k_colstats<<<nblk(n), 256, 0, st>>>(n, s.indptr, s.indices, s.data, P<double>(ws.diag), P<double>(ws.rns),
                                        P<int>(ws.rowcnt), P<int>(ws.keys), P<int>(ws.colof), P<int>(ws.rowmin));
    ++launches;
  }
  if (n_c > 0) {
    k_mark<<<nblk(n_c), 256, 0, st>>>(n, n_c, s.col_i, s.col_j, P<int>(ws.mark), P<int>(ws.flags));
    ++launches;
  }
  VFPI_CK(cudaGetLastError());
  VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.rowcnt), P<int64_t>(ws.row_ptr), n + 1, st));
  ++launches;
  if (n > 0) {
    k_unit_keys<<<nblk(n), 256, 0, st>>>(n, P<int>(ws.mark), s.col_i, s.col_j, P<int>(ws.rowmin), P<int>(ws.ukey),
                                         P<int>(ws.uval), opt.anchor_order ? 1 : 0);
    // natural order: keys are already the start rows (non-starts = n stay
    // interleaved as empty units), so only the anchor order needs a sort
    int* skey = P<int>(ws.ukey);
    int* uord = P<int>(ws.uval);
    if (opt.anchor_order) {
      size_t tu = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tu, P<int>(ws.ukey), P<int>(ws.ukey_s), P<int>(ws.uval),
                                      P<int>(ws.uorder), n, 0, end_bit_for(n), st);
      VFPI_CK(ensure(ws.cub_tmp, tu));
      tb = ws.cub_tmp.cap;
      VFPI_CK(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.p, tb, P<int>(ws.ukey), P<int>(ws.ukey_s), P<int>(ws.uval),
                                              P<int>(ws.uorder), n, 0, end_bit_for(n), st));
      skey = P<int>(ws.ukey_s);
      uord = P<int>(ws.uorder);
    }
    ws.unit_order_is_sorted = opt.anchor_order;
    k_units<<<nblk(n + 1), 256, 0, st>>>(n, skey, uord, P<int>(ws.mark), s.col_i, s.col_j,
                                         P<int>(ws.rowcnt), P<int64_t>(ws.ucost), P<int>(ws.urows), P<int>(ws.ucont),
                                         P<int>(ws.ucr), P<int>(ws.ufr), opt.entry_cost, opt.row_cost,
                                         opt.contact_cost);
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int64_t>(ws.ucost), P<int64_t>(ws.cpos), n, st));
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.urows), P<int>(ws.rpos), n, st));
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.ucont), P<int>(ws.kpos), n, st));
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.ucr), P<int>(ws.cposc), n + 1, st));
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.ufr), P<int>(ws.cposf), n + 1, st));
    if (opt.scene_row_ptr) {
      // scene batch: CTA b = scene b; in natural unit order the rows of earlier
      // scenes precede every unit of scene b, so its start is scene_row_ptr[b]
      VFPI_CK(cudaMemcpyAsync(ws.blk_row.p, opt.scene_row_ptr, 4 * (size_t)(G + 1), cudaMemcpyDeviceToDevice, st));
      VFPI_CK(cudaMemcpyAsync(ws.blk_ct.p, opt.scene_ct_ptr, 4 * (size_t)(G + 1), cudaMemcpyDeviceToDevice, st));
      VFPI_CK(cudaMemcpyAsync(ws.blk_first.p, opt.scene_row_ptr, 4 * (size_t)(G + 1), cudaMemcpyDeviceToDevice, st));
    } else {
      k_blocks<<<nblk(n), 256, 0, st>>>(n, G, P<int64_t>(ws.ucost), P<int64_t>(ws.cpos), P<int>(ws.urows),
                                        P<int>(ws.rpos), P<int>(ws.kpos), P<int>(ws.blk_row), P<int>(ws.blk_ct),
                                        P<int>(ws.blk_first));
    }
    launches += 7;
  } else {
    VFPI_CK(cudaMemsetAsync(ws.cposc.p, 0, 4, st));
  }
  k_blocks_fix<<<1, kFixThreads, 0, st>>>(n, n_c, G, P<int>(ws.blk_row), P<int>(ws.blk_ct), P<int>(ws.blk_slice),
                                P<int>(ws.blk_first), P<int>(ws.blk_cr), P<int>(ws.cposc),
                                P<SetupSummary>(ws.summary));
  ++launches;
  // with the length sort, k_fill writes a scratch list that the permutation
  // copies into row_list (fixed buffer roles: replayable as a captured graph)
  const bool lsort = opt.length_sort && n > 0 && G <= 4096;
  if (lsort) {
    VFPI_CK(ensure(ws.row_list2, 4 * (size_t)n));
    VFPI_CK(ensure(ws.row_slot2, 4 * (size_t)n));
  }
  int* fill_list = lsort ? P<int>(ws.row_list2) : P<int>(ws.row_list);
  int* fill_slot = lsort ? P<int>(ws.row_slot2) : P<int>(ws.row_slot);
  if (n > 0) {
    k_fill<<<nblk(n), 256, 0, st>>>(n, G, opt.anchor_order ? P<int>(ws.uorder) : P<int>(ws.uval), P<int>(ws.mark),
                                    s.col_i, s.col_j, P<int>(ws.urows),
                                    P<int>(ws.rpos),
                                    P<int>(ws.kpos), P<int>(ws.cposc), P<int>(ws.cposf), P<int>(ws.blk_row),
                                    P<int>(ws.blk_ct), P<int>(ws.blk_first), P<int>(ws.blk_cr), fill_list,
                                    fill_slot, P<int>(ws.cont_list), P<int>(ws.cont_q));
    ++launches;
  }
  VFPI_CK(cudaGetLastError());
  if (lsort) {
    k_row_keys<<<nblk(n), 256, 0, st>>>(n, G, fill_list, fill_slot, P<int>(ws.rowcnt),
                                        P<int>(ws.blk_row), P<int>(ws.ukey), P<int>(ws.uval));
    size_t tr = 0;
    const int eb = end_bit_for((int64_t)G << 9);
    cub::DeviceRadixSort::SortPairs(nullptr, tr, P<int>(ws.ukey), P<int>(ws.ukey_s), P<int>(ws.uval),
                                    P<int>(ws.uorder), n, 0, eb, st);
    VFPI_CK(ensure(ws.cub_tmp, tr));
    tb = ws.cub_tmp.cap;
    VFPI_CK(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.p, tb, P<int>(ws.ukey), P<int>(ws.ukey_s), P<int>(ws.uval),
                                            P<int>(ws.uorder), n, 0, eb, st));
    k_row_permute<<<nblk(n), 256, 0, st>>>(n, P<int>(ws.uorder), fill_list, fill_slot, P<int>(ws.row_list),
                                           P<int>(ws.row_slot));
    launches += 2 + 2 + (eb + 7) / 8;
  }
  // slice count is data dependent but bounded by S_max; slices past the real
  // count get width 0, so one scan over S_max+1 entries suffices.
  k_slice_width<<<nblk((int64_t)(S_max + 1) * 32), 256, 0, st>>>(S_max, G, P<SetupSummary>(ws.summary), P<int>(ws.blk_slice),
                                                 P<int>(ws.blk_row), P<int>(ws.row_list), P<int>(ws.rowcnt),
                                                 P<int64_t>(ws.slice_w));
  VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int64_t>(ws.slice_w), P<int64_t>(ws.slice_off),
                                        S_max + 1, st));
  k_poslen<<<nblk(n + 1), 256, 0, st>>>(n, P<int>(ws.row_list), P<int>(ws.rowcnt), P<int64_t>(ws.pos_len));
  VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int64_t>(ws.pos_len), P<int64_t>(ws.pos_ptr), n + 1,
                                        st));
  // gather plan of the resident kernel (remote 32-byte sectors per CTA)
  VFPI_CK(ensure(ws.rowpos, 4 * (size_t)std::max(n, 1)));
  VFPI_CK(ensure(ws.sec_key, 4 * (size_t)std::max<int64_t>(nnz, 1)));
  VFPI_CK(ensure(ws.sec_skey, 4 * (size_t)std::max<int64_t>(nnz, 1)));
  VFPI_CK(ensure(ws.sec_flag, 4 * (size_t)std::max<int64_t>(nnz, 1)));
  VFPI_CK(ensure(ws.sec_upos, 4 * (size_t)std::max<int64_t>(nnz, 1)));
  VFPI_CK(ensure(ws.secs, 4 * (size_t)std::max<int64_t>(nnz, 1)));
  VFPI_CK(ensure(ws.sec_ptr, 4 * (size_t)(G + 1)));
  VFPI_CK(cudaMemsetAsync(ws.sec_ptr.p, 0xff, 4 * (size_t)(G + 1), st));
  if (n > 0 && nnz > 0 && G <= 256 && n < (1 << 26)) {
    VFPI_CK(ensure(ws.rowblk, 4 * (size_t)n));
    k_rowpos<<<nblk(n), 256, 0, st>>>(n, G, P<int>(ws.row_list), P<int>(ws.blk_row), P<int>(ws.rowpos),
                                      P<int>(ws.rowblk));
    // key bits: CTA above the sector id; every real key stays below the
    // all-ones kNoSector (both fields strictly below their maxima)
    int SB = end_bit_for((n - 1) / 4 + 1);
    int KB = SB + end_bit_for(G);
    if (KB > 32) { SB = 24; KB = 32; }
    k_sec_keys<<<nblk(n), 256, 0, st>>>(n, s.indptr, s.indices, s.data, P<int>(ws.rowblk), P<unsigned>(ws.sec_key),
                                        SB);
    size_t tk = 0, tsc = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tk, P<unsigned>(ws.sec_key), P<unsigned>(ws.sec_skey), (int)nnz, 0, KB,
                                   st);
    cub::DeviceScan::ExclusiveSum(nullptr, tsc, P<int>(ws.sec_flag), P<int>(ws.sec_upos), (int)nnz, st);
    VFPI_CK(ensure(ws.cub_tmp, std::max(tk, tsc)));
    tb = ws.cub_tmp.cap;
    VFPI_CK(cub::DeviceRadixSort::SortKeys(ws.cub_tmp.p, tb, P<unsigned>(ws.sec_key), P<unsigned>(ws.sec_skey),
                                           (int)nnz, 0, KB, st));
    k_sec_flags<<<nblk(nnz), 256, 0, st>>>(nnz, P<unsigned>(ws.sec_skey), P<int>(ws.sec_flag));
    VFPI_CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tb, P<int>(ws.sec_flag), P<int>(ws.sec_upos), (int)nnz, st));
    k_sec_emit<<<nblk(nnz), 256, 0, st>>>(nnz, P<unsigned>(ws.sec_skey), P<int>(ws.sec_flag), P<int>(ws.sec_upos),
                                          P<unsigned>(ws.secs), P<int>(ws.sec_ptr), SB);
    k_sec_ptr_fix<<<1, 1024, 0, st>>>(G, nnz, P<int>(ws.sec_flag), P<int>(ws.sec_upos), P<int>(ws.sec_ptr));
    launches += 12;
  } else {
    VFPI_CK(cudaMemsetAsync(ws.sec_ptr.p, 0, 4 * (size_t)(G + 1), st));
  }
  k_summary<<<1, kFixThreads, 0, st>>>(n, G, P<int64_t>(ws.row_ptr), P<int64_t>(ws.slice_off), P<int64_t>(ws.pos_ptr),
                             P<int>(ws.blk_row), P<int>(ws.blk_ct), P<int>(ws.blk_cr), P<int>(ws.blk_slice),
                             P<int>(ws.sec_ptr), P<int>(ws.flags), P<SetupSummary>(ws.summary));
  launches += 6;
  VFPI_CK(cudaGetLastError());
  return VFPI_OK;
}

int setup_layout_finish(Workspace& ws, cudaStream_t st, SetupSummary* hs, std::string& err) {
  VFPI_CK(cudaMemcpyAsync(hs, ws.summary.p, sizeof(SetupSummary), cudaMemcpyDeviceToHost, st));
  VFPI_CK(cudaStreamSynchronize(st));
  if (hs->flags & 2) { err = "contact column index out of range"; return VFPI_BAD_ARGUMENT; }
  if (hs->flags & 1) {
    err = "two contacts share a node column (nodalization guarantees one contact per node, contacts.py:242-268)";
    return VFPI_UNSUPPORTED;
  }

  return VFPI_OK;
}

// Phase 2: stable radix sort of CSC entries by row -> per-row increasing
// column order (scipy's accumulation order), then packing for the kernel.
int setup_pack(Workspace& ws, const vfpi_system& s, int G, bool resident, const SetupSummary& hs, cudaStream_t st,
               std::string& err, int64_t& launches) {
  ++ws.layout_epoch;
  const int n = (int)s.n;
  const int64_t nnz = s.nnz;
  const int S = hs.n_slices;
  VFPI_CK(ensure(ws.vals, 4 * (size_t)nnz));
  VFPI_CK(ensure(ws.perm, 4 * (size_t)nnz));
  VFPI_CK(ensure(ws.keys_sorted, 4 * (size_t)nnz));
  if (nnz > 0) {
    const int eb = end_bit_for(n);
    size_t ts = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, ts, P<int>(ws.keys), P<int>(ws.keys_sorted), P<int>(ws.vals),
                                    P<int>(ws.perm), (int)nnz, 0, eb, st);
    VFPI_CK(ensure(ws.cub_tmp, ts));
    size_t tb = ws.cub_tmp.cap;
    k_iota<<<nblk(nnz), 256, 0, st>>>(nnz, P<int>(ws.vals));
    VFPI_CK(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.p, tb, P<int>(ws.keys), P<int>(ws.keys_sorted),
                                            P<int>(ws.vals), P<int>(ws.perm), (int)nnz, 0, eb, st));
    launches += 3 + (eb + 7) / 8;  // iota, histogram, exclusive-sum, one onesweep pass per 8 key bits
  }
  VFPI_CK(ensure(ws.sell_val, 8 * (size_t)std::max<int64_t>(hs.sell_elems, 1)));
  VFPI_CK(ensure(ws.sell_col, 4 * (size_t)std::max<int64_t>(hs.sell_elems, 1)));
  if (S > 0) {
    k_pack<<<nblk((int64_t)S * 32), 256, 0, st>>>(S, G, P<int>(ws.blk_slice), P<int>(ws.blk_row),
                                                  P<int>(ws.row_list), P<int>(ws.rowcnt), P<int64_t>(ws.row_ptr),
                                                  P<int>(ws.perm), P<int>(ws.colof), s.data,
                                                  P<int64_t>(ws.slice_off), P<double>(ws.sell_val),
                                                  P<int>(ws.sell_col));
    ++launches;
  }
  if (resident) {
    VFPI_CK(ensure(ws.sell_map, 4 * (size_t)std::max<int64_t>(hs.sell_elems, 1)));
    if (S > 0) {
      k_sell_map<<<G, 1024, 0, st>>>(G, P<int>(ws.blk_slice), P<int>(ws.blk_row), P<int64_t>(ws.slice_off),
                                    P<int>(ws.sell_col), P<int>(ws.rowpos), P<unsigned>(ws.secs), P<int>(ws.sec_ptr),
                                    P<unsigned>(ws.sell_map));
      ++launches;
    }
  }
  VFPI_CK(cudaGetLastError());
  return VFPI_OK;
}

// W (frobenius / fixed-alpha / cached) and gamma; flags reported through ws.flags
int setup_step_matrix(Workspace& ws, const vfpi_system& s, const vfpi_config& cfg, const double* d_w_cached,
                      cudaStream_t st, std::string& err, int64_t& launches, const int* d_nc) {
  const int n = (int)s.n, n_c = (int)s.n_c;
  VFPI_CK(ensure(ws.w, 8 * (size_t)n));
  VFPI_CK(ensure(ws.gamma, 8 * (size_t)n_c));
  VFPI_CK(ensure(ws.w_mean, 16));
  double* w = P<double>(ws.w);
  if (cfg.step_strategy == VFPI_STEP_FIXED_ALPHA) {
    if (std::isnan(cfg.fixed_alpha)) {
      k_absmax_alpha<<<1, 256, 0, st>>>(n, P<double>(ws.diag), P<double>(ws.w_mean) + 1);
      ++launches;
    } else {
      VFPI_CK(cudaMemcpyAsync(P<double>(ws.w_mean) + 1, &cfg.fixed_alpha, 8, cudaMemcpyHostToDevice, st));
    }
    if (n > 0) {
      k_fill_alpha<<<nblk(n), 256, 0, st>>>(n, P<double>(ws.w_mean) + 1, w);
      ++launches;
    }
  } else if (d_w_cached != nullptr) {
    VFPI_CK(cudaMemcpyAsync(w, d_w_cached, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  } else {
    if (n > 0) {
      k_w_frob<<<nblk(n), 256, 0, st>>>(n, P<double>(ws.diag), P<double>(ws.rns), w, P<int>(ws.flags));
      ++launches;
    }
    if (n_c > 0) {
      k_tie<<<nblk(n_c), 256, 0, st>>>(n_c, cfg.op == VFPI_OP_PROXIMAL ? 1 : 0, s.col_i, s.col_j,
                                       P<double>(ws.diag), P<double>(ws.rns), w, d_nc);
      ++launches;
    }
  }
  if (n_c > 0) {
    k_gamma<<<nblk(n_c), 256, 0, st>>>(n_c, s.col_i, s.col_j, w, cfg.omega, P<double>(ws.gamma), P<int>(ws.flags),
                                       d_nc);
    ++launches;
  }
  const bool bb = cfg.step_strategy >= VFPI_STEP_BB1 && cfg.step_strategy <= VFPI_STEP_BB_ALTERNATING;
  if (bb) {
    k_mean<<<1, 256, 0, st>>>(n, w, P<double>(ws.w_mean));
    ++launches;
  }
  VFPI_CK(cudaGetLastError());
  return VFPI_OK;
}


namespace {

// contact k of the CTA (scene) b whose contact range holds k: its rows get
// slots (k - ct[b]) * 6 + q, the row order itself is unchanged
__global__ void k_refresh_slots(int n_c, int G, const int* __restrict__ ci, const int* __restrict__ cj,
                                const int* __restrict__ ct, const int* __restrict__ rowpos, int* __restrict__ row_slot,
                                int* __restrict__ cont_list) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_c) return;
  const int b = owner(ct, G, k);
  const int loc = (k - ct[b]) * kSlotsPerContact;
  cont_list[k] = k;
  const int i = ci[k], j = cj[k];
  for (int q = 0; q < 3; ++q) row_slot[rowpos[i + q]] = loc + q;
  if (j >= 0)
    for (int q = 0; q < 3; ++q) row_slot[rowpos[j + q]] = loc + 3 + q;
}

__global__ void k_rowpos_only(int n, const int* __restrict__ row_list, int* __restrict__ rowpos) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) rowpos[row_list[q]] = q;
}

}  // namespace

int setup_rowpos(Workspace& ws, int n, int G, cudaStream_t st, std::string& err) {
  (void)G;
  VFPI_CK(ensure(ws.rowpos, 4 * (size_t)std::max(n, 1)));
  if (n > 0) k_rowpos_only<<<nblk(n), 256, 0, st>>>(n, P<int>(ws.row_list), P<int>(ws.rowpos));
  VFPI_CK(cudaGetLastError());
  return VFPI_OK;
}

int setup_contacts_refresh(Workspace& ws, const vfpi_system& s, int G, const int* d_scene_ct_ptr, cudaStream_t st,
                           std::string& err, int64_t& launches) {
  const int n = (int)s.n, n_c = (int)s.n_c;
  VFPI_CK(ensure(ws.cont_list, 4 * (size_t)std::max(n_c, 1)));
  VFPI_CK(cudaMemsetAsync(ws.row_slot.p, 0xff, 4 * (size_t)std::max(n, 1), st));
  VFPI_CK(cudaMemcpyAsync(ws.blk_ct.p, d_scene_ct_ptr, 4 * (size_t)(G + 1), cudaMemcpyDeviceToDevice, st));
  VFPI_CK(cudaMemsetAsync(ws.flags.p, 0, 16, st));
  if (n_c > 0) {
    k_refresh_slots<<<nblk(n_c), 256, 0, st>>>(n_c, G, s.col_i, s.col_j, d_scene_ct_ptr, P<int>(ws.rowpos),
                                                P<int>(ws.row_slot), P<int>(ws.cont_list));
    ++launches;
  }
  VFPI_CK(cudaGetLastError());
  return VFPI_OK;
}

}  // namespace vfpi
