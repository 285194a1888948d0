// Virtual-node augmentation of the dynamics on the device:
// the reference's augment_dynamics (condsim/contacts.py:343-375),
//
//   A = [[A_o + k_v J_v^T J_v, -k_v J_v^T],      b = [b_o; 0]
//        [-k_v J_v,             k_v I    ]]
//
// evaluated with the same floating-point operations, in the same order, and
// with the same stored-entry rules as its scipy expression, so the output CSC
// arrays equal SparseSymmetric.from_scipy(sp.bmat(...)) bit for bit:
//   * J_v^T J_v is scipy's csr_matmat of jv.T (rows i) with jv: entry (i, j)
//     = 0 + sum over virtual rows r ascending of jv[r,i] * jv[r,j]; sums that
//     are exactly 0 are not stored;
//   * k_v * (J_v^T J_v) scales the stored values;
//   * A_o + that is scipy's csr_binop (op = plus): entries of the union of
//     both patterns, a + t, a + 0 or 0 + t, and a result of exactly 0 is
//     not stored (explicit zeros of A_o vanish here);
//   * the off-diagonal blocks keep every stored entry of J_v, explicit zeros
//     included, with value (-k_v) * x; the identity block is k_v * 1.0;
//   * with no virtual nodes A is A_o unchanged (contacts.py:349-350).
// Products with a zero factor are skipped in the sums: adding a signed zero to
// a running sum never changes it, and an all-zero sum is dropped either way.
//
// Layout of the work (all O(entries), one host read of the output size):
//   1. per J_v row: (nonzeros)^2 products keyed (j << 32 | i), written in
//      row order; a stable radix sort by key keeps r ascending in every run;
//   2. runs are summed sequentially by their head thread (run lengths are the
//      number of virtual nodes tied to both i and j: a handful);
//   3. J_v transposed to CSC by a stable sort on its columns (r ascending);
//   4. per column of A_o: a two-pointer merge with the (i, t) run list of that
//      column counts the surviving entries, a scan gives the output column
//      pointers, the same merge writes them, followed by the J_v column.
#include <cub/cub.cuh>

#include "vfpi_internal.cuh"
#include "vfpi_math.cuh"

namespace vfpi {

namespace {

constexpr int kT = 256;

inline unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

// nonzero entries per J_v row -> products per row (count^2)
// (also validates J_v: columns inside [0, n_o), strictly increasing per row)
__global__ void k_aug_prod_count(int rows, int n_o, int64_t jnnz, const int* __restrict__ jp,
                                 const int* __restrict__ jc, const double* __restrict__ jx, int64_t* __restrict__ cnt,
                                 int* __restrict__ bad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > rows) return;
  if (r == rows) {
    cnt[r] = 0;
    if (jp[0] != 0 || jp[rows] != jnnz) atomicExch(bad, 1);
    return;
  }
  if (jp[r] < 0 || jp[r] > jp[r + 1] || jp[r + 1] > jnnz) {  // not a CSR row pointer: do not walk it
    atomicExch(bad, 1);
    cnt[r] = 0;
    return;
  }
  int64_t c = 0;
  int prev = -1;
  for (int e = jp[r]; e < jp[r + 1]; ++e) {
    c += (jx[e] != 0.0);
    const int col = jc[e];
    if (col <= prev || col >= n_o) atomicExch(bad, 1);
    prev = col;
  }
  cnt[r] = c * c;
}

__global__ void k_aug_zero(int* p) { *p = 0; }

// A_o must be CSC with strictly increasing row indices in [0, n_o) per column
__global__ void k_aug_check_a(int n_o, int64_t nnz, const int* __restrict__ ap, const int* __restrict__ ai,
                              int* __restrict__ bad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_o) return;
  if (c == n_o) {
    if (ap[0] != 0 || ap[n_o] != nnz) atomicExch(bad, 1);
    return;
  }
  const int e0 = ap[c], e1 = ap[c + 1];
  if (e0 < 0 || e0 > e1 || e1 > nnz) { atomicExch(bad, 1); return; }
  int prev = -1;
  for (int e = e0; e < e1; ++e) {
    const int r = ai[e];
    if (r <= prev || r >= n_o) { atomicExch(bad, 1); return; }
    prev = r;
  }
}

// products of row r in (i-entry, j-entry) order; key = (j << 32) | i
__global__ void k_aug_prod_fill(int rows, const int* __restrict__ jp, const int* __restrict__ jc,
                                const double* __restrict__ jx, const int64_t* __restrict__ off,
                                unsigned long long* __restrict__ key, double* __restrict__ val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t o = off[r];
  for (int ea = jp[r]; ea < jp[r + 1]; ++ea) {
    const double xa = jx[ea];
    if (xa == 0.0) continue;
    const unsigned long long i = (unsigned)jc[ea];
    for (int eb = jp[r]; eb < jp[r + 1]; ++eb) {
      const double xb = jx[eb];
      if (xb == 0.0) continue;
      key[o] = ((unsigned long long)(unsigned)jc[eb] << 32) | i;
      val[o] = dmul(xa, xb);  // scipy csr_matmat: v * Bx[kk] with v = (jv.T)[i, r]
      ++o;
    }
  }
}

// run heads of the sorted product keys
__global__ void k_aug_heads(int64_t m, const unsigned long long* __restrict__ key, int* __restrict__ head) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p > m) return;
  if (p == m) { head[p] = 0; return; }
  head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}

// each head sums its run in order (0 + p0 + p1 + ...); zero sums are marked
// dropped (row -1); survivors are scaled by k_v (scipy's k_v * JtJ)
__global__ void k_aug_runs(int64_t m, const unsigned long long* __restrict__ key, const double* __restrict__ val,
                           const int* __restrict__ head, const int* __restrict__ hpos, double kv,
                           int* __restrict__ t_row, int* __restrict__ t_col, double* __restrict__ t_val) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= m || !head[p]) return;
  double s = 0.0;
  int64_t q = p;
  const unsigned long long k = key[p];
  do {
    s = dadd(s, val[q]);
    ++q;
  } while (q < m && key[q] == k);
  const int o = hpos[p];
  t_col[o] = (int)(k >> 32);
  t_row[o] = s != 0.0 ? (int)(k & 0xffffffffull) : -1;
  t_val[o] = dmul(s, kv);
}

// first run of every column (runs sorted by (col, row)); col_start[n_o] = runs
__global__ void k_aug_col_start(int n_o, int64_t runs, const int* __restrict__ t_col, int64_t* __restrict__ cs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n_o) return;
  int64_t lo = 0, hi = runs;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t_col[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  cs[j] = lo;
}

// J_v CSR -> entry keys for the column sort (stable: r ascending per column)
__global__ void k_aug_jv_rows(int rows, const int* __restrict__ jp, int* __restrict__ row_of) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (int e = jp[r]; e < jp[r + 1]; ++e) row_of[e] = r;
}

__global__ void k_aug_iota(int64_t n, int* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int)i;
}

// column pointers of J_v's CSC view from its sorted column keys
__global__ void k_aug_jv_colptr(int n_o, int64_t nnz, const int* __restrict__ col_sorted, int64_t* __restrict__ cp) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n_o) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col_sorted[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  cp[j] = lo;
}

// merge of A_o column j with the k_v JtJ runs of column j (scipy csr_binop,
// op = plus, zero results dropped). WRITE = false: count only.
template <bool WRITE>
__global__ void k_aug_merge(int n_o, int n_v3, const int* __restrict__ ap, const int* __restrict__ ai,
                            const double* __restrict__ ax, const int64_t* __restrict__ cs,
                            const int* __restrict__ t_row, const double* __restrict__ t_val,
                            const int64_t* __restrict__ jcp, const int* __restrict__ jperm,
                            const int* __restrict__ jrow_of, const double* __restrict__ jx,
                            const int* __restrict__ jp, const int* __restrict__ jc, double neg_kv, double kv,
                            int64_t* __restrict__ cnt, const int64_t* __restrict__ outp, int* __restrict__ oi,
                            double* __restrict__ ox) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_o + n_v3) return;
  int64_t o = WRITE ? outp[c] : 0;
  int64_t k = 0;
  auto put = [&](int row, double v) {
    if (WRITE) {
      oi[o] = row;
      ox[o] = v;
      ++o;
    } else {
      ++k;
    }
  };
  if (c < n_o) {
    int pa = ap[c];
    const int ea = ap[c + 1];
    int64_t pt = cs[c];
    const int64_t et = cs[c + 1];
    while (pt < et && t_row[pt] < 0) ++pt;
    while (pa < ea || pt < et) {
      const int ra = pa < ea ? ai[pa] : INT_MAX;
      const int rt = pt < et ? t_row[pt] : INT_MAX;
      double r;
      int row;
      if (ra == rt) {
        r = dadd(ax[pa], t_val[pt]);
        row = ra;
        ++pa;
        ++pt;
      } else if (ra < rt) {
        r = dadd(ax[pa], 0.0);
        row = ra;
        ++pa;
      } else {
        r = dadd(0.0, t_val[pt]);
        row = rt;
        ++pt;
      }
      while (pt < et && t_row[pt] < 0) ++pt;
      if (r != 0.0) put(row, r);
    }
    // block [1][0] = -k_v J_v: column c holds J_v[:, c] (r ascending)
    for (int64_t q = jcp[c]; q < jcp[c + 1]; ++q) {
      const int e = jperm[q];
      put(n_o + jrow_of[e], dmul(neg_kv, jx[e]));
    }
  } else {
    // block [0][1] = -k_v J_v^T: column n_o + r holds J_v[r, :]; then k_v I
    const int r = c - n_o;
    for (int e = jp[r]; e < jp[r + 1]; ++e) put(jc[e], dmul(neg_kv, jx[e]));
    put(c, dmul(kv, 1.0));
  }
  if (!WRITE) cnt[c] = k;
}

__global__ void k_aug_to_i32(int64_t n, const int64_t* __restrict__ a, int* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = (int)a[i];
}

template <class T>
T* B(Workspace::Buf& b) { return reinterpret_cast<T*>(b.p); }

}  // namespace

#define AK(x)                                                        \
  do {                                                               \
    cudaError_t e_ = (x);                                            \
    if (e_ != cudaSuccess) {                                         \
      err = std::string("augment: ") + #x + ": " + cudaGetErrorString(e_); \
      return VFPI_CUDA_ERROR;                                        \
    }                                                                \
  } while (0)

int augment_device(AugmentWork& w, const AugmentIn& in, cudaStream_t st, AugmentOut& out, std::string& err,
                   int64_t& launches) {
  const int n_o = in.n_o, rows = in.n_v3;
  const int n = n_o + rows;
  out.n = n;
  if (n_o < 0 || rows < 0 || rows % 3 != 0 || in.a_nnz < 0 || in.jv_nnz < 0) {
    err = "augment: bad sizes";
    return VFPI_BAD_ARGUMENT;
  }
  if (rows == 0) {  // contacts.py:349-350: A_o unchanged
    AK(ensure(w.out_p, sizeof(int) * (size_t)(n_o + 1)));
    AK(ensure(w.out_i, sizeof(int) * (size_t)in.a_nnz));
    AK(ensure(w.out_x, sizeof(double) * (size_t)in.a_nnz));
    AK(cudaMemcpyAsync(w.out_p.p, in.a_indptr, sizeof(int) * (size_t)(n_o + 1), cudaMemcpyDeviceToDevice, st));
    if (in.a_nnz) {
      AK(cudaMemcpyAsync(w.out_i.p, in.a_indices, sizeof(int) * (size_t)in.a_nnz, cudaMemcpyDeviceToDevice, st));
      AK(cudaMemcpyAsync(w.out_x.p, in.a_data, sizeof(double) * (size_t)in.a_nnz, cudaMemcpyDeviceToDevice, st));
    }
    out.nnz = in.a_nnz;
    out.indptr = B<int>(w.out_p);
    out.indices = B<int>(w.out_i);
    out.data = B<double>(w.out_x);
    return VFPI_OK;
  }
  const int64_t jnnz = in.jv_nnz;
  // 1. products
  AK(ensure(w.pcnt, sizeof(int64_t) * (size_t)(rows + 1)));
  AK(ensure(w.poff, sizeof(int64_t) * (size_t)(rows + 1)));
  AK(ensure(w.cs, sizeof(int64_t) * (size_t)(n_o + 1)));  // its first word doubles as the validation flag
  k_aug_zero<<<1, 1, 0, st>>>(B<int>(w.cs));
  k_aug_prod_count<<<grid_for(rows + 1), kT, 0, st>>>(rows, n_o, jnnz, in.jv_indptr, in.jv_indices, in.jv_data,
                                                      B<int64_t>(w.pcnt), B<int>(w.cs));
  k_aug_check_a<<<grid_for(n_o + 1), kT, 0, st>>>(n_o, in.a_nnz, in.a_indptr, in.a_indices, B<int>(w.cs));
  size_t tb = 0;
  AK(cub::DeviceScan::ExclusiveSum(nullptr, tb, B<int64_t>(w.pcnt), B<int64_t>(w.poff), rows + 1, st));
  AK(ensure(w.tmp, tb));
  AK(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, B<int64_t>(w.pcnt), B<int64_t>(w.poff), rows + 1, st));
  AK(cudaMemcpyAsync(w.h_small, B<int64_t>(w.poff) + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  AK(cudaMemcpyAsync(&w.h_small[1], B<int>(w.cs), sizeof(int), cudaMemcpyDeviceToHost, st));
  AK(cudaStreamSynchronize(st));
  const int64_t m = w.h_small[0];
  if (reinterpret_cast<int*>(&w.h_small[1])[0]) {
    err = "augment: J_v is not canonical CSR with columns in [0, n_o), or A_o not canonical CSC";
    return VFPI_BAD_ARGUMENT;
  }
  launches += 2;
  AK(ensure(w.pkey, sizeof(unsigned long long) * (size_t)m));
  AK(ensure(w.pkey2, sizeof(unsigned long long) * (size_t)m));
  AK(ensure(w.pval, sizeof(double) * (size_t)m));
  AK(ensure(w.pval2, sizeof(double) * (size_t)m));
  AK(ensure(w.head, sizeof(int) * (size_t)(m + 1)));
  AK(ensure(w.hpos, sizeof(int) * (size_t)(m + 1)));
  k_aug_prod_fill<<<grid_for(rows), kT, 0, st>>>(rows, in.jv_indptr, in.jv_indices, in.jv_data, B<int64_t>(w.poff),
                                                 B<unsigned long long>(w.pkey), B<double>(w.pval));
  int hi_bit = 64;
  {
    int b = 0;
    while ((1ll << b) < (int64_t)n_o) ++b;
    hi_bit = 32 + std::max(b, 1);
  }
  if (m > 0) {
    tb = 0;
    AK(cub::DeviceRadixSort::SortPairs(nullptr, tb, B<unsigned long long>(w.pkey), B<unsigned long long>(w.pkey2),
                                       B<double>(w.pval), B<double>(w.pval2), m, 0, hi_bit, st));
    AK(ensure(w.tmp, tb));
    AK(cub::DeviceRadixSort::SortPairs(w.tmp.p, tb, B<unsigned long long>(w.pkey), B<unsigned long long>(w.pkey2),
                                       B<double>(w.pval), B<double>(w.pval2), m, 0, hi_bit, st));
  }
  // 2. runs
  k_aug_heads<<<grid_for(m + 1), kT, 0, st>>>(m, B<unsigned long long>(w.pkey2), B<int>(w.head));
  tb = 0;
  AK(cub::DeviceScan::ExclusiveSum(nullptr, tb, B<int>(w.head), B<int>(w.hpos), m + 1, st));
  AK(ensure(w.tmp, tb));
  AK(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, B<int>(w.head), B<int>(w.hpos), m + 1, st));
  int h_runs = 0;
  AK(cudaMemcpyAsync(&w.h_small[1], B<int>(w.hpos) + m, sizeof(int), cudaMemcpyDeviceToHost, st));
  // 3. J_v columns (overlaps the read above)
  AK(ensure(w.jrow, sizeof(int) * (size_t)std::max<int64_t>(jnnz, 1)));
  AK(ensure(w.jcol_s, sizeof(int) * (size_t)std::max<int64_t>(jnnz, 1)));
  AK(ensure(w.jidx, sizeof(int) * (size_t)std::max<int64_t>(jnnz, 1)));
  AK(ensure(w.jperm, sizeof(int) * (size_t)std::max<int64_t>(jnnz, 1)));
  AK(ensure(w.jcp, sizeof(int64_t) * (size_t)(n_o + 1)));
  k_aug_jv_rows<<<grid_for(rows), kT, 0, st>>>(rows, in.jv_indptr, B<int>(w.jrow));
  k_aug_iota<<<grid_for(jnnz), kT, 0, st>>>(jnnz, B<int>(w.jidx));
  if (jnnz > 0) {
    int cb = 1;
    while ((1ll << cb) < (int64_t)n_o) ++cb;
    tb = 0;
    AK(cub::DeviceRadixSort::SortPairs(nullptr, tb, in.jv_indices, B<int>(w.jcol_s), B<int>(w.jidx), B<int>(w.jperm),
                                       jnnz, 0, cb, st));
    AK(ensure(w.tmp2, tb));
    AK(cub::DeviceRadixSort::SortPairs(w.tmp2.p, tb, in.jv_indices, B<int>(w.jcol_s), B<int>(w.jidx),
                                       B<int>(w.jperm), jnnz, 0, cb, st));
  }
  k_aug_jv_colptr<<<grid_for(n_o + 1), kT, 0, st>>>(n_o, jnnz, B<int>(w.jcol_s), B<int64_t>(w.jcp));
  AK(cudaStreamSynchronize(st));
  h_runs = (int)reinterpret_cast<int*>(&w.h_small[1])[0];
  launches += 8;
  AK(ensure(w.t_row, sizeof(int) * (size_t)std::max(h_runs, 1)));
  AK(ensure(w.t_col, sizeof(int) * (size_t)std::max(h_runs, 1)));
  AK(ensure(w.t_val, sizeof(double) * (size_t)std::max(h_runs, 1)));
  AK(ensure(w.cs, sizeof(int64_t) * (size_t)(n_o + 1)));
  k_aug_runs<<<grid_for(m), kT, 0, st>>>(m, B<unsigned long long>(w.pkey2), B<double>(w.pval2), B<int>(w.head),
                                         B<int>(w.hpos), in.k_v, B<int>(w.t_row), B<int>(w.t_col),
                                         B<double>(w.t_val));
  k_aug_col_start<<<grid_for(n_o + 1), kT, 0, st>>>(n_o, h_runs, B<int>(w.t_col), B<int64_t>(w.cs));
  // 4. count, scan, write
  AK(ensure(w.ccnt, sizeof(int64_t) * (size_t)(n + 1)));
  AK(ensure(w.cptr, sizeof(int64_t) * (size_t)(n + 1)));
  const double neg_kv = -in.k_v;
  k_aug_merge<false><<<grid_for(n), kT, 0, st>>>(n_o, rows, in.a_indptr, in.a_indices, in.a_data, B<int64_t>(w.cs),
                                                 B<int>(w.t_row), B<double>(w.t_val), B<int64_t>(w.jcp),
                                                 B<int>(w.jperm), B<int>(w.jrow), in.jv_data, in.jv_indptr,
                                                 in.jv_indices, neg_kv, in.k_v, B<int64_t>(w.ccnt), nullptr, nullptr,
                                                 nullptr);
  AK(cudaMemsetAsync(B<int64_t>(w.ccnt) + n, 0, sizeof(int64_t), st));
  tb = 0;
  AK(cub::DeviceScan::ExclusiveSum(nullptr, tb, B<int64_t>(w.ccnt), B<int64_t>(w.cptr), n + 1, st));
  AK(ensure(w.tmp, tb));
  AK(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, B<int64_t>(w.ccnt), B<int64_t>(w.cptr), n + 1, st));
  AK(cudaMemcpyAsync(w.h_small, B<int64_t>(w.cptr) + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  AK(cudaStreamSynchronize(st));
  const int64_t nnz = w.h_small[0];
  if (nnz > INT32_MAX) {
    err = "augment: output exceeds 2^31 entries";
    return VFPI_UNSUPPORTED;
  }
  AK(ensure(w.out_p, sizeof(int) * (size_t)(n + 1)));
  AK(ensure(w.out_i, sizeof(int) * (size_t)std::max<int64_t>(nnz, 1)));
  AK(ensure(w.out_x, sizeof(double) * (size_t)std::max<int64_t>(nnz, 1)));
  k_aug_merge<true><<<grid_for(n), kT, 0, st>>>(n_o, rows, in.a_indptr, in.a_indices, in.a_data, B<int64_t>(w.cs),
                                                B<int>(w.t_row), B<double>(w.t_val), B<int64_t>(w.jcp),
                                                B<int>(w.jperm), B<int>(w.jrow), in.jv_data, in.jv_indptr,
                                                in.jv_indices, neg_kv, in.k_v, nullptr, B<int64_t>(w.cptr),
                                                B<int>(w.out_i), B<double>(w.out_x));
  k_aug_to_i32<<<grid_for(n + 1), kT, 0, st>>>(n + 1, B<int64_t>(w.cptr), B<int>(w.out_p));
  launches += 7;
  AK(cudaGetLastError());
  out.nnz = nnz;
  out.indptr = B<int>(w.out_p);
  out.indices = B<int>(w.out_i);
  out.data = B<double>(w.out_x);
  return VFPI_OK;
}

}  // namespace vfpi
