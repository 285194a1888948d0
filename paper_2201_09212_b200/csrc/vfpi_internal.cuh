// Internal declarations shared by the V-FPI translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/vfpi.h"

namespace vfpi {

constexpr int kThreads = 256;      // threads per CTA of the iteration kernel
constexpr int kSlotsPerContact = 6;  // rows of a contact unit (3 for S, 6 for D)
constexpr int kPartialStride = 8;  // doubles per CTA per parity in the partials ring

// Device-side summary written at the end of layout setup (one D2H read).
struct SetupSummary {
  int64_t nnz_num;       // numeric (non-zero) entries of A
  int64_t sell_elems;    // padded SELL-32 element count
  int32_t n_slices;
  int32_t max_ct_per_blk;
  int32_t flags;         // bit0 overlap, bit1 bad column index
  int32_t pad;
};

// Device-side status written by the iteration kernel.
struct SolveStatus {
  int32_t iterations;
  int32_t converged;
  int32_t diverged;
  int32_t final_vbuf;
  double consistency;
  int32_t flags;         // bit0 zero row norm, bit1 tie violation
  int32_t pad;
};

// Everything the persistent iteration kernel reads.
struct IterParams {
  int n, n_c, G;
  // block partition of the row list (contacts co-located with their rows)
  const int* row_list;      // [n] position -> global row
  const int* row_slot;      // [n] position -> shared-memory contact slot, -1 = free row
  const int* blk_row;       // [G+1]
  const int* blk_slice;     // [G+1]
  const int* blk_ct;        // [G+1]
  const int64_t* slice_off; // [S+1] element offset of every SELL-32 slice
  const double* sell_val;   // [sell_elems]
  const int* sell_col;      // [sell_elems], -1 = padding
  const int* cont_list;     // [n_c] contact ids in partition order
  // system
  const double* b;
  const double* w;          // [n] step matrix (iteration 1 for BB)
  const double* gamma;      // [n_c]
  const int* col_i;
  const int* col_j;
  const double* frames;     // [n_c*9]
  const double* mu;
  const double* mu2;
  const double* phi;
  const double* w_mean;     // [1] mean(w) = BB fallback alpha (solver.py:381)
  // iterate state
  double* vbuf0;
  double* vbuf1;
  double* vbuf2;
  double* lam0;
  double* lam1;
  double* partials;         // [2][G][kPartialStride]
  double* trace;            // [max_iters]
  SolveStatus* status;
  double* out_v;
  double* out_lam;
  // SolverConfig
  int max_iters, cheby_start, step;
  double tol, under_relax, omega, cfactor;
};

// ---- setup (vfpi_setup.cu) -------------------------------------------------
struct Workspace;  // device buffers owned by a handle

// Layout + step-matrix setup on the handle stream. Returns VFPI_* code.
int setup_layout(Workspace& ws, const vfpi_system& dsys, int G, cudaStream_t st, SetupSummary* host_summary,
                 std::string& err, int64_t& launches);
int setup_step_matrix(Workspace& ws, const vfpi_system& dsys, const vfpi_config& cfg, const double* d_w_cached,
                      cudaStream_t st, std::string& err, int64_t& launches);

// ---- iteration (vfpi_solve.cu) ---------------------------------------------
int launch_iterate(const IterParams& p, int op, bool cheb, bool bb, int smem_bytes, cudaStream_t st,
                   std::string& err);
int iterate_max_blocks_per_sm(int op, bool cheb, bool bb, int smem_bytes);
int launch_scc_final(const IterParams& p, double* scc, cudaStream_t st);

// ---- per-op kernels (vfpi_ops.cu) -----------------------------------------
void launch_apply_jc(int64_t n_c, const int* ci, const int* cj, const double* fr, const double* v, double* eta,
                     cudaStream_t st);
void launch_apply_jc_t(int64_t n, int64_t n_c, const int* ci, const int* cj, const double* fr, const double* lam,
                       double* out, bool overlap, cudaStream_t st);
void launch_oneshot(int64_t n_c, const double* gamma, const double* eta, const double* phi, const double* mu,
                    const double* mu2, int op, double* lam, cudaStream_t st);
void launch_scc(int64_t n_c, const double* vc, const double* lam, const double* phi, const double* mu, double* out,
                cudaStream_t st);
void launch_spmv_csr_rows(int64_t n, const int64_t* row_ptr, const int* perm, const int* colof, const double* data,
                          const double* x, double* y, cudaStream_t st);
void launch_const_fill(double* p, double v, int64_t n, cudaStream_t st);

// ---- device workspace ------------------------------------------------------
struct Workspace {
  int device = 0;
  std::vector<void*> owned;
  // grow-only buffers
  struct Buf { void* p = nullptr; size_t cap = 0; };
  Buf b_indptr, b_indices, b_data, b_b, b_ci, b_cj, b_frames, b_mu, b_mu2, b_phi, b_warm, b_wc;
  Buf b_out_v, b_out_lam, b_trace, b_scc, b_w_out;
  Buf diag, rns, w, gamma, w_mean;
  Buf rowcnt, row_ptr, keys, keys_sorted, vals, perm, colof, mark;
  Buf ucost, cpos, urows, rpos, ucont, kpos;
  Buf blk_row, blk_ct, blk_slice, row_list, row_slot, cont_list;
  Buf slice_w, slice_off, sell_val, sell_col;
  Buf vbuf, lambuf, partials, status, summary, flags, cub_tmp;
  Buf x, y;  // scratch for per-op entry points
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  SetupSummary* h_summary = nullptr;  // pinned
  SolveStatus* h_status = nullptr;    // pinned
  int num_sms = 148;
};

cudaError_t ensure(Workspace::Buf& b, size_t bytes);

}  // namespace vfpi
