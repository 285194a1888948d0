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
constexpr unsigned kSecIdMask = 0x3fffffffu;  // staged-sector entries: id | half marks << 30

// Shared-memory layout of one CTA of the resident iteration kernel: EP SELL-32
// elements (values + gather map) of its R rows (the first CR belong to its C
// contacts) and NS staged 32-byte sectors of remote v, followed directly by the
// CTA's own rows of v^(l-1): one x array, indexed by the gather map.
struct ResLayout {
  size_t o_sv, o_map, o_xs, o_sec, o_sb, o_len, o_row, o_b, o_w, o_v0, o_v1, o_cm, o_cq, o_fr, o_par, o_lam, o_vs,
      o_jt, total;
  __host__ __device__ ResLayout(int64_t EP, int R, int C, int CR, int NS) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
      const size_t r = o;
      o += (bytes + 15) & ~size_t(15);
      return r;
    };
    const int NSL = (R + 31) / 32;
    o_sv = take(8 * (size_t)EP);
    o_map = take(4 * (size_t)EP);
    o_xs = take(32 * (size_t)NS + 8 * (size_t)R);  // staged sectors, then own rows of v^(l-1)
    o_v0 = o_xs + 32 * (size_t)NS;
    o_sec = take(4 * (size_t)NS);
    o_sb = take(4 * (size_t)(NSL + 1));
    o_len = take(4 * (size_t)R);
    o_row = take(4 * (size_t)R);
    o_b = take(8 * (size_t)R);
    o_w = take(8 * (size_t)R);
    o_v1 = take(8 * (size_t)R);    // own rows of v^(l)
    o_cm = take(4 * (size_t)C);
    o_cq = take(4 * (size_t)C);
    o_fr = take(72 * (size_t)C);
    o_par = take(32 * (size_t)C);
    o_lam = take(48 * (size_t)C);  // two parities
    o_vs = take(8 * (size_t)CR);   // v* of contact rows
    o_jt = take(8 * (size_t)CR);   // J_c^T lam of contact rows
    total = o;
  }
};

// Device-side summary written at the end of layout setup (one D2H read).
struct SetupSummary {
  int64_t nnz_num;          // numeric (non-zero) entries of A
  int64_t sell_elems;       // padded SELL-32 element count
  int64_t max_ent_per_blk;  // numeric entries of the largest CTA partition
  int64_t max_res_bytes;    // largest per-CTA ResLayout footprint
  int32_t n_slices;
  int32_t max_ct_per_blk;
  int32_t max_rows_per_blk;
  int32_t flags;            // bit0 overlap, bit1 bad column index
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
  const int64_t* pos_ptr;   // [n+1] entry offset of every row-list position (resident kernel)
  const unsigned* sell_map; // [sell_elems] gather map of every SELL element (resident kernel)
  const unsigned* secs;     // [sum NS] 32-byte sectors of v each CTA stages per iteration
  const int* sec_ptr;       // [G+1] per-CTA range in secs
  const int* blk_cr;        // [G+1] contact rows at the head of every CTA range
  const int* cont_q;        // [n_c] rank of a two-sided contact among its CTA's (row a of side j: 3C + a*CD + rank)
  int* bar_flags;           // [G] epoch flags of the flag barrier
  long long* prof;          // optional [G][4][8] phase timestamps (NULL = off)
  const double* diag;       // [n] diagonal of A (per-scene fixed-alpha default)
  int fixed_alpha_default;  // fixed-alpha strategy with fixed_alpha = None
  size_t trace_stride;      // scene batches: residual_trace row stride per scene
  int prof_iter0;           // first of the 4 profiled iterations
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

// Layout setup on the stream: statistics, contact-aware CTA partition and
// sizes (ends with one host read of the summary). Returns VFPI_* code.
struct LayoutOptions {
  bool anchor_order = true;   // order units by their smallest referenced column
  bool length_sort = true;    // free rows of a CTA by decreasing length
  int entry_cost = 24, row_cost = 40, contact_cost = 0;  // partition cost model
  int res_row_cost = 20;  // row cost of the shared-memory-resident attempt (configs[1]: best of 0-80)
  // scene batches: CTA b = scene b (device arrays, G+1 entries each); contacts
  // must be grouped by scene and never couple two scenes
  const int* scene_row_ptr = nullptr;
  const int* scene_ct_ptr = nullptr;
};
// setup_layout = setup_layout_async (kernels only, capturable into a graph) +
// setup_layout_finish (the one host read of the summary, input checks)
int setup_layout_async(Workspace& ws, const vfpi_system& dsys, int G, cudaStream_t st, std::string& err,
                       int64_t& launches, const LayoutOptions& opt);
int setup_layout_finish(Workspace& ws, cudaStream_t st, SetupSummary* host_summary, std::string& err);
inline int setup_layout(Workspace& ws, const vfpi_system& dsys, int G, cudaStream_t st, SetupSummary* host_summary,
                        std::string& err, int64_t& launches, const LayoutOptions& opt = LayoutOptions()) {
  const int rc = setup_layout_async(ws, dsys, G, st, err, launches, opt);
  return rc ? rc : setup_layout_finish(ws, st, host_summary, err);
}
// generation counter of workspace (re)allocations (captured setup graphs key on it)
uint64_t alloc_generation();
// Row-sorted entries packed for the chosen iteration kernel:
// resident = CTA-contiguous CSR (pos_ptr/pk_val/pk_col), else SELL-32.
int setup_pack(Workspace& ws, const vfpi_system& dsys, int G, bool resident, const SetupSummary& hs,
               cudaStream_t st, std::string& err, int64_t& launches);
// d_nc != nullptr: dsys.n_c is an upper bound and *d_nc (device) the contact count
int setup_step_matrix(Workspace& ws, const vfpi_system& dsys, const vfpi_config& cfg, const double* d_w_cached,
                      cudaStream_t st, std::string& err, int64_t& launches, const int* d_nc = nullptr);

// ---- iteration (vfpi_solve.cu) ---------------------------------------------
int launch_iterate(const IterParams& p, int op, bool cheb, bool bb, int smem_bytes, cudaStream_t st,
                   std::string& err);
int iterate_max_blocks_per_sm(int op, bool cheb, bool bb, int smem_bytes, bool scenes = false);
// shared-memory resident variant (whole CTA partition of A on chip)
int launch_iterate_resident(const IterParams& p, int op, bool cheb, bool bb, size_t smem_bytes, cudaStream_t st,
                            std::string& err);
#ifndef VFPI_RES_THREADS
#define VFPI_RES_THREADS 480  // 15 warps: measured best of 384-1024 with the 8-deep free-row sums
#endif
constexpr int kResThreads = VFPI_RES_THREADS;
int launch_scc_final(const IterParams& p, double* scc, cudaStream_t st);
// independent scenes, one CTA each (layout with one CTA range per scene)
int launch_iterate_scenes(const IterParams& p, int op, bool cheb, bool bb, int smem_bytes, cudaStream_t st,
                          std::string& err);

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
  uint64_t layout_epoch = 0;  // bumped by every layout/pack (cached layouts compare against it)
  std::vector<void*> owned;
  // grow-only buffers
  struct Buf { void* p = nullptr; size_t cap = 0; };
  Buf b_indptr, b_indices, b_data, b_b, b_ci, b_cj, b_frames, b_mu, b_mu2, b_phi, b_warm, b_wc;
  Buf b_out_v, b_out_lam, b_trace, b_scc, b_w_out;
  Buf diag, rns, w, gamma, w_mean;
  Buf rowcnt, row_ptr, keys, keys_sorted, vals, perm, colof, mark;
  Buf ucost, cpos, urows, rpos, ucont, kpos;
  Buf blk_row, blk_ct, blk_slice, row_list, row_slot, cont_list;
  Buf slice_w, slice_off, sell_val, sell_col, pos_len, pos_ptr, pk_val, pk_col, bar_flags;
  Buf ucr, ufr, cposc, cposf, blk_first, blk_cr, cont_q, ps_col, ps_src, seg_beg, seg_end, rowpos;
  Buf sec_key, sec_skey, sec_idx, sec_sidx, sec_flag, sec_upos, sell_map, secs, sec_ptr;
  Buf rowmin, ukey, ukey_s, uval, uorder, row_list2, row_slot2, rowblk, scene_rows, scene_cts;
  Buf vbuf, lambuf, partials, status, summary, flags, cub_tmp;
  Buf x, y;  // scratch for per-op entry points
  Buf cg_vec, cg_part;  // contact-free CG fallback (vfpi_cg_device)
  Buf prof;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // host-buffer solves: the inputs the layout setup does not read (b, frames,
  // mu, mu2, phi, warm) are uploaded on a side stream while the setup runs
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main_h2d = nullptr, ev_side = nullptr;
  bool side_pending = false;
  SetupSummary* h_summary = nullptr;  // pinned
  SolveStatus* h_status = nullptr;    // pinned
  int num_sms = 148;
  int max_smem_optin = 232448;
  bool unit_order_is_sorted = false;
};

cudaError_t ensure(Workspace::Buf& b, size_t bytes);
// the library's device memory cache (vfpi_setup.cu): every Workspace::Buf is
// allocated and released through these
cudaError_t dev_alloc(void** p, size_t bytes, size_t* got);
void dev_free(void* p);
// Raise a kernel's dynamic shared-memory limit to the device maximum, once per
// kernel, under a lock (the attribute is process-wide; concurrent solves on
// several threads must never shrink it under each other).
cudaError_t ensure_max_dynamic_smem(const void* fn);


// Scene batches whose matrix stays fixed while contacts change (the FEM step
// pipeline): the row layout is built once without contacts (setup_layout +
// setup_pack with n_c = 0, then setup_rowpos); each step only re-marks the
// contact rows (row_slot), the contact list and the CTA contact ranges.
int setup_rowpos(Workspace& ws, int n, int G, cudaStream_t st, std::string& err);
int setup_contacts_refresh(Workspace& ws, const vfpi_system& dsys, int G, const int* d_scene_ct_ptr, cudaStream_t st,
                           std::string& err, int64_t& launches);

// ---- virtual-node augmentation (vfpi_augment.cu) ----------------------------
struct AugmentIn {
  int n_o = 0, n_v3 = 0;  // original dimension, rows of J_v (3 per virtual node)
  int64_t a_nnz = 0, jv_nnz = 0;
  const int* a_indptr = nullptr;   // CSC of A_o (device), canonical
  const int* a_indices = nullptr;
  const double* a_data = nullptr;
  const int* jv_indptr = nullptr;  // CSR of J_v (device), canonical
  const int* jv_indices = nullptr;
  const double* jv_data = nullptr;
  double k_v = 0.0;
};
struct AugmentOut {
  int n = 0;
  int64_t nnz = 0;
  int* indptr = nullptr;  // device, owned by the AugmentWork
  int* indices = nullptr;
  double* data = nullptr;
};
struct AugmentWork {
  Workspace::Buf pcnt, poff, pkey, pkey2, pval, pval2, head, hpos, tmp, tmp2;
  Workspace::Buf jrow, jcol_s, jidx, jperm, jcp, t_row, t_col, t_val, cs, ccnt, cptr;
  Workspace::Buf out_p, out_i, out_x;
  int64_t* h_small = nullptr;  // pinned [2]
};
int augment_device(AugmentWork& w, const AugmentIn& in, cudaStream_t st, AugmentOut& out, std::string& err,
                   int64_t& launches);

// ---- cube-pile contacts (vfpi_pile.cu) ---------------------------------------
struct PileGeometry {
  int64_t nodes = 0, n_surf = 0, n_tris = 0;
  int n_o = 0;                   // 3 * nodes
  const int* surf = nullptr;     // [n_surf] ascending
  const int* tris = nullptr;     // [n_tris*3] outward
  const int* node_body = nullptr;
  const int* tri_body = nullptr;
  double reach = 0, cell = 0, neg_half_h = 0, margin = 0;
  double mu = 0, neg_beta_dt = 0, e_rest = 0, rest_threshold = 0;
};
struct PileContactsOut {
  int n_ground = 0, n_face = 0, n_virtual = 0, jv_nnz = 0;
  int* col_i = nullptr;
  int* col_j = nullptr;
  double* frames = nullptr;
  double* mu = nullptr;
  double* phi = nullptr;
  int* jv_indptr = nullptr;
  int* jv_indices = nullptr;
  double* jv_data = nullptr;
};
struct PileWork {
  Workspace::Buf tcnt, toff, flag, key, key2, own, own2, btri, best, gflag, gpos, fflag, fpos, nvirt, vpos, njv,
      jpos, ci, cj, fr, mu, phi, jrp, jci, jcx, tmp;
  int64_t* h_small = nullptr;  // pinned [4]
};
int pile_contacts_device(PileWork& w, const PileGeometry& g, const double* x, const double* v, cudaStream_t st,
                         PileContactsOut& out, std::string& err, int64_t& launches);

// ---- nodalization (vfpi_nodalize.cu) -----------------------------------------
struct NodalizeIn {
  int64_t n_c = 0;
  int n_o = 0;  // velocity dimension
  int n_bodies = 0;
  int64_t n_q = 0;                   // entries of q
  const int* first_kind = nullptr;   // 0 node (ref = velocity offset), 1 rigid (ref = body)
  const int* first_ref = nullptr;
  const int* second_kind = nullptr;  // -1 static, 0 node, 1 rigid
  const int* second_ref = nullptr;
  const double* point = nullptr;     // [n_c*3]
  const double* normal = nullptr;    // [n_c*3]
  const double* depth = nullptr;     // [n_c]
  const double* q = nullptr;         // generalized coordinates
  const double* v = nullptr;         // velocities [n_o]
  const int* body_q = nullptr;       // per body: coordinate offset
  const int* body_v = nullptr;       // per body: velocity offset
  double mu = 0, mu2 = 0, neg_beta_dt = 0, e_rest = 0, rest_threshold = 0;
};
struct NodalizeOut {
  int n_virtual = 0, jv_nnz = 0;
  int* col_i = nullptr;
  int* col_j = nullptr;
  double* frames = nullptr;
  double* phi = nullptr;
  double* mu = nullptr;
  double* mu2 = nullptr;
  int* jv_indptr = nullptr;
  int* jv_indices = nullptr;
  double* jv_data = nullptr;
};
struct NodalizeWork {
  Workspace::Buf first, vflag, vpos, jcnt, jpos, flag, tmp, ci, cj, fr, phi, mu, mu2, jrp, jci, jcx;
  int64_t* h_small = nullptr;  // pinned [2]
};
int nodalize_device(NodalizeWork& w, const NodalizeIn& in, cudaStream_t st, NodalizeOut& out, std::string& err,
                    int64_t& launches);

// ---- FEM scene-batch step pipeline (vfpi_fem.cu) ----------------------------
void launch_fem_rhs(int64_t n, const int64_t* krp, const int* kc, const double* kv, const double* x, const double* X,
                    const double* v, const double* m, const double* g, double twodt, double* b, cudaStream_t st);
void launch_fem_sell_width(int64_t n, const int64_t* krp, int64_t* width, cudaStream_t st);
void launch_fem_sell_pack(int64_t n, const int64_t* krp, const int* kc, const double* kv, const int64_t* off,
                          double* sv, int* sc, cudaStream_t st);
void launch_fem_rhs_sell(int64_t n, const int64_t* off, const double* sv, const int* sc, const double* x,
                         const double* X, const double* v, const double* m, const double* g, double twodt, double* b,
                         cudaStream_t st);
// node-plane detection of a FEM batch: scan of the below-margin predicate
// (cub, 2 launches) + one pass writing scene pointers and contact parameters
size_t fem_detect_tmp_bytes(int64_t nodes);
int launch_fem_detect(int64_t nodes, int S, int nodes_per_scene, const double* x, const double* v, double margin,
                      void* tmp, size_t tmp_bytes, int* pos, int* cts, const double* frame, double mu,
                      double neg_beta_dt, double e_rest, double thr, int* ci, int* cj, double* frames, double* muv,
                      double* mu2v, double* phi, double* lam0, double* lam1, cudaStream_t st);
void launch_fem_advance(int64_t n, double dt, const double* vh, double* x, double* v, double* warm, cudaStream_t st);
void launch_csr_matvec(int64_t rows, const int* rp, const int* ci, const double* cx, const double* x, double* y,
                       cudaStream_t st);
void launch_fem_run_stats(int S, const SolveStatus* st, const int* cts, int step, unsigned long long* acc,
                          int* its_out, int* cts_out, cudaStream_t stream, int* perm = nullptr);
void launch_iota_int(int n, int* v, cudaStream_t st);

// ---- configs[3] heightfield detection (vfpi_heightfield.cu) -----------------
struct HfParams {
  double amp, freq, slope, margin, mu, neg_beta_dt;
};
struct HfContactsOut {
  int64_t n_c = 0;
  int* col_i = nullptr;
  int* col_j = nullptr;
  double* frames = nullptr;
  double* mu = nullptr;
  double* phi = nullptr;
};
struct HfWork {
  Workspace::Buf flag, pos, tmp, ci, cj, fr, mu, phi;
  int64_t* h_small = nullptr;  // pinned [2]
};
int heightfield_contacts_device(HfWork& w, const HfParams& p, int64_t N, const double* x, cudaStream_t st,
                                HfContactsOut& out, std::string& err, int64_t& launches);
void launch_add_inplace(int64_t n, const double* f, double* b, cudaStream_t st);

// ---- contact-free CG fallback of a diverged solve (vfpi_cg.cu) --------------
int launch_cg_scenes(int num, const int32_t* scene_list, int64_t rows_per_scene, const int32_t* indptr,
                     const int32_t* indices, const double* data, const double* b, double* x, double* r, double* p,
                     double* q, double rtol, int64_t maxiter, int32_t* iters_out, cudaStream_t st);
// device-driven variant: CTA b steps scene b iff status[b].diverged (no host round trip)
int launch_cg_scenes_status(int S, int64_t rows_per_scene, const int32_t* indptr, const int32_t* indices,
                            const double* data, const double* b, double* x, double* r, double* p, double* q,
                            double rtol, int64_t maxiter, const SolveStatus* status, const int* cts, double* lam,
                            cudaStream_t st);
int cg_grid_partials(int device);
// scene batches: perm = scenes by decreasing iteration count of their last
// solve (ties by index), so the CTAs the block scheduler dispatches first run
// the scenes predicted to take longest (counts change by < 1 per step)
void launch_scene_order(int S, const SolveStatus* st, int* perm, cudaStream_t stream);
constexpr int kMaxOrderedScenes = 2048;

int launch_cg_grid(int G, int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                   const double* b, double* x, double* r, double* p, double* q, double* partial, double rtol,
                   int64_t maxiter, int32_t* iters_out, cudaStream_t st);

// ---- node-block SELL scene kernel (vfpi_nodes.cu; FEM batches) ---------------
struct NodeLayoutDev {
  int nn = 0, nsl = 0;                 // nodes and node slices (per scene for batches, of the system for grids)
  const int* blk_slice = nullptr;      // [G+1] node slices of every CTA
  const int* blk_pos = nullptr;        // [G+1] node positions of every CTA
  int cluster = 1;                     // scene batches: CTAs per scene (thread-block cluster) when > 1
  int has_d = 1;                       // any two-node contact (else no contact phase / barrier)
  double* vs_g = nullptr;              // grid / cluster mode: v* of contact rows [6 n_c]
  double* jt_g = nullptr;              // grid mode: J_c^T lam of contact rows [6 n_c]
  const int* node_list = nullptr;      // [S*nn] position -> global node
  int* node_slot = nullptr;            // [S*nn] global node -> contact slot base (6 per contact) or -1
  const int64_t* slice_off = nullptr;  // [S*nsl+1] k-step offset of every slice
  const unsigned* desc = nullptr;      // [k][lane]: block column | mask << 23
  const double* val = nullptr;         // [k][9][lane]
  const int* scene_perm = nullptr;     // scene batches: CTA (cluster) c runs scene scene_perm[c] (longest first)
  const int64_t* voff = nullptr;       // packed values (single systems): [k] first value slot of k-step k, [K] total
  // FEM batches: the template's block columns [k_scene][32] (-1 = padding); the
  // kernel takes block columns from here instead of streaming descriptors
  // (absent entries are stored as +0 and added: bit-neutral, see vfpi_nodes.cu)
  const int* tcol = nullptr;
  int64_t k_scene = 0;
};
struct NodeLayoutHost {
  int nn = 0, nsl = 0;
  int64_t k_scene = 0;                 // k-steps per scene
  Workspace::Buf t_order, t_off, t_bcol, desc, val, slice_off, node_list, node_slot, blk_slice, blk_pos, vs, jt, perm;
  std::vector<int64_t> t_off_host;
};
struct NodeGridWork {  // single-system node-block layout (rebuilt per solve)
  Workspace::Buf blk_pos, blk_slice, key, key2, val_i, node_list, cnt, node_slot, width, slice_off, flags, vs, jt,
      tmp, desc, val, wt, wpre, hsh, ek, voff, tot;
  int64_t* h_small = nullptr;  // pinned [2]
  std::vector<int> h_bpos;     // CTA split points of the last build
  bool packed = false;         // the last build packed its block values
  int64_t k_total = 0;
};
int node_grid_build(NodeGridWork& w, const vfpi_system& d, int G, const int64_t* row_ptr, const int* rowcnt,
                    const int* perm, const int* colof, cudaStream_t st, NodeLayoutDev& out, std::string& err,
                    int64_t& launches, int contact_cost = 8, int pack_mode = 2);
int node_layout_build(NodeLayoutHost& h, int S, const int* d_a_ptr, const int* d_a_idx, const double* d_a_val,
                      NodeLayoutDev& out, int* d_flags, cudaStream_t st, int cluster,
                      const std::vector<int64_t>& t_off_host);
int node_cluster_size(int S, int nsl, int num_sms);  // CTAs per scene so a small batch fills the GPU
// a second matrix on the same node-block template (FEM batches: K for the
// right-hand side), every stored entry kept (explicit zeros included)
int node_fill_matrix(const NodeLayoutHost& h, int S, const int64_t* d_ptr, const int* d_idx, const double* d_val,
                     Workspace::Buf& desc, Workspace::Buf& val, int* d_flags, cudaStream_t st);
// b = ((2/dt) m) v - K (x - X) + m g with K in the node-block layout
// (slice_off / node_list of the batch's A layout, desc / val of K)
void launch_fem_rhs_nodes(int S, int nn, int nsl, const int64_t* slice_off, const int* node_list,
                          const unsigned* kdesc, const double* kval, const double* x, const double* X,
                          const double* v, const double* m, const double* g, double twodt, double* b,
                          cudaStream_t st);
int node_slots_refresh(const NodeLayoutDev& L, int S, int n_c, const int* ci, const int* cj, const int* d_nc,
                       cudaStream_t st);
int node_kernel_smem(int max_ct, int mode = 0);
// mode: 0 one CTA per scene, 1 one system over a cooperative grid, 2 one cluster per scene
int node_kernel_blocks_per_sm(int op, bool cheb, int max_ct, int mode = 0);
int launch_iterate_nodes(const IterParams& p, const NodeLayoutDev& L, int op, bool cheb, int max_ct, cudaStream_t st,
                         std::string& err, int mode = 0);

}  // namespace vfpi
