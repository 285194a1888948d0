/*
 * vfpi.h — C ABI of the B200-native V-FPI contact solver (libvfpi.so).
 *
 * Drop-in boundary for the reference's hot path
 *   condsim.solver.solve_vfpi(aug, cfg, warm, w_cached=None, project_override=None)
 *   (/root/reference/pkg/src/condsim/solver.py:345-461)
 * and for the per-iteration subsystems it drives (see each entry point).
 *
 * Plain C: pointers and sizes only, fp64 values, int32 indices. All entry
 * points except vfpi_solve_device/vfpi_wait take HOST pointers, copy to the
 * device, compute with the sm_100a kernels, copy back and return when done.
 * A handle is one CUDA stream plus its device workspace; it is not
 * thread-safe — use one handle per calling thread (the reference calls
 * solve_vfpi concurrently from a ThreadPoolExecutor, harness.py:762-767).
 * There is no CPU fallback: without a usable CUDA device every call returns
 * VFPI_CUDA_ERROR.
 */
#ifndef VFPI_H
#define VFPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (errors.py:8-40 taxonomy) */
#define VFPI_OK 0
#define VFPI_DIVERGED 1          /* DivergenceError: non-finite iterate, trace valid (solver.py:424-427) */
#define VFPI_INVALID_MATRIX 2    /* InvalidMatrixError: zero row norm (solver.py:220-221) */
#define VFPI_TIE_VIOLATION 3     /* InvalidMatrixError: broken tie group (solver.py:256-259) */
#define VFPI_DIM_MISMATCH 4      /* DimensionMismatchError (sparse.py:100-101) */
#define VFPI_CUDA_ERROR 5
#define VFPI_UNSUPPORTED 6       /* e.g. two contacts sharing a node column */
#define VFPI_BAD_ARGUMENT 7

/* SolverConfig.operator (solver.py:33) */
#define VFPI_OP_STRICT 0
#define VFPI_OP_PROXIMAL 1
#define VFPI_OP_STRICT_ANISOTROPIC 2
/* SolverConfig.step_strategy (solver.py:34) */
#define VFPI_STEP_FROBENIUS 0
#define VFPI_STEP_BB1 1
#define VFPI_STEP_BB2 2
#define VFPI_STEP_BB_ALTERNATING 3
#define VFPI_STEP_FIXED_ALPHA 4

typedef struct vfpi_handle vfpi_handle;

/* One augmented system = contacts.AugmentedDynamics (contacts.py:118-128). */
typedef struct vfpi_system {
  int64_t n;               /* aug.n: augmented velocity dimension */
  int64_t n_c;             /* number of nodalized contacts */
  int64_t nnz;             /* stored entries of aug.a (CSC, both triangles) */
  const int32_t* indptr;   /* [n+1] SparseSymmetric.indptr  (sparse.py:30-37) */
  const int32_t* indices;  /* [nnz] SparseSymmetric.indices (row of each entry) */
  const double* data;      /* [nnz] SparseSymmetric.data */
  const double* b;         /* [n]   aug.b */
  const int32_t* col_i;    /* [n_c] aug.col_i: first velocity offset of node i */
  const int32_t* col_j;    /* [n_c] aug.col_j: node j offset, -1 for S contacts */
  const double* frames;    /* [n_c*9] aug.frames, row-major rows (n, t1, t2) */
  const double* mu;        /* [n_c] Contact.mu */
  const double* mu2;       /* [n_c] Contact.mu2 (mu when None, solver.py:340) */
  const double* phi;       /* [n_c] Contact.phi_n */
} vfpi_system;

/* SolverConfig (solver.py:50-62). fixed_alpha = NaN means None. */
typedef struct vfpi_config {
  int32_t op;
  int32_t step_strategy;
  int32_t max_iters;
  int32_t chebyshev;
  int32_t cheby_start;
  int32_t reserved;
  double residual_tol;
  double under_relax;
  double omega;
  double fixed_alpha;
  double consistency_factor;
} vfpi_config;

/* Outputs of one solve (the (v, lam, SolverReport) triple, solver.py:65-74). */
typedef struct vfpi_result {
  double* v;               /* [n] out: v_hat */
  double* lam;             /* [n_c*3] out: contact-frame impulses */
  double* residual_trace;  /* [max(max_iters,1)] out: theta per iteration */
  double* scc;             /* [n_c] out or NULL: SolverReport.scc_residuals */
  double* w;               /* [n] out or NULL: the step matrix used */
  int32_t iterations;
  int32_t converged;
  int32_t diverged;
  int32_t status;          /* return code of the solve */
  double consistency;      /* ||A v - b - J_c^T lam|| */
  double setup_ms;         /* device time of W/gamma/layout setup */
  double loop_ms;          /* device time of the iteration kernel */
} vfpi_result;

int vfpi_create(int device, vfpi_handle** out);
void vfpi_destroy(vfpi_handle* h);
const char* vfpi_last_error(const vfpi_handle* h);
int vfpi_version(void);

/* solve_vfpi (solver.py:345-461). warm: [n]. w_cached: [n] or NULL
 * (solver.py:349, 370-371). Host pointers; synchronous. Returns VFPI_OK,
 * VFPI_DIVERGED (res->residual_trace[0..iterations) valid), or an error. */
int vfpi_solve(vfpi_handle* h, const vfpi_system* sys, const vfpi_config* cfg,
               const double* warm, const double* w_cached, vfpi_result* res);

/* Same solve with every pointer in sys/warm/w_cached/res already in device
 * memory; enqueued on `stream` (cudaStream_t, NULL = the handle's stream)
 * without a host synchronisation. vfpi_wait() synchronises and fills the
 * scalar fields of res (iterations, converged, ...). */
int vfpi_solve_device(vfpi_handle* h, const vfpi_system* sys, const vfpi_config* cfg,
                      const double* warm, const double* w_cached, vfpi_result* res, void* stream);
int vfpi_wait(vfpi_handle* h, vfpi_result* res);

/* Per-scene outputs of a scene batch. Arrays are concatenated in scene order:
 * v [sum n_s], lam [3 * sum n_c_s], scc [sum n_c_s] (or NULL), residual_trace
 * [num_scenes * max(max_iters,1)] (row s = scene s), and one entry per scene in
 * iterations / converged / diverged / consistency. */
typedef struct vfpi_scene_result {
  double* v;
  double* lam;
  double* residual_trace;
  double* scc;
  int32_t* iterations;
  int32_t* converged;
  int32_t* diverged;
  double* consistency;
  double setup_ms;
  double loop_ms;
} vfpi_scene_result;

/* A batch of independent systems (e.g. configs[2]'s 1024 FEM scenes), solved
 * concurrently with one CTA per scene, each with its own iteration count,
 * convergence test and divergence flag (solve_vfpi semantics per scene).
 * sys holds the block-diagonal concatenation (host pointers); scene_row_ptr
 * [num_scenes+1] and scene_ct_ptr [num_scenes+1] delimit each scene's rows
 * and contacts (contacts grouped by scene, never coupling two scenes).
 * num_scenes <= 1024 per call. A diverged scene does not fail the call. */
int vfpi_solve_scenes(vfpi_handle* h, const vfpi_system* sys, int32_t num_scenes, const int32_t* scene_row_ptr,
                      const int32_t* scene_ct_ptr, const vfpi_config* cfg, const double* warm,
                      const double* w_cached, vfpi_scene_result* res);

/* ---- FEM scene batch stepped on the device (configs[0]/[2]) ---------------
 * SURVEY §8(f) item 1; reference analogues harness.run (harness.py:526-619),
 * assemble_step (dynamics.py:176-218, here the linear-FEM right-hand side
 * b = (2/dt) M v - K (x - X) + M g), detect_contacts node-plane branch
 * (contacts.py:159-200), stabilization_term (contacts.py:230-239) and
 * integrate (dynamics.py:237-255). The batch keeps A (block diagonal, CSC),
 * K (block diagonal, CSR, for b) and the state x, v on the device; each
 * vfpi_fem_step assembles b, detects node-plane contacts (z < margin, frame
 * `frame9` for every contact), solves all scenes with vfpi_solve_scenes
 * semantics (warm start = the previous step's solution) and integrates.
 * A scene whose solve diverges takes the reference's flagged contact-free
 * step instead (harness.py:586-593): v_hat = CG(A, b, rtol 1e-10, maxiter
 * 10 n) of that scene on the device, lam = 0; it is counted in
 * diverged_scenes (the harness's any_diverged).
 * The handle is borrowed and must outlive the batch. */
typedef struct vfpi_fem_batch vfpi_fem_batch;
typedef struct vfpi_fem_params {
  double dt, margin, beta_err, e_rest, rest_threshold, mu;
} vfpi_fem_params;
typedef struct vfpi_fem_step_stats {
  int64_t contacts;            /* contacts of the step, all scenes */
  int64_t contact_iterations;  /* sum over scenes of n_c(scene) * iterations(scene) */
  int64_t iterations;          /* sum over scenes */
  int32_t max_iterations;
  int32_t diverged_scenes;
  double setup_ms, loop_ms, step_ms;  /* solve setup, iteration kernel, whole step (device events) */
} vfpi_fem_step_stats;
int vfpi_fem_create(vfpi_handle* h, int32_t num_scenes, int32_t nodes_per_scene, const vfpi_system* a_batch,
                    const int64_t* k_rowptr, const int32_t* k_cols, const double* k_vals, const double* mass,
                    const double* gravity, const double* rest_x, const double* x, const double* v,
                    const double* frame9, const vfpi_fem_params* params, vfpi_fem_batch** out);
int vfpi_fem_step(vfpi_fem_batch* fb, const vfpi_config* cfg, vfpi_fem_step_stats* stats,
                  int32_t* iterations_per_scene /* optional [num_scenes] */);
int vfpi_fem_state(vfpi_fem_batch* fb, double* x, double* v);
/* `steps` steps of every scene without a host round trip per step: contact
 * counts, W / gamma sizes, the diverged-scene fallback and the counters stay
 * on the device (one synchronisation at the end), so the steps run back to
 * back on the handle's stream. Same results as `steps` calls of vfpi_fem_step.
 * Needs the node layout (vfpi_fem_set_node_layout) and a non-BB step; falls
 * back to vfpi_fem_step per step otherwise (host_synced = 1). Optional
 * outputs: iterations [steps][num_scenes], contacts [steps]. */
typedef struct vfpi_fem_run_stats {
  int64_t contacts;            /* sum over steps of the step's contacts */
  int64_t contact_iterations;  /* sum over steps and scenes of n_c(scene) * iterations(scene) */
  int64_t iterations;          /* sum over steps and scenes */
  int32_t max_iterations;
  int32_t diverged_scene_steps;
  double loop_ms;              /* summed iteration-kernel time (device events) */
  double run_ms;               /* the whole run (device events) */
  int32_t host_synced;
  int32_t reserved;
} vfpi_fem_run_stats;
int vfpi_fem_run(vfpi_fem_batch* fb, const vfpi_config* cfg, int32_t steps, vfpi_fem_run_stats* stats,
                 int32_t* iterations, int32_t* contacts);
/* Node-block SELL layout for the batch's iteration kernel (csrc/vfpi_nodes.cu):
 * one lane per node, 3x3 blocks (descriptor + 9 values) instead of entries,
 * the same template for every scene: `order` (nodes_per_scene) = node
 * positions (32 per slice), `slice_off` (n_slices + 1, n_slices =
 * ceil(nodes/32)) = k-step offsets, `block_cols` (32 * slice_off[n_slices])
 * = [k][lane] block column of the lane's k-th block (ascending per node),
 * -1 = padding. A must be symmetric with every stored entry inside the
 * template (VFPI_UNSUPPORTED otherwise). Later steps then use the node-block
 * kernel (identical v and lam; not for Barzilai-Borwein steps). */
int vfpi_fem_set_node_layout(vfpi_fem_batch* fb, int32_t nodes_per_scene, const int32_t* order, int32_t n_slices,
                             const int64_t* slice_off, const int32_t* block_cols);
/* The node layout the batch's iteration kernel streams: CTAs per scene
 * (thread-block cluster size) and the bytes one V-FPI iteration of one scene
 * moves from memory (block values, descriptors where streamed, and the row
 * operands b, w, v^(l-1), v^(l)); VFPI_UNSUPPORTED before
 * vfpi_fem_set_node_layout succeeded. */
int vfpi_fem_layout_info(vfpi_fem_batch* fb, int32_t* cluster, int64_t* bytes_per_scene_iteration);
/* Restore the state the batch was created with (x, v; zero warm start),
 * enqueued on the handle's stream: device-to-device, no host traffic. */
int vfpi_fem_reset(vfpi_fem_batch* fb);
/* Device pointers of the batch state x, v (n doubles each, scene-major),
 * valid until vfpi_fem_destroy; ordered after work on the handle's stream. */
int vfpi_fem_state_device(vfpi_fem_batch* fb, const double** x, const double** v);
void vfpi_fem_destroy(vfpi_fem_batch* fb);

/* ---- configs[3] heightfield step pieces (device pointers, on `stream`) ----
 * Node-vs-heightfield detection for z = amp sin(freq x) sin(freq y), the
 * detect_contacts (contacts.py:159-227) + nodalize (contacts.py:271-321)
 * contract for a surface the reference does not have: every node with
 * z < h + margin is an S-contact on its own node (col_i = 3 node, col_j = -1),
 * in node order; phi = neg_beta_dt * max(0, h - z); frame
 * contact_frame((-hx, -hy, 1)/norm) with hx = slope cos(freq x) sin(freq y),
 * hy = slope sin(freq x) cos(freq y). x: 3*nodes device doubles. Outputs are
 * handle-owned device buffers valid until the next call; one host read. */
typedef struct vfpi_heightfield_params {
  double amp, freq, slope, margin, mu, neg_beta_dt;
} vfpi_heightfield_params;
typedef struct vfpi_heightfield_contacts {
  int64_t n_c;
  int32_t* col_i;
  int32_t* col_j;
  double* frames;
  double* mu;
  double* phi;
} vfpi_heightfield_contacts;
int vfpi_heightfield_contacts_device(vfpi_handle* h, const vfpi_heightfield_params* p, int64_t nodes,
                                     const double* x, vfpi_heightfield_contacts* out, void* stream);
/* b[i] += f[i] (the external load term of the right-hand side). */
int vfpi_add_device(vfpi_handle* h, int64_t n, const double* f, double* b, void* stream);

/* Contact-free fallback step of a diverged solve (harness.py:586-593):
 * x = CG(A, b, rtol, maxiter) from x0 = 0 with scipy.sparse.linalg.cg's
 * recurrence, on device CSC arrays of the contact-free n x n system (read as
 * rows), one cooperative grid, enqueued on `stream` (NULL = handle stream);
 * returns after the solve with the iteration count in *iterations. */
int vfpi_cg_device(vfpi_handle* h, int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                   const double* b, double* x, double rtol, int64_t maxiter, int32_t* iterations, void* stream);

/* The handle's own CUDA stream (cudaStream_t): calls that take NULL for
 * `stream`, and the FEM batch pipeline, enqueue their kernels here, so callers
 * can time them with events recorded on it. */
void* vfpi_stream(vfpi_handle* h);

/* Number of kernels this library launched on the handle since creation. */
int64_t vfpi_launch_count(const vfpi_handle* h);
/* Layout chosen by the last solve: shared-memory resident kernel (1) or the
 * streaming SELL-32 kernel (0), and the number of CTAs. */
int vfpi_last_layout(const vfpi_handle* h, int* resident, int* ctas);
/* Kernel selection for later solves on h: 0 auto (resident when the largest
 * CTA partition fits in shared memory), 1 force resident, 2 force streaming. */
int vfpi_set_kernel(vfpi_handle* h, int mode);
/* Tuning aid: when iter0 > 0, later resident solves record per-CTA phase
 * timestamps of iterations iter0..iter0+3 ([G][4][8] int64: clock64 at
 * phase starts 0..5, globaltimer at 7); vfpi_get_profile copies them out. */
int vfpi_set_profile(vfpi_handle* h, int iter0);
int vfpi_get_profile(vfpi_handle* h, long long* out, int64_t max_count);
/* Tuning knobs. key 1: order units by their smallest referenced column (default 1; 0 = row order);
 * key 2: sort each CTA's free rows by decreasing length (default 1);
 * keys 3/4/5: partition cost per entry / row / contact (defaults 24 / 40 / 0; the
 * shared-memory-resident layout uses row cost 20 unless key 4 sets both);
 * key 6: FEM batches use the node-block kernel when a node layout is set
 * (default 1); key 7 (query, value ignored): 1 if the last scene-batch solve
 * ran the node-block kernel; key 8: small FEM batches run one thread-block cluster
 * per scene (default 1); key 9: force the CTAs per scene (1/2/4/8, 0 = automatic) of FEM
 * batches created afterwards; key 11: partition weight of a single-node contact, in
 * node blocks, when a single system is split over the grid (default 8); key 12: packed
 * block values for single systems whose blocks store <= 7 of 9 entries on average
 * (0 off, 1 on, 2 on + nodes grouped by block-mask sequence, 3 always -- tests; default 2);
 * key 13 (query):
 * 1 if the last single-system grid layout packed its block values. */
int vfpi_set_tuning(vfpi_handle* h, int key, int value);

/* Pinned host memory helpers (cudaMallocHost) for fast host<->device copies. */
void* vfpi_host_alloc(int64_t bytes);
void vfpi_host_free(void* p);

/* ---- per-subsystem entry points (host pointers, synchronous) ---------- */
/* spmv (sparse.py:97-102): y = A x over the CSC arrays of sys */
int vfpi_spmv(vfpi_handle* h, const vfpi_system* sys, const double* x, double* y);
/* row_norms_sq (sparse.py:105-108) and SparseSymmetric.diagonal (:67-68) */
int vfpi_row_norms_sq(vfpi_handle* h, const vfpi_system* sys, double* out);
int vfpi_diagonal(vfpi_handle* h, const vfpi_system* sys, double* out);
/* step_matrix_frobenius (solver.py:216-229); tie groups from sys contacts */
int vfpi_step_matrix_frobenius(vfpi_handle* h, const vfpi_system* sys, int pair_tie, double* w);
/* surrogate_gamma (solver.py:244-253) */
int vfpi_surrogate_gamma(vfpi_handle* h, const vfpi_system* sys, const double* w, double omega, double* gamma);
/* apply_jc (contacts.py:402-411): eta [n_c*3] */
int vfpi_apply_jc(vfpi_handle* h, const vfpi_system* sys, const double* v, double* eta);
/* apply_jc_t (contacts.py:414-423): out [n] */
int vfpi_apply_jc_t(vfpi_handle* h, const vfpi_system* sys, const double* lam, double* out);
/* contact_solve_oneshot (solver.py:262-281): lam [n_c*3] */
int vfpi_contact_solve_oneshot(vfpi_handle* h, int64_t n_c, const double* gamma, const double* eta,
                               const double* phi, const double* mu, const double* mu2, int op, double* lam);
/* scc_residual (solver.py:304-334) */
int vfpi_scc_residual(vfpi_handle* h, int64_t n_c, const double* vc, const double* lam,
                      const double* phi, const double* mu, double* out);
/* inverse_contact (solver.py:468-475) */
int vfpi_inverse_contact(vfpi_handle* h, const vfpi_system* sys, const double* v, double omega, int op,
                         double* lam);

/* ---- virtual-node augmentation ------------------ */
/* Replaces condsim.contacts.augment_dynamics (contacts.py:343-375):
 *   A = [[A_o + k_v J_v^T J_v, -k_v J_v^T], [-k_v J_v, k_v I]]
 * with the reference's exact scipy arithmetic and stored-entry rules
 * (zero sums of J_v^T J_v and zero results of the top-left sum are not
 * stored; J_v's stored entries, explicit zeros included, are kept in the
 * off-diagonal blocks; no virtual node = A_o unchanged), so the output CSC
 * equals SparseSymmetric.from_scipy(...) of the reference bit for bit.
 * b of the augmented system is [b_o; 0] (the caller appends the zeros).
 * A_o: canonical CSC (sorted rows, no duplicates), n_o x n_o.
 * J_v: canonical CSR, n_v3 x n_o (n_v3 = 3 * NodalContactSet.n_virtual),
 *      as nodalize builds it (contacts.py:311-320). */
typedef struct vfpi_augment_input {
  int64_t n_o;
  int64_t n_v3;
  int64_t a_nnz;
  const int32_t* a_indptr;
  const int32_t* a_indices;
  const double* a_data;
  int64_t jv_nnz;
  const int32_t* jv_indptr;
  const int32_t* jv_indices;
  const double* jv_data;
  double k_v;
} vfpi_augment_input;

typedef struct vfpi_augmented {
  int64_t n;          /* n_o + n_v3 */
  int64_t nnz;        /* stored entries */
  int32_t* indptr;    /* [n+1] */
  int32_t* indices;   /* [nnz] */
  double* data;       /* [nnz] */
} vfpi_augmented;

/* Device pointers in; out->indptr/indices/data point at device buffers owned
 * by the handle, valid until the next augmentation call on it or
 * vfpi_destroy. Enqueued on `stream` (NULL = handle stream); returns after
 * the output size is known (two small host reads). */
int vfpi_augment_device(vfpi_handle* h, const vfpi_augment_input* in, vfpi_augmented* out, void* stream);
/* Host pointers in and out (synchronous). out->indptr/indices/data are
 * caller buffers; out->nnz holds their capacity on entry (an upper bound is
 * a_nnz + sum over J_v rows of nonzeros^2 + 2 jv_nnz + n_v3) and the stored
 * entry count on return (VFPI_BAD_ARGUMENT if the capacity is too small). */
int vfpi_augment(vfpi_handle* h, const vfpi_augment_input* in, vfpi_augmented* out);

/* ---- step-pipeline primitives (device pointers, enqueued on `stream`) -- */
/* b = (2/dt) m v - K (x - X) + m g: the elastic right-hand side of the FEM
 * scenes (Eq. 10 with e = u; the reference's assemble_step analogue,
 * dynamics.py:176-218), K in CSR (int64 row pointers), rows summed in
 * increasing column order like scipy's matvec. */
int vfpi_fem_rhs_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, const int32_t* k_indices,
                        const double* k_data, const double* x, const double* X, const double* v, const double* m,
                        const double* g, double dt, double* b, void* stream);
/* The same right-hand side with K packed once as SELL-32 (slices of 32 rows,
 * entry k of row r at slice_off[r/32] + 32 k + r%32, padding column -1):
 * coalesced streaming of K, identical bits. vfpi_sell_layout_device fills
 * slice_off [ceil(n/32)+1] and returns the element count; the caller
 * allocates sell_val/sell_col and calls vfpi_sell_pack_device. */
int vfpi_sell_layout_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, int64_t* slice_off,
                            int64_t* elems);
int vfpi_sell_pack_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, const int32_t* k_indices,
                          const double* k_data, const int64_t* slice_off, double* sell_val, int32_t* sell_col);
int vfpi_fem_rhs_sell_device(vfpi_handle* h, int64_t n, const int64_t* slice_off, const double* sell_val,
                             const int32_t* sell_col, const double* x, const double* X, const double* v,
                             const double* m, const double* g, double dt, double* b, void* stream);
/* y = J x, J in CSR (scipy csr_matvec order): the warm start's virtual-node
 * extension v0[n_o:] = J_v v0[:n_o] (harness._warm_velocity, harness.py:502-512). */
int vfpi_csr_matvec_device(vfpi_handle* h, int64_t rows, const int32_t* indptr, const int32_t* indices,
                           const double* data, const double* x, double* y, void* stream);
/* midpoint integration of the original coordinates (dynamics.py:237-255):
 * x += dt v_hat; v = 2 v_hat - v. */
int vfpi_advance_device(vfpi_handle* h, int64_t n, double dt, const double* v_hat, double* x, double* v,
                        void* stream);

/* ---- cube-pile contacts (configs[4]) -------------- */
/* Plane z = 0 and node-to-face contacts of deformable bodies, detected with a
 * spatial hash and nodalized on the device -- the reference's
 * detect_contacts + nodalize (contacts.py:159-321) extended with a face side
 * (virtual node tied to a triangle by J_v = [w0 I, w1 I, w2 I]); restates
 * paper_2201_09212_b200.pile.CubePile.detect/nodalize bit for bit. */
typedef struct vfpi_pile_geometry {
  int64_t nodes;               /* all nodes (3 DOF each) */
  int64_t n_surf;              /* surface nodes */
  int64_t n_tris;              /* surface triangles */
  const int32_t* surf;         /* [n_surf] ascending node ids */
  const int32_t* tris;         /* [n_tris*3] outward-oriented node ids */
  const int32_t* node_body;    /* [nodes] body of every node */
  const int32_t* tri_body;     /* [n_tris] body of every triangle */
  double reach;                /* bounding-box growth (max(h/2, margin)) */
  double cell;                 /* hash cell edge (2h) */
  double neg_half_h;           /* deepest signed distance accepted (-h/2) */
  double margin;               /* contact margin (contacts.py:28) */
  double mu;                   /* friction coefficient of every contact */
  double neg_beta_dt;          /* -(beta_err / dt) (stabilization_term) */
  double e_rest;
  double rest_threshold;
} vfpi_pile_geometry;

typedef struct vfpi_pile_contacts {  /* device buffers owned by the handle */
  int64_t n_c, n_ground, n_face, n_virtual, jv_nnz;
  int32_t* col_i;
  int32_t* col_j;
  double* frames;      /* [n_c*9] */
  double* mu;          /* [n_c] */
  double* phi;         /* [n_c] */
  int32_t* jv_indptr;  /* [3 n_virtual + 1] canonical CSR of J_v */
  int32_t* jv_indices;
  double* jv_data;
} vfpi_pile_contacts;

/* x, v: device state [3*nodes]; outputs valid until the next call on h. */
int vfpi_pile_contacts_device(vfpi_handle* h, const vfpi_pile_geometry* g, const double* x, const double* v,
                              vfpi_pile_contacts* out, void* stream);
/* ---- nodalization ------------------------------- */
/* condsim.contacts.nodalize (contacts.py:271-321) on the device: raw contacts
 * (sides: 0 node with ref = velocity offset, 1 rigid with ref = body index,
 * -1 static for the second side) -> nodal contacts (slots as augmented
 * columns, virtual nodes, J_v canonical CSR with every block entry stored),
 * frames (contact_frame, :131-149) and phi (stabilization_term, :230-239),
 * bit-identical to the reference. Device pointers in; outputs are device
 * buffers owned by the handle, valid until the next call. mu2 = NaN: None.
 * Side kinds, node offsets and body ids are checked (VFPI_BAD_ARGUMENT). */
typedef struct vfpi_nodalize_input {
  int64_t n_c;
  int64_t n_o;                 /* velocity dimension (columns of J_v) */
  const int32_t* first_kind;
  const int32_t* first_ref;
  const int32_t* second_kind;
  const int32_t* second_ref;
  const double* point;         /* [n_c*3] */
  const double* normal;        /* [n_c*3] (normalised inside, as contact_frame does) */
  const double* depth;         /* [n_c] */
  const double* q;             /* generalized coordinates (rigid: position + quaternion) */
  const double* v;             /* [n_o] velocities */
  const int32_t* body_q;       /* per body: coordinate offset (Body.q_offset) */
  const int32_t* body_v;       /* per body: velocity offset (Body.v_offset) */
  double mu, mu2, beta_err, dt, e_rest, rest_threshold;
  int64_t n_bodies;            /* entries of body_q / body_v (rigid side ids are checked against it) */
  int64_t n_q;                 /* entries of q: a rigid side needs body_q + 3 <= n_q and body_v + 6 <= n_o */
} vfpi_nodalize_input;

typedef struct vfpi_nodal_contacts {
  int64_t n_c, n_virtual, jv_nnz;
  int32_t* col_i;       /* augmented column of side i */
  int32_t* col_j;       /* augmented column of side j, -1 for S contacts */
  double* frames;       /* [n_c*9] */
  double* phi;
  double* mu;
  double* mu2;
  int32_t* jv_indptr;   /* [3 n_virtual + 1] */
  int32_t* jv_indices;
  double* jv_data;
} vfpi_nodal_contacts;

int vfpi_nodalize_device(vfpi_handle* h, const vfpi_nodalize_input* in, vfpi_nodal_contacts* out, void* stream);

/* synchronous device-to-device copy (reading handle-owned outputs into caller buffers) */
int vfpi_memcpy_d2d(void* dst, const void* src, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* VFPI_H */
