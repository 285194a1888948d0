// C-ABI (include/vfpi.h): handles, host<->device staging, solve orchestration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "vfpi_internal.cuh"

using vfpi::Workspace;

cudaError_t vfpi::ensure_max_dynamic_smem(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  cudaFuncAttributes a{};
  cudaError_t e = cudaFuncGetAttributes(&a, fn);
  if (e != cudaSuccess) return e;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({dev, fn});
  return e;
}

// A captured setup phase: replayed as one graph launch when the next solve has
// the same shapes, input pointers, options and workspace allocations (key).
struct SetupGraph {
  std::vector<uint64_t> key, last_key;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  uint64_t used = 0;  // LRU tick
};
// two graphs per phase: a caller that alternates two input buffers (double-
// buffered uploads overlapping the previous solve) replays both
struct SetupGraphSet {
  SetupGraph slot[2];
  uint64_t tick = 0;
};

struct vfpi_handle {
  Workspace ws;
  SetupGraphSet graph_layout, graph_pack;
  int use_graphs = 1;
  std::string err;
  int64_t launches = 0;
  // last solve (device path) bookkeeping for vfpi_wait
  int pending = 0;
  int max_iters = 0;
  int last_resident = 0;
  int kernel_mode = 0;  // 0 auto, 1 force shared-memory resident, 2 force streaming
  int prof_iter0 = 0;   // >0: record phase timestamps of iterations prof_iter0..+3
  int node_kernel = 1;  // FEM batches: node-block SELL kernel when a node layout is set (tuning key 6)
  int node_cluster = 1; // small FEM batches: one thread-block cluster per scene (tuning key 8; set before the layout)
  int node_cluster_force = 0;  // > 0: CTAs per scene of FEM batches created afterwards (tuning key 9)
  int grid_contact_cost = 8;   // single systems: partition weight of a single-node contact in blocks (key 11)
  int grid_pack = 2;           // single systems: packed block values (0 off, 1 auto, 2 auto + mask-grouped nodes, 3 always; key 12)
  int last_node_kernel = 0;
  vfpi::LayoutOptions layout_opt;
  vfpi::AugmentWork aug;
  vfpi::PileWork pile;
  vfpi::NodalizeWork nod;
  vfpi::HfWork hf;
  vfpi::NodeGridWork ngw;  // node-block layout of the last single-system solve
  int last_G = 0;
  int* h_flags = nullptr;  // pinned
};

namespace {

#define CK(x)                                                     \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) {                                      \
      h->err = std::string(#x) + ": " + cudaGetErrorString(e_);   \
      return VFPI_CUDA_ERROR;                                     \
    }                                                             \
  } while (0)

template <class T>
T* P(Workspace::Buf& b) { return reinterpret_cast<T*>(b.p); }

// CTAs for the global-memory (streaming) kernel: a multiple of the SM count
// so every SM carries the same share of the cost-balanced partition.
int choose_blocks(const vfpi_system& s, int num_sms) {
  const int64_t by_nnz = (s.nnz + 4095) / 4096;
  if (by_nnz < num_sms) return (int)std::max<int64_t>(1, by_nnz);
  if (by_nnz >= 4 * num_sms) return 4 * num_sms;  // HBM streaming wants several CTAs per SM
  return by_nnz >= 2 * num_sms ? 2 * num_sms : num_sms;
}

// CTAs for the shared-memory-resident kernel: one per SM at most.
int choose_blocks_resident(const vfpi_system& s, int num_sms) {
  const int64_t by_nnz = (s.nnz + 2047) / 2048;
  return (int)std::max<int64_t>(1, std::min<int64_t>(by_nnz, num_sms));
}

// Run a setup phase: eagerly the first time a key is seen (this is where the
// workspace grows), captured into a graph the second time, replayed after.
template <class F>
int run_setup_phase(vfpi_handle* h, SetupGraphSet& gs, std::vector<uint64_t> key, cudaStream_t st, F&& body) {
  const bool capturable = h->use_graphs && st != nullptr && st != cudaStreamLegacy && st != cudaStreamPerThread;
  key.push_back(vfpi::alloc_generation());
  key.push_back((uint64_t)(uintptr_t)st);
  if (!capturable) return body();
  int si = -1;
  for (int i = 0; i < 2 && si < 0; ++i)
    if (gs.slot[i].key == key || gs.slot[i].last_key == key) si = i;
  if (si < 0) si = gs.slot[0].used <= gs.slot[1].used ? 0 : 1;
  SetupGraph& g = gs.slot[si];
  g.used = ++gs.tick;
  if (g.exec && g.key == key) {
    CK(cudaGraphLaunch(g.exec, st));
    h->launches += g.launches;
    return VFPI_OK;
  }
  if (g.last_key != key) {
    g.last_key = key;
    return body();
  }
  const int64_t l0 = h->launches;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  const int rc = body();
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &graph);
  if (rc != VFPI_OK || e != cudaSuccess || vfpi::alloc_generation() != key[key.size() - 2]) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    g.last_key.clear();
    h->launches = l0;
    return rc != VFPI_OK ? rc : body();  // capture not possible: run eagerly
  }
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g.exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    g.exec = nullptr;
    g.last_key.clear();
    h->launches = l0;
    return body();
  }
  g.key = key;
  g.launches = h->launches - l0;
  CK(cudaGraphLaunch(g.exec, st));
  return VFPI_OK;
}

std::vector<uint64_t> system_key(const vfpi_system& d, int G) {
  return {(uint64_t)d.n, (uint64_t)d.n_c, (uint64_t)d.nnz, (uint64_t)G, (uint64_t)(uintptr_t)d.indptr,
          (uint64_t)(uintptr_t)d.indices, (uint64_t)(uintptr_t)d.data, (uint64_t)(uintptr_t)d.b,
          (uint64_t)(uintptr_t)d.col_i, (uint64_t)(uintptr_t)d.col_j, (uint64_t)(uintptr_t)d.frames,
          (uint64_t)(uintptr_t)d.mu, (uint64_t)(uintptr_t)d.mu2, (uint64_t)(uintptr_t)d.phi};
}

int upload(vfpi_handle* h, Workspace::Buf& b, const void* src, size_t bytes, cudaStream_t st = nullptr) {
  if (bytes == 0) return VFPI_OK;
  CK(vfpi::ensure(b, bytes));
  CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, st ? st : h->ws.stream));
  return VFPI_OK;
}

// host-side validation common to all entry points (sizes only; the device
// checks column ranges and overlaps)
int check_system(vfpi_handle* h, const vfpi_system* s) {
  if (!s) { h->err = "null system"; return VFPI_BAD_ARGUMENT; }
  if (s->n < 0 || s->n_c < 0 || s->nnz < 0 || s->n > (int64_t)1 << 30 || s->nnz > ((int64_t)1 << 31) - 1) {
    h->err = "system sizes out of range";
    return VFPI_BAD_ARGUMENT;
  }
  return VFPI_OK;
}

// copy a host system into the handle's device input buffers. With
// `overlap`, the arrays the layout setup does not read (b, frames, mu, mu2,
// phi) go on the side stream after the others, so they cross PCIe while the
// setup kernels run (the solve waits for them before its first use).
int stage_system(vfpi_handle* h, const vfpi_system* s, vfpi_system* d, bool overlap = false) {
  Workspace& ws = h->ws;
  const size_t n = (size_t)s->n, nc = (size_t)s->n_c, nnz = (size_t)s->nnz;
  int rc;
  // allocate everything first (ensure may free/realloc and synchronise)
  for (auto& pr : {std::make_pair(&ws.b_indptr, 4 * (n + 1)), std::make_pair(&ws.b_indices, 4 * nnz),
                   std::make_pair(&ws.b_data, 8 * nnz), std::make_pair(&ws.b_b, 8 * n),
                   std::make_pair(&ws.b_ci, 4 * nc), std::make_pair(&ws.b_cj, 4 * nc),
                   std::make_pair(&ws.b_frames, 72 * nc), std::make_pair(&ws.b_mu, 8 * nc),
                   std::make_pair(&ws.b_mu2, 8 * nc), std::make_pair(&ws.b_phi, 8 * nc)})
    if (pr.second) CK(vfpi::ensure(*pr.first, pr.second));
  if ((rc = upload(h, ws.b_indptr, s->indptr, 4 * (n + 1)))) return rc;
  if ((rc = upload(h, ws.b_indices, s->indices, 4 * nnz))) return rc;
  if ((rc = upload(h, ws.b_data, s->data, 8 * nnz))) return rc;
  if (nc) {
    if ((rc = upload(h, ws.b_ci, s->col_i, 4 * nc))) return rc;
    if ((rc = upload(h, ws.b_cj, s->col_j, 4 * nc))) return rc;
  }
  cudaStream_t late = ws.stream;
  if (overlap) {
    CK(cudaEventRecord(ws.ev_main_h2d, ws.stream));
    CK(cudaStreamWaitEvent(ws.side, ws.ev_main_h2d, 0));
    late = ws.side;
  }
  if (s->b && (rc = upload(h, ws.b_b, s->b, 8 * n, late))) return rc;
  if (nc) {
    if ((rc = upload(h, ws.b_frames, s->frames, 72 * nc, late))) return rc;
    if (s->mu && (rc = upload(h, ws.b_mu, s->mu, 8 * nc, late))) return rc;
    if (s->mu2 && (rc = upload(h, ws.b_mu2, s->mu2, 8 * nc, late))) return rc;
    if (s->phi && (rc = upload(h, ws.b_phi, s->phi, 8 * nc, late))) return rc;
  }
  *d = *s;
  d->indptr = P<int32_t>(ws.b_indptr);
  d->indices = P<int32_t>(ws.b_indices);
  d->data = P<double>(ws.b_data);
  d->b = P<double>(ws.b_b);
  d->col_i = P<int32_t>(ws.b_ci);
  d->col_j = P<int32_t>(ws.b_cj);
  d->frames = P<double>(ws.b_frames);
  d->mu = P<double>(ws.b_mu);
  d->mu2 = P<double>(ws.b_mu2);
  d->phi = P<double>(ws.b_phi);
  return VFPI_OK;
}

int flags_to_code(vfpi_handle* h, int flags) {
  if (flags & 2) { h->err = "contact column index out of range"; return VFPI_BAD_ARGUMENT; }
  if (flags & 1) { h->err = "two contacts share a node column"; return VFPI_UNSUPPORTED; }
  if (flags & 4) { h->err = "zero row norm in step-matrix computation"; return VFPI_INVALID_MATRIX; }
  if (flags & 8) { h->err = "step matrix violates the per-node tie groups"; return VFPI_TIE_VIOLATION; }
  return VFPI_OK;
}

// layout for the per-op entry points (CSR order, no contact partition needed)
int op_layout(vfpi_handle* h, const vfpi_system& d, bool with_contacts) {
  vfpi_system dd = d;
  if (!with_contacts) dd.n_c = 0;
  vfpi::SetupSummary* hs = h->ws.h_summary;
  int rc = vfpi::setup_layout(h->ws, dd, 1, h->ws.stream, hs, h->err, h->launches);
  if (rc) return rc;
  return vfpi::setup_pack(h->ws, dd, 1, true, *hs, h->ws.stream, h->err, h->launches);
}

}  // namespace

extern "C" {

int vfpi_version(void) { return 1; }

int vfpi_create(int device, vfpi_handle** out) {
  if (!out) return VFPI_BAD_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0 || device < 0 || device >= count)
    return VFPI_CUDA_ERROR;
  if (cudaSetDevice(device) != cudaSuccess) return VFPI_CUDA_ERROR;
  vfpi_handle* h = new vfpi_handle();
  h->ws.device = device;
  cudaDeviceGetAttribute(&h->ws.num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&h->ws.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (cudaStreamCreateWithFlags(&h->ws.stream, cudaStreamNonBlocking) != cudaSuccess) { delete h; return VFPI_CUDA_ERROR; }
  for (auto& e : h->ws.ev) cudaEventCreate(&e);
  cudaStreamCreateWithFlags(&h->ws.side, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&h->ws.ev_main_h2d, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ws.ev_side, cudaEventDisableTiming);
  cudaMallocHost(&h->ws.h_summary, sizeof(vfpi::SetupSummary));
  cudaMallocHost(&h->ws.h_status, sizeof(vfpi::SolveStatus));
  cudaMallocHost(&h->h_flags, 16);
  cudaMallocHost(&h->aug.h_small, 2 * sizeof(int64_t));
  cudaMallocHost(&h->pile.h_small, 4 * sizeof(int64_t));
  cudaMallocHost(&h->nod.h_small, 2 * sizeof(int64_t));
  *out = h;
  return VFPI_OK;
}

void vfpi_destroy(vfpi_handle* h) {
  if (!h) return;
  cudaSetDevice(h->ws.device);
  cudaStreamSynchronize(h->ws.stream);
  Workspace::Buf* bufs[] = {&h->ws.b_indptr, &h->ws.b_indices, &h->ws.b_data, &h->ws.b_b, &h->ws.b_ci,
                            &h->ws.b_cj, &h->ws.b_frames, &h->ws.b_mu, &h->ws.b_mu2, &h->ws.b_phi,
                            &h->ws.b_warm, &h->ws.b_wc, &h->ws.b_out_v, &h->ws.b_out_lam, &h->ws.b_trace,
                            &h->ws.b_scc, &h->ws.b_w_out, &h->ws.diag, &h->ws.rns, &h->ws.w, &h->ws.gamma,
                            &h->ws.w_mean, &h->ws.rowcnt, &h->ws.row_ptr, &h->ws.keys, &h->ws.keys_sorted,
                            &h->ws.vals, &h->ws.perm, &h->ws.colof, &h->ws.mark, &h->ws.ucost, &h->ws.cpos,
                            &h->ws.urows, &h->ws.rpos, &h->ws.ucont, &h->ws.kpos, &h->ws.blk_row, &h->ws.blk_ct,
                            &h->ws.blk_slice, &h->ws.row_list, &h->ws.row_slot, &h->ws.cont_list,
                            &h->ws.slice_w, &h->ws.slice_off, &h->ws.sell_val, &h->ws.sell_col, &h->ws.pos_len, &h->ws.pos_ptr,
                            &h->ws.pk_val, &h->ws.pk_col, &h->ws.bar_flags, &h->ws.ucr, &h->ws.ufr,
                            &h->ws.cposc, &h->ws.cposf, &h->ws.blk_first, &h->ws.blk_cr, &h->ws.cont_q,
                            &h->ws.ps_col, &h->ws.ps_src, &h->ws.seg_beg, &h->ws.seg_end, &h->ws.rowpos, &h->ws.sec_key,
                            &h->ws.sec_skey, &h->ws.sec_idx, &h->ws.sec_sidx, &h->ws.sec_flag, &h->ws.sec_upos,
                            &h->ws.sell_map, &h->ws.secs, &h->ws.sec_ptr, &h->ws.rowmin, &h->ws.ukey, &h->ws.ukey_s,
                            &h->ws.uval, &h->ws.uorder, &h->ws.row_list2, &h->ws.row_slot2, &h->ws.rowblk,
                            &h->ws.scene_rows, &h->ws.scene_cts, &h->ws.vbuf,
                            &h->ws.lambuf, &h->ws.partials, &h->ws.status, &h->ws.summary, &h->ws.flags,
                            &h->ws.cub_tmp, &h->ws.x, &h->ws.y, &h->ws.prof, &h->ws.cg_vec, &h->ws.cg_part};
  for (auto* b : bufs)
    if (b->p) vfpi::dev_free(b->p);
  vfpi::AugmentWork& aw = h->aug;
  for (Workspace::Buf* b : {&aw.pcnt, &aw.poff, &aw.pkey, &aw.pkey2, &aw.pval, &aw.pval2, &aw.head, &aw.hpos, &aw.tmp,
                            &aw.tmp2, &aw.jrow, &aw.jcol_s, &aw.jidx, &aw.jperm, &aw.jcp, &aw.t_row, &aw.t_col,
                            &aw.t_val, &aw.cs, &aw.ccnt, &aw.cptr, &aw.out_p, &aw.out_i, &aw.out_x})
    if (b->p) vfpi::dev_free(b->p);
  if (aw.h_small) cudaFreeHost(aw.h_small);
  vfpi::PileWork& pw = h->pile;
  for (Workspace::Buf* b : {&pw.tcnt, &pw.toff, &pw.flag, &pw.key, &pw.key2, &pw.own, &pw.own2, &pw.btri, &pw.best,
                            &pw.gflag, &pw.gpos, &pw.fflag, &pw.fpos, &pw.nvirt, &pw.vpos, &pw.njv, &pw.jpos, &pw.ci,
                            &pw.cj, &pw.fr, &pw.mu, &pw.phi, &pw.jrp, &pw.jci, &pw.jcx, &pw.tmp})
    if (b->p) vfpi::dev_free(b->p);
  if (pw.h_small) cudaFreeHost(pw.h_small);
  vfpi::NodalizeWork& nw = h->nod;
  for (Workspace::Buf* b : {&nw.first, &nw.vflag, &nw.vpos, &nw.jcnt, &nw.jpos, &nw.flag, &nw.tmp, &nw.ci, &nw.cj,
                            &nw.fr, &nw.phi, &nw.mu, &nw.mu2, &nw.jrp, &nw.jci, &nw.jcx})
    if (b->p) vfpi::dev_free(b->p);
  if (nw.h_small) cudaFreeHost(nw.h_small);
  vfpi::HfWork& hw = h->hf;
  for (auto* b : {&hw.flag, &hw.pos, &hw.tmp, &hw.ci, &hw.cj, &hw.fr, &hw.mu, &hw.phi})
    if (b->p) vfpi::dev_free(b->p);
  if (hw.h_small) cudaFreeHost(hw.h_small);
  vfpi::NodeGridWork& gw = h->ngw;
  for (auto* b : {&gw.blk_pos, &gw.blk_slice, &gw.key, &gw.key2, &gw.val_i, &gw.node_list, &gw.cnt, &gw.node_slot,
                  &gw.width, &gw.slice_off, &gw.flags, &gw.vs, &gw.jt, &gw.tmp, &gw.desc, &gw.val})
    if (b->p) vfpi::dev_free(b->p);
  if (gw.h_small) cudaFreeHost(gw.h_small);
  for (auto& e : h->ws.ev)
    if (e) cudaEventDestroy(e);
  for (SetupGraphSet* gs : {&h->graph_layout, &h->graph_pack})
    for (SetupGraph& g : gs->slot)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  if (h->ws.stream) cudaStreamDestroy(h->ws.stream);
  if (h->ws.side) cudaStreamDestroy(h->ws.side);
  if (h->ws.ev_main_h2d) cudaEventDestroy(h->ws.ev_main_h2d);
  if (h->ws.ev_side) cudaEventDestroy(h->ws.ev_side);
  if (h->ws.h_summary) cudaFreeHost(h->ws.h_summary);
  if (h->ws.h_status) cudaFreeHost(h->ws.h_status);
  if (h->h_flags) cudaFreeHost(h->h_flags);
  delete h;
}

const char* vfpi_last_error(const vfpi_handle* h) { return h ? h->err.c_str() : "null handle"; }

int64_t vfpi_launch_count(const vfpi_handle* h) { return h ? h->launches : 0; }

void* vfpi_stream(vfpi_handle* h) { return h ? (void*)h->ws.stream : nullptr; }

int vfpi_cg_device(vfpi_handle* h, int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                   const double* b, double* x, double rtol, int64_t maxiter, int32_t* iterations, void* stream) {
  if (!h || n < 0 || (n > 0 && (!indptr || !indices || !data || !b || !x))) return VFPI_BAD_ARGUMENT;
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  if (n == 0) {
    if (iterations) *iterations = 0;
    return VFPI_OK;
  }
  Workspace& ws = h->ws;
  const int G = vfpi::cg_grid_partials(ws.device);
  CK(vfpi::ensure(ws.cg_vec, 8 * 3 * (size_t)n));
  CK(vfpi::ensure(ws.cg_part, 8 * 2 * (size_t)G + 8));
  double* r = P<double>(ws.cg_vec);
  if (vfpi::launch_cg_grid(G, n, indptr, indices, data, b, x, r, r + n, r + 2 * n, P<double>(ws.cg_part), rtol,
                           maxiter, P<int32_t>(ws.cg_part) + 4 * G, st)) {
    h->err = "fallback CG launch failed";
    return VFPI_CUDA_ERROR;
  }
  ++h->launches;
  int32_t it = 0;
  CK(cudaMemcpyAsync(&it, P<int32_t>(ws.cg_part) + 4 * G, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (iterations) *iterations = it;
  return VFPI_OK;
}

int vfpi_set_tuning(vfpi_handle* h, int key, int value) {
  if (!h) return VFPI_BAD_ARGUMENT;
  if (key == 1) { h->layout_opt.anchor_order = value != 0; return VFPI_OK; }
  if (key == 2) { h->layout_opt.length_sort = value != 0; return VFPI_OK; }
  if (key == 3 && value > 0) { h->layout_opt.entry_cost = value; return VFPI_OK; }
  if (key == 4 && value > 0) {
    h->layout_opt.row_cost = h->layout_opt.res_row_cost = value;
    return VFPI_OK;
  }
  if (key == 5 && value >= 0) { h->layout_opt.contact_cost = value; return VFPI_OK; }
  if (key == 6) { h->node_kernel = value != 0; return VFPI_OK; }
  if (key == 7) return h->last_node_kernel;  // query: did the last scene solve use the node-block kernel
  if (key == 8) { h->node_cluster = value != 0; return VFPI_OK; }
  if (key == 11 && value >= 0) { h->grid_contact_cost = value; return VFPI_OK; }
  if (key == 12 && value >= 0 && value <= 3) { h->grid_pack = value; return VFPI_OK; }
  if (key == 13) return h->ngw.packed ? 1 : 0;  // query: did the last single-system grid layout pack its values
  if (key == 9 && (value == 0 || value == 1 || value == 2 || value == 4 || value == 8)) {
    h->node_cluster_force = value;
    return VFPI_OK;
  }
  return VFPI_BAD_ARGUMENT;
}

int vfpi_set_profile(vfpi_handle* h, int iter0) {
  if (!h || iter0 < 0) return VFPI_BAD_ARGUMENT;
  h->prof_iter0 = iter0;
  return VFPI_OK;
}

int vfpi_get_profile(vfpi_handle* h, long long* out, int64_t max_count) {
  if (!h || !out) return VFPI_BAD_ARGUMENT;
  const int64_t cnt = std::min<int64_t>(max_count, 64 * (int64_t)h->last_G);
  if (!h->ws.prof.p || cnt <= 0) return VFPI_BAD_ARGUMENT;
  cudaSetDevice(h->ws.device);
  CK(cudaStreamSynchronize(h->ws.stream));
  CK(cudaMemcpy(out, h->ws.prof.p, sizeof(long long) * (size_t)cnt, cudaMemcpyDeviceToHost));
  return VFPI_OK;
}

int vfpi_set_kernel(vfpi_handle* h, int mode) {
  if (!h || mode < 0 || mode > 2) return VFPI_BAD_ARGUMENT;
  h->kernel_mode = mode;
  return VFPI_OK;
}

int vfpi_last_layout(const vfpi_handle* h, int* resident, int* ctas) {
  if (!h) return VFPI_BAD_ARGUMENT;
  if (resident) *resident = h->last_resident;
  if (ctas) *ctas = h->last_G;
  return VFPI_OK;
}

void* vfpi_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, (size_t)std::max<int64_t>(bytes, 8)) != cudaSuccess) return nullptr;
  return p;
}

void vfpi_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int vfpi_solve_device(vfpi_handle* h, const vfpi_system* d, const vfpi_config* cfg, const double* warm,
                      const double* w_cached, vfpi_result* res, void* stream_) {
  if (!h || !cfg || !res || !warm) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, d);
  if (rc) return rc;
  if (cfg->op < 0 || cfg->op > 2 || cfg->step_strategy < 0 || cfg->step_strategy > 4 || cfg->max_iters < 0) {
    h->err = "bad solver config";
    return VFPI_BAD_ARGUMENT;
  }
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  Workspace& ws = h->ws;
  cudaStream_t st = stream_ ? (cudaStream_t)stream_ : ws.stream;
  const int n = (int)d->n, n_c = (int)d->n_c;
  const bool cheb = cfg->chebyshev != 0;
  const bool bb = cfg->step_strategy >= VFPI_STEP_BB1 && cfg->step_strategy <= VFPI_STEP_BB_ALTERNATING;

  CK(cudaEventRecord(ws.ev[0], st));
  vfpi::SetupSummary* hs = ws.h_summary;
  // first choice: the whole partition of every CTA resident in shared memory.
  // Skipped when it cannot fit: every valid row needs >= 52 B on chip (40 B of
  // row state + one numeric entry of 12 B; a row without one is a zero row)
  int G = choose_blocks_resident(*d, ws.num_sms);
  const bool maybe_resident =
      h->kernel_mode == 1 || (int64_t)n * 52 <= (int64_t)ws.max_smem_optin * (int64_t)ws.num_sms;
  if (maybe_resident) {
    std::vector<uint64_t> key = system_key(*d, G);
    vfpi::LayoutOptions res_opt = h->layout_opt;
    res_opt.row_cost = res_opt.res_row_cost;
    const vfpi::LayoutOptions& o = res_opt;
    for (uint64_t x : {(uint64_t)o.anchor_order, (uint64_t)o.length_sort, (uint64_t)o.entry_cost,
                       (uint64_t)o.row_cost, (uint64_t)o.contact_cost})
      key.push_back(x);
    rc = run_setup_phase(h, h->graph_layout, key, st, [&] {
      return vfpi::setup_layout_async(ws, *d, G, st, h->err, h->launches, res_opt);
    });
    if (rc) return rc;
    rc = vfpi::setup_layout_finish(ws, st, hs, h->err);
    if (rc) return rc;
  }
  const size_t smem_res = maybe_resident ? (size_t)hs->max_res_bytes : 0;
  const bool fits = maybe_resident && hs->max_ent_per_blk < (1 << 24) &&
                    smem_res + 2048 <= (size_t)ws.max_smem_optin && G <= 256;
  if (h->kernel_mode == 1 && !fits) { h->err = "partition does not fit in shared memory"; return VFPI_UNSUPPORTED; }
  bool resident = fits && h->kernel_mode != 2;
  int smem = 0;
  if (!resident) {
    G = choose_blocks(*d, ws.num_sms);
    for (int attempt = 0; attempt < 4; ++attempt) {
      rc = vfpi::setup_layout(ws, *d, G, st, hs, h->err, h->launches, h->layout_opt);
      if (rc) return rc;
      smem = 2 * vfpi::kSlotsPerContact * 8 * hs->max_ct_per_blk;
      const int bps = vfpi::iterate_max_blocks_per_sm(cfg->op, cheb, bb, smem);
      if (bps <= 0) { h->err = "iteration kernel does not fit on an SM"; return VFPI_UNSUPPORTED; }
      if (G <= bps * ws.num_sms) break;
      G = bps * ws.num_sms;
    }
  }
  if (resident) {
    std::vector<uint64_t> key = system_key(*d, G);
    for (uint64_t x : {(uint64_t)hs->n_slices, (uint64_t)hs->sell_elems, (uint64_t)hs->nnz_num})
      key.push_back(x);
    rc = run_setup_phase(h, h->graph_pack, key, st, [&] {
      return vfpi::setup_pack(ws, *d, G, true, *hs, st, h->err, h->launches);
    });
  } else {
    rc = vfpi::setup_pack(ws, *d, G, false, *hs, st, h->err, h->launches);
  }
  if (rc) return rc;
  // single systems that do not fit on chip: the node-block streaming kernel
  // (csrc/vfpi_nodes.cu) when every contact column is node aligned and the
  // step is not Barzilai-Borwein; otherwise the row-SELL streaming kernel
  bool use_nodes = false;
  int G_nodes = 0;
  vfpi::NodeLayoutDev nl;
  if (!resident && h->node_kernel && !bb && n % 3 == 0) {
    const int bps = vfpi::node_kernel_blocks_per_sm(cfg->op, cheb, 0, 1);
    if (bps > 0) {
      G_nodes = bps * ws.num_sms;
      rc = vfpi::node_grid_build(h->ngw, *d, G_nodes, P<int64_t>(ws.row_ptr), P<int>(ws.rowcnt), P<int>(ws.perm),
                                 P<int>(ws.colof), st, nl, h->err, h->launches,
                                 h->grid_contact_cost, h->grid_pack);
      if (rc == VFPI_OK) use_nodes = true;
      else if (rc != VFPI_UNSUPPORTED) return rc;
    }
  }
  const size_t smem_res_full = smem_res;
  rc = vfpi::setup_step_matrix(ws, *d, *cfg, w_cached, st, h->err, h->launches);
  if (rc) return rc;

  const int tr = std::max(cfg->max_iters, 1);
  // v ring: each buffer 32-byte aligned with 4 spare doubles, because the
  // resident kernel stages whole 32-byte sectors
  const size_t npad = (((size_t)std::max(n, 1) + 3) / 4) * 4 + 4;
  CK(vfpi::ensure(ws.vbuf, 3 * 8 * npad));
  if (ws.side_pending) {  // host-buffer solve: b, frames, mu, mu2, phi, warm came on the side stream
    CK(cudaStreamWaitEvent(st, ws.ev_side, 0));
    ws.side_pending = false;
  }
  CK(cudaMemsetAsync(ws.vbuf.p, 0, 3 * 8 * npad, st));
  CK(vfpi::ensure(ws.lambuf, 2 * 24 * (size_t)std::max(n_c, 1)));
  if (use_nodes) G = G_nodes;
  CK(vfpi::ensure(ws.partials, 2 * 8 * (size_t)G * vfpi::kPartialStride));
  CK(vfpi::ensure(ws.status, sizeof(vfpi::SolveStatus)));
  CK(vfpi::ensure(ws.bar_flags, 4 * (size_t)G));
  CK(cudaMemsetAsync(ws.bar_flags.p, 0, 4 * (size_t)G, st));
  double* vb = P<double>(ws.vbuf);
  double* lb = P<double>(ws.lambuf);
  if (n > 0) {
    CK(cudaMemcpyAsync(vb, warm, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(vb + 2 * npad, warm, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaMemsetAsync(lb, 0, 2 * 24 * (size_t)std::max(n_c, 1), st));
  CK(cudaMemsetAsync(ws.status.p, 0, sizeof(vfpi::SolveStatus), st));
  CK(cudaEventRecord(ws.ev[1], st));

  vfpi::IterParams p{};
  p.n = n;
  p.n_c = n_c;
  p.G = G;
  p.row_list = P<int>(ws.row_list);
  p.row_slot = P<int>(ws.row_slot);
  p.blk_row = P<int>(ws.blk_row);
  p.blk_slice = P<int>(ws.blk_slice);
  p.blk_ct = P<int>(ws.blk_ct);
  p.slice_off = P<int64_t>(ws.slice_off);
  p.sell_val = P<double>(ws.sell_val);
  p.sell_col = P<int>(ws.sell_col);
  p.pos_ptr = P<int64_t>(ws.pos_ptr);
  p.sell_map = P<unsigned>(ws.sell_map);
  p.secs = P<unsigned>(ws.secs);
  p.sec_ptr = P<int>(ws.sec_ptr);
  p.blk_cr = P<int>(ws.blk_cr);
  p.cont_q = P<int>(ws.cont_q);
  p.bar_flags = P<int>(ws.bar_flags);
  p.prof = nullptr;
  p.prof_iter0 = 0;
  p.diag = P<double>(ws.diag);
  p.fixed_alpha_default = 0;
  p.trace_stride = 0;
  if (h->prof_iter0 > 0) {
    CK(vfpi::ensure(ws.prof, sizeof(long long) * 64 * (size_t)G));
    CK(cudaMemsetAsync(ws.prof.p, 0, sizeof(long long) * 64 * (size_t)G, st));
    p.prof = P<long long>(ws.prof);
    p.prof_iter0 = h->prof_iter0;
  }
  p.cont_list = P<int>(ws.cont_list);
  p.b = d->b;
  p.w = P<double>(ws.w);
  p.gamma = P<double>(ws.gamma);
  p.col_i = d->col_i;
  p.col_j = d->col_j;
  p.frames = d->frames;
  p.mu = d->mu;
  p.mu2 = d->mu2;
  p.phi = d->phi;
  p.w_mean = P<double>(ws.w_mean);
  p.vbuf0 = vb;
  p.vbuf1 = vb + npad;
  p.vbuf2 = vb + 2 * npad;
  p.lam0 = lb;
  p.lam1 = lb + 3 * (size_t)std::max(n_c, 1);
  p.partials = P<double>(ws.partials);
  p.trace = res->residual_trace;
  p.status = P<vfpi::SolveStatus>(ws.status);
  p.out_v = res->v;
  p.out_lam = res->lam;
  p.max_iters = cfg->max_iters;
  p.cheby_start = cfg->cheby_start;
  p.step = cfg->step_strategy;
  p.tol = cfg->residual_tol;
  p.under_relax = cfg->under_relax;
  p.omega = cfg->omega;
  p.cfactor = cfg->consistency_factor;
  (void)tr;
  if (use_nodes) {
    rc = vfpi::launch_iterate_nodes(p, nl, cfg->op, cheb, 0, st, h->err, 1);
  } else {
    rc = resident ? vfpi::launch_iterate_resident(p, cfg->op, cheb, bb, smem_res_full, st, h->err)
                  : vfpi::launch_iterate(p, cfg->op, cheb, bb, smem, st, h->err);
  }
  if (rc) return rc;
  h->last_node_kernel = use_nodes ? 1 : 0;
  h->last_resident = resident ? 1 : 0;
  h->last_G = G;
  ++h->launches;
  CK(cudaEventRecord(ws.ev[2], st));
  if (res->scc && n_c > 0) {
    rc = vfpi::launch_scc_final(p, res->scc, st);
    if (rc) { h->err = "scc kernel launch failed"; return rc; }
    ++h->launches;
  }
  if (res->w && n > 0) CK(cudaMemcpyAsync(res->w, ws.w.p, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(ws.h_status, ws.status.p, sizeof(vfpi::SolveStatus), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->h_flags, ws.flags.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ws.ev[3], st));
  h->pending = 1;
  h->max_iters = cfg->max_iters;
  return VFPI_OK;
}

int vfpi_wait(vfpi_handle* h, vfpi_result* res) {
  if (!h || !res) return VFPI_BAD_ARGUMENT;
  if (!h->pending) { h->err = "no solve pending"; return VFPI_BAD_ARGUMENT; }
  cudaSetDevice(h->ws.device);
  h->pending = 0;
  CK(cudaEventSynchronize(h->ws.ev[3]));
  const vfpi::SolveStatus& s = *h->ws.h_status;
  res->iterations = s.iterations;
  res->converged = s.converged;
  res->diverged = s.diverged;
  res->consistency = s.consistency;
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, h->ws.ev[0], h->ws.ev[1]);
  cudaEventElapsedTime(&b, h->ws.ev[1], h->ws.ev[2]);
  res->setup_ms = a;
  res->loop_ms = b;
  int rc = flags_to_code(h, *h->h_flags);
  if (!rc && s.diverged) {
    h->err = "non-finite iterate in V-FPI";
    rc = VFPI_DIVERGED;
  }
  res->status = rc;
  return rc;
}

int vfpi_solve(vfpi_handle* h, const vfpi_system* s, const vfpi_config* cfg, const double* warm,
               const double* w_cached, vfpi_result* res) {
  if (!h || !cfg || !res || !warm) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  Workspace& ws = h->ws;
  vfpi_system d;
  const size_t n = (size_t)s->n, nc = (size_t)s->n_c;
  CK(vfpi::ensure(ws.b_warm, 8 * std::max<size_t>(n, 1)));
  if ((rc = stage_system(h, s, &d, true))) return rc;
  if ((rc = upload(h, ws.b_warm, warm, 8 * n, ws.side))) return rc;
  CK(cudaEventRecord(ws.ev_side, ws.side));
  ws.side_pending = true;
  const double* dwc = nullptr;
  if (w_cached) {
    if ((rc = upload(h, ws.b_wc, w_cached, 8 * n))) return rc;
    dwc = P<double>(ws.b_wc);
  }
  const size_t tr = (size_t)std::max(cfg->max_iters, 1);
  CK(vfpi::ensure(ws.b_out_v, 8 * std::max<size_t>(n, 1)));
  CK(vfpi::ensure(ws.b_out_lam, 24 * std::max<size_t>(nc, 1)));
  CK(vfpi::ensure(ws.b_trace, 8 * tr));
  CK(vfpi::ensure(ws.b_scc, 8 * std::max<size_t>(nc, 1)));
  CK(vfpi::ensure(ws.b_w_out, 8 * std::max<size_t>(n, 1)));
  vfpi_result dres = *res;
  dres.v = P<double>(ws.b_out_v);
  dres.lam = P<double>(ws.b_out_lam);
  dres.residual_trace = P<double>(ws.b_trace);
  dres.scc = res->scc ? P<double>(ws.b_scc) : nullptr;
  dres.w = res->w ? P<double>(ws.b_w_out) : nullptr;
  rc = vfpi_solve_device(h, &d, cfg, P<double>(ws.b_warm), dwc, &dres, ws.stream);
  if (rc) {
    cudaStreamSynchronize(ws.side);
    cudaStreamSynchronize(ws.stream);
    ws.side_pending = false;
    return rc;
  }
  if (n) CK(cudaMemcpyAsync(res->v, dres.v, 8 * n, cudaMemcpyDeviceToHost, ws.stream));
  if (nc) CK(cudaMemcpyAsync(res->lam, dres.lam, 24 * nc, cudaMemcpyDeviceToHost, ws.stream));
  if (res->residual_trace && cfg->max_iters > 0)
    CK(cudaMemcpyAsync(res->residual_trace, dres.residual_trace, 8 * (size_t)cfg->max_iters, cudaMemcpyDeviceToHost,
                       ws.stream));
  if (res->scc && nc) CK(cudaMemcpyAsync(res->scc, dres.scc, 8 * nc, cudaMemcpyDeviceToHost, ws.stream));
  if (res->w && n) CK(cudaMemcpyAsync(res->w, dres.w, 8 * n, cudaMemcpyDeviceToHost, ws.stream));
  // the copies above are ordered after ev[3] on the same stream
  CK(cudaStreamSynchronize(ws.stream));
  rc = vfpi_wait(h, &dres);
  res->iterations = dres.iterations;
  res->converged = dres.converged;
  res->diverged = dres.diverged;
  res->consistency = dres.consistency;
  res->setup_ms = dres.setup_ms;
  res->loop_ms = dres.loop_ms;
  res->status = rc;
  return rc;
}

}  // extern "C" (reopened below)

// Scene-batch solve on device arrays (system, scene pointers, warm start and
// outputs all on the device). Returns per-scene status in `stat` (host) after
// one stream synchronisation.
int vfpi_scenes_core(vfpi_handle* h, const vfpi_system& d, int S, const int32_t* d_scene_rows,
                     const int32_t* d_scene_cts, const vfpi_config* cfg, const double* d_warm, const double* d_wc,
                     double* d_out_v, double* d_out_lam, double* d_trace, double* d_scc, vfpi::SolveStatus* h_stat,
                     cudaStream_t st, float* setup_ms, float* loop_ms, int refresh_max_ct = -1,
                     const vfpi::NodeLayoutDev* nodes = nullptr) {
  // refresh_max_ct >= 0: the workspace holds this batch's contact-free row
  // layout (FEM pipeline); only the contact marks are rebuilt, and
  // refresh_max_ct is the largest per-scene contact count
  Workspace& ws = h->ws;
  const int n = (int)d.n, n_c = (int)d.n_c;
  const bool cheb = cfg->chebyshev != 0;
  const bool bb = cfg->step_strategy >= VFPI_STEP_BB1 && cfg->step_strategy <= VFPI_STEP_BB_ALTERNATING;
  int rc;
  CK(cudaEventRecord(ws.ev[0], st));
  vfpi::LayoutOptions opt;
  opt.anchor_order = false;
  opt.length_sort = h->layout_opt.length_sort;
  opt.scene_row_ptr = d_scene_rows;
  opt.scene_ct_ptr = d_scene_cts;
  vfpi::SetupSummary* hs = ws.h_summary;
  const int G = S;
  if (refresh_max_ct < 0) {
    rc = vfpi::setup_layout(ws, d, G, st, hs, h->err, h->launches, opt);
    if (rc) return rc;
    rc = vfpi::setup_pack(ws, d, G, false, *hs, st, h->err, h->launches);
    if (rc) return rc;
  } else {
    rc = vfpi::setup_contacts_refresh(ws, d, G, d_scene_cts, st, h->err, h->launches);
    if (rc) return rc;
  }
  rc = vfpi::setup_step_matrix(ws, d, *cfg, d_wc, st, h->err, h->launches);
  if (rc) return rc;
  const int max_ct = refresh_max_ct < 0 ? hs->max_ct_per_blk : refresh_max_ct;
  const int smem = 2 * vfpi::kSlotsPerContact * 8 * max_ct;
  if (vfpi::iterate_max_blocks_per_sm(cfg->op, cheb, bb, smem, true) <= 0) {
    h->err = "a scene has too many contacts for one CTA";
    return VFPI_UNSUPPORTED;
  }
  const size_t tr = (size_t)std::max(cfg->max_iters, 1);
  const size_t npad = (((size_t)std::max(n, 1) + 3) / 4) * 4 + 4;
  CK(vfpi::ensure(ws.vbuf, 3 * 8 * npad));
  CK(cudaMemsetAsync(ws.vbuf.p, 0, 3 * 8 * npad, st));
  CK(vfpi::ensure(ws.lambuf, 2 * 24 * (size_t)std::max(n_c, 1)));
  CK(vfpi::ensure(ws.status, sizeof(vfpi::SolveStatus) * (size_t)S));
  if (!d_trace) {
    CK(vfpi::ensure(ws.b_trace, 8 * tr * (size_t)S));
    d_trace = P<double>(ws.b_trace);
  }
  double* vb = P<double>(ws.vbuf);
  double* lb = P<double>(ws.lambuf);
  if (n > 0) {
    CK(cudaMemcpyAsync(vb, d_warm, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(vb + 2 * npad, d_warm, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaMemsetAsync(lb, 0, 2 * 24 * (size_t)std::max(n_c, 1), st));
  CK(cudaMemsetAsync(ws.status.p, 0, sizeof(vfpi::SolveStatus) * (size_t)S, st));
  CK(cudaEventRecord(ws.ev[1], st));
  vfpi::IterParams p{};
  p.n = n;
  p.n_c = n_c;
  p.G = G;
  p.row_list = P<int>(ws.row_list);
  p.row_slot = P<int>(ws.row_slot);
  p.blk_row = P<int>(ws.blk_row);
  p.blk_slice = P<int>(ws.blk_slice);
  p.blk_ct = P<int>(ws.blk_ct);
  p.slice_off = P<int64_t>(ws.slice_off);
  p.sell_val = P<double>(ws.sell_val);
  p.sell_col = P<int>(ws.sell_col);
  p.cont_list = P<int>(ws.cont_list);
  p.b = d.b;
  p.w = P<double>(ws.w);
  p.gamma = P<double>(ws.gamma);
  p.col_i = d.col_i;
  p.col_j = d.col_j;
  p.frames = d.frames;
  p.mu = d.mu;
  p.mu2 = d.mu2;
  p.phi = d.phi;
  p.w_mean = P<double>(ws.w_mean);
  p.diag = P<double>(ws.diag);
  p.fixed_alpha_default = (cfg->step_strategy == VFPI_STEP_FIXED_ALPHA && std::isnan(cfg->fixed_alpha)) ? 1 : 0;
  p.vbuf0 = vb;
  p.vbuf1 = vb + npad;
  p.vbuf2 = vb + 2 * npad;
  p.lam0 = lb;
  p.lam1 = lb + 3 * (size_t)std::max(n_c, 1);
  p.trace = d_trace;
  p.trace_stride = tr;
  p.status = P<vfpi::SolveStatus>(ws.status);
  p.out_v = d_out_v;
  p.out_lam = d_out_lam;
  p.max_iters = cfg->max_iters;
  p.cheby_start = cfg->cheby_start;
  p.step = cfg->step_strategy;
  p.tol = cfg->residual_tol;
  p.under_relax = cfg->under_relax;
  p.omega = cfg->omega;
  p.cfactor = cfg->consistency_factor;
  const int nmode = (nodes && nodes->cluster > 1) ? 2 : 0;  // one CTA or one cluster per scene
  const bool use_nodes = nodes && !bb && h->node_kernel &&
                         vfpi::node_kernel_blocks_per_sm(cfg->op, cheb, std::max(max_ct, 1), nmode) > 0;
  if (use_nodes) {
    if (vfpi::node_slots_refresh(*nodes, S, n_c, d.col_i, d.col_j, nullptr, st)) {
      h->err = "node slot refresh failed";
      return VFPI_CUDA_ERROR;
    }
    ++h->launches;
    CK(cudaEventRecord(ws.ev[1], st));  // the loop timing covers the iteration kernel only
    rc = vfpi::launch_iterate_nodes(p, *nodes, cfg->op, cheb, std::max(max_ct, 1), st, h->err, nmode);
    if (rc == VFPI_OK && nodes->scene_perm) {  // next solve: longest predicted scenes first
      vfpi::launch_scene_order(S, P<vfpi::SolveStatus>(ws.status), const_cast<int*>(nodes->scene_perm), st);
      ++h->launches;
    }
  } else {
    rc = vfpi::launch_iterate_scenes(p, cfg->op, cheb, bb, smem, st, h->err);
  }
  if (rc) return rc;
  ++h->launches;
  h->last_node_kernel = use_nodes ? 1 : 0;
  CK(cudaEventRecord(ws.ev[2], st));
  if (d_scc && n_c > 0) {
    rc = vfpi::launch_scc_final(p, d_scc, st);
    if (rc) { h->err = "scc kernel launch failed"; return rc; }
    ++h->launches;
  }
  CK(cudaMemcpyAsync(h_stat, ws.status.p, sizeof(vfpi::SolveStatus) * (size_t)S, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->h_flags, ws.flags.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float a = 0.f, b2 = 0.f;
  cudaEventElapsedTime(&a, ws.ev[0], ws.ev[1]);
  cudaEventElapsedTime(&b2, ws.ev[1], ws.ev[2]);
  if (setup_ms) *setup_ms = a;
  if (loop_ms) *loop_ms = b2;
  return flags_to_code(h, *h->h_flags);
}

extern "C" {

int vfpi_solve_scenes(vfpi_handle* h, const vfpi_system* s, int32_t S, const int32_t* scene_row_ptr,
                      const int32_t* scene_ct_ptr, const vfpi_config* cfg, const double* warm,
                      const double* w_cached, vfpi_scene_result* res) {
  if (!h || !cfg || !res || !warm || !scene_row_ptr || !scene_ct_ptr || S < 1 || S > 1024) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  if (scene_row_ptr[0] != 0 || scene_row_ptr[S] != s->n || scene_ct_ptr[0] != 0 || scene_ct_ptr[S] != s->n_c) {
    h->err = "scene pointers do not cover the system";
    return VFPI_BAD_ARGUMENT;
  }
  for (int k = 0; k < S; ++k)
    if (scene_row_ptr[k + 1] < scene_row_ptr[k] || scene_ct_ptr[k + 1] < scene_ct_ptr[k]) {
      h->err = "scene pointers must be non-decreasing";
      return VFPI_BAD_ARGUMENT;
    }
  if (cfg->op < 0 || cfg->op > 2 || cfg->step_strategy < 0 || cfg->step_strategy > 4 || cfg->max_iters < 0) {
    h->err = "bad solver config";
    return VFPI_BAD_ARGUMENT;
  }
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  Workspace& ws = h->ws;
  cudaStream_t st = ws.stream;
  const int n = (int)s->n, n_c = (int)s->n_c;
  vfpi_system d;
  if ((rc = stage_system(h, s, &d))) return rc;
  if ((rc = upload(h, ws.b_warm, warm, 8 * (size_t)n))) return rc;
  CK(vfpi::ensure(ws.b_warm, 8 * (size_t)std::max(n, 1)));
  const double* dwc = nullptr;
  if (w_cached) {
    if ((rc = upload(h, ws.b_wc, w_cached, 8 * (size_t)n))) return rc;
    dwc = P<double>(ws.b_wc);
  }
  if ((rc = upload(h, ws.scene_rows, scene_row_ptr, 4 * (size_t)(S + 1)))) return rc;
  if ((rc = upload(h, ws.scene_cts, scene_ct_ptr, 4 * (size_t)(S + 1)))) return rc;
  const size_t tr = (size_t)std::max(cfg->max_iters, 1);
  CK(vfpi::ensure(ws.b_out_v, 8 * (size_t)std::max(n, 1)));
  CK(vfpi::ensure(ws.b_out_lam, 24 * (size_t)std::max(n_c, 1)));
  CK(vfpi::ensure(ws.b_trace, 8 * tr * (size_t)S));
  CK(vfpi::ensure(ws.b_scc, 8 * (size_t)std::max(n_c, 1)));
  std::vector<vfpi::SolveStatus> stat((size_t)S);
  float su = 0.f, lo = 0.f;
  rc = vfpi_scenes_core(h, d, S, P<int32_t>(ws.scene_rows), P<int32_t>(ws.scene_cts), cfg, P<double>(ws.b_warm),
                        dwc, P<double>(ws.b_out_v), P<double>(ws.b_out_lam), P<double>(ws.b_trace),
                        res->scc ? P<double>(ws.b_scc) : nullptr, stat.data(), st, &su, &lo);
  if (rc) return rc;
  if (n) CK(cudaMemcpyAsync(res->v, ws.b_out_v.p, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
  if (n_c) CK(cudaMemcpyAsync(res->lam, ws.b_out_lam.p, 24 * (size_t)n_c, cudaMemcpyDeviceToHost, st));
  if (res->residual_trace && cfg->max_iters > 0)
    CK(cudaMemcpyAsync(res->residual_trace, ws.b_trace.p, 8 * tr * (size_t)S, cudaMemcpyDeviceToHost, st));
  if (res->scc && n_c) CK(cudaMemcpyAsync(res->scc, ws.b_scc.p, 8 * (size_t)n_c, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int k = 0; k < S; ++k) {
    if (res->iterations) res->iterations[k] = stat[k].iterations;
    if (res->converged) res->converged[k] = stat[k].converged;
    if (res->diverged) res->diverged[k] = stat[k].diverged;
    if (res->consistency) res->consistency[k] = stat[k].consistency;
  }
  res->setup_ms = su;
  res->loop_ms = lo;
  return VFPI_OK;
}

// ---- per-subsystem entry points -------------------------------------------

int vfpi_spmv(vfpi_handle* h, const vfpi_system* s, const double* x, double* y) {
  if (!h || !x || !y) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  vfpi_system d, s0 = *s;
  s0.n_c = 0;
  if ((rc = stage_system(h, &s0, &d))) return rc;
  const size_t n = (size_t)s->n;
  if ((rc = upload(h, ws.x, x, 8 * n))) return rc;
  CK(vfpi::ensure(ws.y, 8 * std::max<size_t>(n, 1)));
  if ((rc = op_layout(h, d, false))) return rc;
  vfpi::launch_spmv_csr_rows((int64_t)n, P<int64_t>(ws.row_ptr), P<int>(ws.perm), P<int>(ws.colof), d.data,
                             P<double>(ws.x), P<double>(ws.y), ws.stream);
  ++h->launches;
  CK(cudaGetLastError());
  if (n) CK(cudaMemcpyAsync(y, ws.y.p, 8 * n, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}

static int stats_op(vfpi_handle* h, const vfpi_system* s, double* out, bool rns) {
  if (!h || !out) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  vfpi_system d, s0 = *s;
  s0.n_c = 0;
  if ((rc = stage_system(h, &s0, &d))) return rc;
  if ((rc = op_layout(h, d, false))) return rc;
  const size_t n = (size_t)s->n;
  if (n) CK(cudaMemcpyAsync(out, rns ? h->ws.rns.p : h->ws.diag.p, 8 * n, cudaMemcpyDeviceToHost, h->ws.stream));
  CK(cudaStreamSynchronize(h->ws.stream));
  return VFPI_OK;
}

int vfpi_row_norms_sq(vfpi_handle* h, const vfpi_system* s, double* out) { return stats_op(h, s, out, true); }
int vfpi_diagonal(vfpi_handle* h, const vfpi_system* s, double* out) { return stats_op(h, s, out, false); }

int vfpi_step_matrix_frobenius(vfpi_handle* h, const vfpi_system* s, int pair_tie, double* w) {
  if (!h || !w) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  vfpi_system d;
  if ((rc = stage_system(h, s, &d))) return rc;
  if ((rc = op_layout(h, d, true))) return rc;
  vfpi_config cfg{};
  cfg.op = pair_tie ? VFPI_OP_PROXIMAL : VFPI_OP_STRICT;
  cfg.step_strategy = VFPI_STEP_FROBENIUS;
  if ((rc = vfpi::setup_step_matrix(h->ws, d, cfg, nullptr, h->ws.stream, h->err, h->launches))) return rc;
  const size_t n = (size_t)s->n;
  if (n) CK(cudaMemcpyAsync(w, h->ws.w.p, 8 * n, cudaMemcpyDeviceToHost, h->ws.stream));
  CK(cudaMemcpyAsync(h->h_flags, h->ws.flags.p, 4, cudaMemcpyDeviceToHost, h->ws.stream));
  CK(cudaStreamSynchronize(h->ws.stream));
  return flags_to_code(h, *h->h_flags);
}

int vfpi_surrogate_gamma(vfpi_handle* h, const vfpi_system* s, const double* w, double omega, double* gamma) {
  if (!h || !w || !gamma) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  vfpi_system d;
  if ((rc = stage_system(h, s, &d))) return rc;
  if ((rc = upload(h, h->ws.b_wc, w, 8 * (size_t)s->n))) return rc;
  vfpi_config cfg{};
  cfg.op = VFPI_OP_STRICT;
  cfg.step_strategy = VFPI_STEP_FROBENIUS;
  cfg.omega = omega;
  CK(vfpi::ensure(h->ws.flags, 16));
  CK(cudaMemsetAsync(h->ws.flags.p, 0, 16, h->ws.stream));
  if ((rc = vfpi::setup_step_matrix(h->ws, d, cfg, P<double>(h->ws.b_wc), h->ws.stream, h->err, h->launches)))
    return rc;
  const size_t nc = (size_t)s->n_c;
  if (nc) CK(cudaMemcpyAsync(gamma, h->ws.gamma.p, 8 * nc, cudaMemcpyDeviceToHost, h->ws.stream));
  CK(cudaMemcpyAsync(h->h_flags, h->ws.flags.p, 4, cudaMemcpyDeviceToHost, h->ws.stream));
  CK(cudaStreamSynchronize(h->ws.stream));
  return flags_to_code(h, *h->h_flags);
}

int vfpi_apply_jc(vfpi_handle* h, const vfpi_system* s, const double* v, double* eta) {
  if (!h || !v || !eta) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  const size_t n = (size_t)s->n, nc = (size_t)s->n_c;
  if ((rc = upload(h, ws.b_ci, s->col_i, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_cj, s->col_j, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_frames, s->frames, 72 * nc))) return rc;
  if ((rc = upload(h, ws.x, v, 8 * n))) return rc;
  CK(vfpi::ensure(ws.y, 24 * std::max<size_t>(nc, 1)));
  vfpi::launch_apply_jc((int64_t)nc, P<int>(ws.b_ci), P<int>(ws.b_cj), P<double>(ws.b_frames), P<double>(ws.x),
                        P<double>(ws.y), ws.stream);
  ++h->launches;
  CK(cudaGetLastError());
  if (nc) CK(cudaMemcpyAsync(eta, ws.y.p, 24 * nc, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}

int vfpi_apply_jc_t(vfpi_handle* h, const vfpi_system* s, const double* lam, double* out) {
  if (!h || !lam || !out) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  const size_t n = (size_t)s->n, nc = (size_t)s->n_c;
  // column overlap decides between the parallel scatter and the ordered one
  bool overlap = false;
  {
    std::vector<unsigned char> used(n + 3, 0);
    for (size_t m = 0; m < nc && !overlap; ++m) {
      const int cols[2] = {s->col_i[m], s->col_j[m]};
      for (int c : cols) {
        if (c < 0) continue;
        if ((size_t)c + 3 > n) { h->err = "contact column out of range"; return VFPI_BAD_ARGUMENT; }
        for (int t = 0; t < 3; ++t) {
          if (used[c + t]) overlap = true;
          used[c + t] = 1;
        }
      }
    }
  }
  if ((rc = upload(h, ws.b_ci, s->col_i, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_cj, s->col_j, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_frames, s->frames, 72 * nc))) return rc;
  if ((rc = upload(h, ws.x, lam, 24 * nc))) return rc;
  CK(vfpi::ensure(ws.y, 8 * std::max<size_t>(n, 1)));
  vfpi::launch_apply_jc_t((int64_t)n, (int64_t)nc, P<int>(ws.b_ci), P<int>(ws.b_cj), P<double>(ws.b_frames),
                          P<double>(ws.x), P<double>(ws.y), overlap, ws.stream);
  ++h->launches;
  CK(cudaGetLastError());
  if (n) CK(cudaMemcpyAsync(out, ws.y.p, 8 * n, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}

int vfpi_contact_solve_oneshot(vfpi_handle* h, int64_t n_c, const double* gamma, const double* eta,
                               const double* phi, const double* mu, const double* mu2, int op, double* lam) {
  if (!h || n_c < 0 || op < 0 || op > 2) return VFPI_BAD_ARGUMENT;
  if (n_c == 0) return VFPI_OK;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  const size_t nc = (size_t)n_c;
  int rc;
  if ((rc = upload(h, ws.gamma, gamma, 8 * nc))) return rc;
  if ((rc = upload(h, ws.x, eta, 24 * nc))) return rc;
  if ((rc = upload(h, ws.b_phi, phi, 8 * nc))) return rc;
  if ((rc = upload(h, ws.b_mu, mu, 8 * nc))) return rc;
  if ((rc = upload(h, ws.b_mu2, mu2 ? mu2 : mu, 8 * nc))) return rc;
  CK(vfpi::ensure(ws.y, 24 * nc));
  vfpi::launch_oneshot(n_c, P<double>(ws.gamma), P<double>(ws.x), P<double>(ws.b_phi), P<double>(ws.b_mu),
                       P<double>(ws.b_mu2), op, P<double>(ws.y), ws.stream);
  ++h->launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(lam, ws.y.p, 24 * nc, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}

int vfpi_scc_residual(vfpi_handle* h, int64_t n_c, const double* vc, const double* lam, const double* phi,
                      const double* mu, double* out) {
  if (!h || n_c < 0) return VFPI_BAD_ARGUMENT;
  if (n_c == 0) return VFPI_OK;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  const size_t nc = (size_t)n_c;
  int rc;
  if ((rc = upload(h, ws.x, vc, 24 * nc))) return rc;
  if ((rc = upload(h, ws.b_out_lam, lam, 24 * nc))) return rc;
  if ((rc = upload(h, ws.b_phi, phi, 8 * nc))) return rc;
  if ((rc = upload(h, ws.b_mu, mu, 8 * nc))) return rc;
  CK(vfpi::ensure(ws.y, 8 * nc));
  vfpi::launch_scc(n_c, P<double>(ws.x), P<double>(ws.b_out_lam), P<double>(ws.b_phi), P<double>(ws.b_mu),
                   P<double>(ws.y), ws.stream);
  ++h->launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, ws.y.p, 8 * nc, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}

int vfpi_inverse_contact(vfpi_handle* h, const vfpi_system* s, const double* v, double omega, int op, double* lam) {
  if (!h || !v || !lam || op < 0 || op > 2) return VFPI_BAD_ARGUMENT;
  int rc = check_system(h, s);
  if (rc) return rc;
  cudaSetDevice(h->ws.device);
  Workspace& ws = h->ws;
  const size_t n = (size_t)s->n, nc = (size_t)s->n_c;
  if (nc == 0) return VFPI_OK;
  if ((rc = upload(h, ws.b_ci, s->col_i, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_cj, s->col_j, 4 * nc))) return rc;
  if ((rc = upload(h, ws.b_frames, s->frames, 72 * nc))) return rc;
  if ((rc = upload(h, ws.b_phi, s->phi, 8 * nc))) return rc;
  if ((rc = upload(h, ws.b_mu, s->mu, 8 * nc))) return rc;
  if ((rc = upload(h, ws.b_mu2, s->mu2 ? s->mu2 : s->mu, 8 * nc))) return rc;
  if ((rc = upload(h, ws.x, v, 8 * n))) return rc;
  CK(vfpi::ensure(ws.y, 24 * nc));
  CK(vfpi::ensure(ws.gamma, 8 * nc));
  CK(vfpi::ensure(ws.b_out_lam, 24 * nc));
  vfpi::launch_const_fill(P<double>(ws.gamma), omega, (int64_t)nc, ws.stream);
  vfpi::launch_apply_jc((int64_t)nc, P<int>(ws.b_ci), P<int>(ws.b_cj), P<double>(ws.b_frames), P<double>(ws.x),
                        P<double>(ws.y), ws.stream);
  vfpi::launch_oneshot((int64_t)nc, P<double>(ws.gamma), P<double>(ws.y), P<double>(ws.b_phi), P<double>(ws.b_mu),
                       P<double>(ws.b_mu2), op, P<double>(ws.b_out_lam), ws.stream);
  h->launches += 3;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(lam, ws.b_out_lam.p, 24 * nc, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaStreamSynchronize(ws.stream));
  return VFPI_OK;
}


// ---- FEM scene batch stepped on the device ---------------------------------

}  // extern "C"

struct vfpi_fem_batch {
  vfpi_handle* h = nullptr;
  int S = 0, Nn = 0;      // scenes, nodes per scene
  int64_t n = 0, nodes = 0;
  vfpi_fem_params prm{};
  vfpi_system A{};        // device CSC of the block-diagonal A
  Workspace::Buf a_indptr, a_indices, a_data, krp, kc, kv, m, g, X, x, v, warm, vhat, lam, b, ci, cj, frames, mu,
      mu2, phi, flag, pos, cts, rows, frame, tmp;
  std::vector<int32_t> h_cts;
  std::vector<vfpi::SolveStatus> stat;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Workspace::Buf zero_cts, ks_off, ks_val, ks_col;  // K in SELL-32
  Workspace::Buf cg_r, cg_p, cg_q, cg_list;        // contact-free fallback of diverged scenes
  Workspace::Buf x0, v0;                           // initial state (vfpi_fem_reset)
  Workspace::Buf run_acc, run_its, run_cts;        // device counters of vfpi_fem_run
  std::vector<cudaEvent_t> run_ev;                 // per-step iteration-kernel events of vfpi_fem_run
  vfpi::NodeLayoutHost nbh;                        // node-block SELL layout (vfpi_fem_set_node_layout)
  vfpi::NodeLayoutDev nbd;
  bool nb_ready = false;
  Workspace::Buf kn_desc, kn_val;  // K on the node-block template (right-hand side)
  bool kn_ready = false;
  uint64_t layout_epoch = ~0ull;  // the handle workspace holds our contact-free layout
};

namespace {

// (1) of a FEM step: b = ((2/dt) m) v - K (x - X) + m g, K streamed as node
// blocks when the batch has its node layout, else as row SELL-32
void fem_rhs(vfpi_fem_batch* fb, double twodt, cudaStream_t st) {
  if (fb->nb_ready && fb->kn_ready)
    vfpi::launch_fem_rhs_nodes(fb->S, fb->Nn, fb->nbd.nsl, fb->nbd.slice_off, fb->nbd.node_list,
                               P<unsigned>(fb->kn_desc), P<double>(fb->kn_val), P<double>(fb->x), P<double>(fb->X),
                               P<double>(fb->v), P<double>(fb->m), P<double>(fb->g), twodt, P<double>(fb->b), st);
  else
    vfpi::launch_fem_rhs_sell(fb->n, P<int64_t>(fb->ks_off), P<double>(fb->ks_val), P<int>(fb->ks_col),
                              P<double>(fb->x), P<double>(fb->X), P<double>(fb->v), P<double>(fb->m), P<double>(fb->g),
                              twodt, P<double>(fb->b), st);
}

int fem_upload(vfpi_handle* h, Workspace::Buf& b, const void* src, size_t bytes) {
  CK(vfpi::ensure(b, std::max<size_t>(bytes, 8)));
  if (bytes) CK(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice));
  return VFPI_OK;
}

}  // namespace

extern "C" {

int vfpi_fem_create(vfpi_handle* h, int32_t S, int32_t Nn, const vfpi_system* a, const int64_t* k_rowptr,
                    const int32_t* k_cols, const double* k_vals, const double* mass, const double* gravity,
                    const double* rest_x, const double* x, const double* v, const double* frame9,
                    const vfpi_fem_params* prm, vfpi_fem_batch** out) {
  if (!h || !a || !k_rowptr || !k_cols || !k_vals || !mass || !gravity || !rest_x || !x || !v || !frame9 || !prm ||
      !out || S < 1 || S > 1024 || Nn < 1)
    return VFPI_BAD_ARGUMENT;
  if (a->n != (int64_t)S * 3 * Nn || a->n_c != 0) {
    h->err = "A must cover num_scenes * 3 * nodes_per_scene rows and carry no contacts";
    return VFPI_DIM_MISMATCH;
  }
  int rc = check_system(h, a);
  if (rc) return rc;
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  auto* fb = new vfpi_fem_batch();
  fb->h = h;
  fb->S = S;
  fb->Nn = Nn;
  fb->n = a->n;
  fb->nodes = (int64_t)S * Nn;
  fb->prm = *prm;
  const size_t n = (size_t)fb->n, nodes = (size_t)fb->nodes, nnz = (size_t)a->nnz, knnz = (size_t)k_rowptr[n];
  auto fail = [&](int code) { vfpi_fem_destroy(fb); return code; };
  if ((rc = fem_upload(h, fb->a_indptr, a->indptr, 4 * (n + 1))) || (rc = fem_upload(h, fb->a_indices, a->indices, 4 * nnz)) ||
      (rc = fem_upload(h, fb->a_data, a->data, 8 * nnz)) || (rc = fem_upload(h, fb->krp, k_rowptr, 8 * (n + 1))) ||
      (rc = fem_upload(h, fb->kc, k_cols, 4 * knnz)) || (rc = fem_upload(h, fb->kv, k_vals, 8 * knnz)) ||
      (rc = fem_upload(h, fb->m, mass, 8 * n)) || (rc = fem_upload(h, fb->g, gravity, 8 * n)) ||
      (rc = fem_upload(h, fb->X, rest_x, 8 * n)) || (rc = fem_upload(h, fb->x, x, 8 * n)) ||
      (rc = fem_upload(h, fb->v, v, 8 * n)) || (rc = fem_upload(h, fb->frame, frame9, 72)))
    return fail(rc);
  if (vfpi::ensure(fb->x0, 8 * n) || vfpi::ensure(fb->v0, 8 * n) ||
      cudaMemcpy(fb->x0.p, fb->x.p, 8 * n, cudaMemcpyDeviceToDevice) ||
      cudaMemcpy(fb->v0.p, fb->v.p, 8 * n, cudaMemcpyDeviceToDevice))
    return fail(VFPI_CUDA_ERROR);
  for (Workspace::Buf* bb : {&fb->warm, &fb->vhat, &fb->b}) {
    if (vfpi::ensure(*bb, 8 * n) != cudaSuccess) return fail(VFPI_CUDA_ERROR);
  }
  if (cudaMemset(fb->warm.p, 0, 8 * n) != cudaSuccess) return fail(VFPI_CUDA_ERROR);
  // contact arrays sized for every node in contact
  if (vfpi::ensure(fb->lam, 24 * nodes) || vfpi::ensure(fb->ci, 4 * nodes) || vfpi::ensure(fb->cj, 4 * nodes) ||
      vfpi::ensure(fb->frames, 72 * nodes) || vfpi::ensure(fb->mu, 8 * nodes) || vfpi::ensure(fb->mu2, 8 * nodes) ||
      vfpi::ensure(fb->phi, 8 * nodes) || vfpi::ensure(fb->pos, 4 * nodes) ||
      vfpi::ensure(fb->cts, 4 * (size_t)(S + 1)))
    return fail(VFPI_CUDA_ERROR);
  std::vector<int32_t> rows((size_t)S + 1);
  for (int k = 0; k <= S; ++k) rows[k] = k * 3 * Nn;
  if ((rc = fem_upload(h, fb->rows, rows.data(), 4 * (size_t)(S + 1)))) return fail(rc);
  std::vector<int32_t> zeros((size_t)S + 1, 0);
  if ((rc = fem_upload(h, fb->zero_cts, zeros.data(), 4 * (size_t)(S + 1)))) return fail(rc);
  const size_t tb = vfpi::fem_detect_tmp_bytes((int64_t)nodes);
  if (vfpi::ensure(fb->tmp, std::max<size_t>(tb, 16))) return fail(VFPI_CUDA_ERROR);
  {  // K -> SELL-32 once (coalesced right-hand-side sums)
    const int64_t nsl = ((int64_t)n + 31) / 32;
    if (vfpi::ensure(fb->ks_off, 8 * (size_t)(nsl + 1))) return fail(VFPI_CUDA_ERROR);
    Workspace::Buf wbuf;
    if (vfpi::ensure(wbuf, 8 * (size_t)(nsl + 1))) return fail(VFPI_CUDA_ERROR);
    vfpi::launch_fem_sell_width((int64_t)n, P<int64_t>(fb->krp), P<int64_t>(wbuf), nullptr);
    size_t t2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t2, P<int64_t>(wbuf), P<int64_t>(fb->ks_off), (int)(nsl + 1));
    Workspace::Buf tb2;
    if (vfpi::ensure(tb2, t2) ||
        cub::DeviceScan::ExclusiveSum(tb2.p, t2, P<int64_t>(wbuf), P<int64_t>(fb->ks_off), (int)(nsl + 1))) {
      vfpi::dev_free(wbuf.p);
      vfpi::dev_free(tb2.p);
      return fail(VFPI_CUDA_ERROR);
    }
    int64_t elems = 0;
    cudaMemcpy(&elems, P<int64_t>(fb->ks_off) + nsl, 8, cudaMemcpyDeviceToHost);
    vfpi::dev_free(wbuf.p);
    vfpi::dev_free(tb2.p);
    if (vfpi::ensure(fb->ks_val, 8 * (size_t)std::max<int64_t>(elems, 1)) ||
        vfpi::ensure(fb->ks_col, 4 * (size_t)std::max<int64_t>(elems, 1)))
      return fail(VFPI_CUDA_ERROR);
    vfpi::launch_fem_sell_pack((int64_t)n, P<int64_t>(fb->krp), P<int>(fb->kc), P<double>(fb->kv),
                               P<int64_t>(fb->ks_off), P<double>(fb->ks_val), P<int>(fb->ks_col), nullptr);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(VFPI_CUDA_ERROR);
  }
  fb->A = *a;
  fb->A.indptr = (const int32_t*)fb->a_indptr.p;
  fb->A.indices = (const int32_t*)fb->a_indices.p;
  fb->A.data = (const double*)fb->a_data.p;
  fb->h_cts.resize((size_t)S + 1);
  fb->stat.resize((size_t)S);
  if (cudaEventCreate(&fb->e0) != cudaSuccess || cudaEventCreate(&fb->e1) != cudaSuccess) return fail(VFPI_CUDA_ERROR);
  *out = fb;
  return VFPI_OK;
}

}  // extern "C"

namespace {

// A's contact-free row layout + column statistics (diagonal, squared row norms
// for W), built once per batch and whenever another solve used the workspace
int fem_contact_free_layout(vfpi_fem_batch* fb) {
  vfpi_handle* h = fb->h;
  Workspace& ws = h->ws;
  cudaStream_t st = ws.stream;
  vfpi_system d0 = fb->A;
  d0.n_c = 0;
  d0.b = P<double>(fb->b);
  d0.col_i = P<int32_t>(fb->ci);
  d0.col_j = P<int32_t>(fb->cj);
  d0.frames = P<double>(fb->frames);
  d0.mu = P<double>(fb->mu);
  d0.mu2 = P<double>(fb->mu2);
  d0.phi = P<double>(fb->phi);
  vfpi::LayoutOptions opt;
  opt.anchor_order = false;
  opt.length_sort = h->layout_opt.length_sort;
  opt.scene_row_ptr = P<int>(fb->rows);
  opt.scene_ct_ptr = P<int>(fb->zero_cts);
  int rc0 = vfpi::setup_layout(ws, d0, fb->S, st, ws.h_summary, h->err, h->launches, opt);
  if (!rc0) rc0 = vfpi::setup_pack(ws, d0, fb->S, false, *ws.h_summary, st, h->err, h->launches);
  if (!rc0) rc0 = vfpi::setup_rowpos(ws, (int)fb->n, fb->S, st, h->err);
  if (rc0) return rc0;
  CK(vfpi::ensure(ws.cont_list, 4 * (size_t)fb->nodes));  // per-step refresh never grows it
  CK(cudaStreamSynchronize(st));
  fb->layout_epoch = ws.layout_epoch;
  return VFPI_OK;
}

}  // namespace

extern "C" {

int vfpi_fem_step(vfpi_fem_batch* fb, const vfpi_config* cfg, vfpi_fem_step_stats* stats,
                  int32_t* iterations_per_scene) {
  if (!fb || !cfg || !stats) return VFPI_BAD_ARGUMENT;
  vfpi_handle* h = fb->h;
  if (cfg->op < 0 || cfg->op > 2 || cfg->step_strategy < 0 || cfg->step_strategy > 4 || cfg->max_iters < 0) {
    h->err = "bad solver config";
    return VFPI_BAD_ARGUMENT;
  }
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  cudaStream_t st = h->ws.stream;
  const vfpi_fem_params& q = fb->prm;
  CK(cudaEventRecord(fb->e0, st));
  // (1) right-hand side of every scene
  fem_rhs(fb, 2.0 / q.dt, st);
  // (2) node-plane contacts: flags, scene-ordered compaction, parameters
  if (vfpi::launch_fem_detect(fb->nodes, fb->S, fb->Nn, P<double>(fb->x), P<double>(fb->v), q.margin, fb->tmp.p,
                              fb->tmp.cap, P<int>(fb->pos), P<int>(fb->cts), P<double>(fb->frame), q.mu,
                              -(q.beta_err / q.dt), q.e_rest, q.rest_threshold, P<int>(fb->ci), P<int>(fb->cj),
                              P<double>(fb->frames), P<double>(fb->mu), P<double>(fb->mu2), P<double>(fb->phi),
                              nullptr, nullptr, st)) {
    h->err = "node-plane detection launch failed";
    return VFPI_CUDA_ERROR;
  }
  h->launches += 4;  // rhs, scan (init + pass), detection
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(fb->h_cts.data(), fb->cts.p, 4 * (size_t)(fb->S + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // (3) solve every scene (vfpi_solve_scenes semantics, warm = previous solution);
  // A is fixed, so its row layout is built once without contacts and only the
  // contact marks are refreshed per step (rebuilt if another solve used the workspace)
  Workspace& ws = h->ws;
  // (layout buffers are only (re)allocated inside setup_layout/setup_pack, which
  // bump the epoch; growth of unrelated workspace buffers leaves them intact)
  if (fb->layout_epoch != ws.layout_epoch) {
    const int rc0 = fem_contact_free_layout(fb);
    if (rc0) return rc0;
  }
  int max_ct = 0;
  for (int k = 0; k < fb->S; ++k) max_ct = std::max(max_ct, fb->h_cts[k + 1] - fb->h_cts[k]);
  vfpi_system d = fb->A;
  d.n_c = fb->h_cts[fb->S];
  d.b = P<double>(fb->b);
  d.col_i = P<int32_t>(fb->ci);
  d.col_j = P<int32_t>(fb->cj);
  d.frames = P<double>(fb->frames);
  d.mu = P<double>(fb->mu);
  d.mu2 = P<double>(fb->mu2);
  d.phi = P<double>(fb->phi);
  float su = 0.f, lo = 0.f;
  int rc = vfpi_scenes_core(h, d, fb->S, P<int32_t>(fb->rows), P<int32_t>(fb->cts), cfg, P<double>(fb->warm),
                            nullptr, P<double>(fb->vhat), P<double>(fb->lam), nullptr, nullptr, fb->stat.data(), st,
                            &su, &lo, max_ct, fb->nb_ready ? &fb->nbd : nullptr);
  if (rc) return rc;
  // (3b) diverged scenes take the flagged contact-free step (harness.py:586-593):
  // v_hat = cg(A, b, rtol=1e-10, maxiter=10 n) of the scene, lam = 0
  {
    std::vector<int32_t> div;
    for (int k = 0; k < fb->S; ++k)
      if (fb->stat[k].diverged) div.push_back(k);
    if (!div.empty()) {
      const size_t n = (size_t)fb->n;
      CK(vfpi::ensure(fb->cg_r, 8 * n));
      CK(vfpi::ensure(fb->cg_p, 8 * n));
      CK(vfpi::ensure(fb->cg_q, 8 * n));
      CK(vfpi::ensure(fb->cg_list, 4 * (size_t)fb->S));
      CK(cudaMemcpyAsync(fb->cg_list.p, div.data(), 4 * div.size(), cudaMemcpyHostToDevice, st));
      const int64_t ns = 3 * (int64_t)fb->Nn;
      if (vfpi::launch_cg_scenes((int)div.size(), P<int32_t>(fb->cg_list), ns, fb->A.indptr, fb->A.indices,
                                 fb->A.data, P<double>(fb->b), P<double>(fb->vhat), P<double>(fb->cg_r),
                                 P<double>(fb->cg_p), P<double>(fb->cg_q), 1e-10, 10 * ns, nullptr, st)) {
        h->err = "fallback CG launch failed";
        return VFPI_CUDA_ERROR;
      }
      ++h->launches;
      for (int k : div) {
        const int c0 = fb->h_cts[k], c1 = fb->h_cts[k + 1];
        if (c1 > c0) CK(cudaMemsetAsync(P<double>(fb->lam) + 3 * (size_t)c0, 0, 24 * (size_t)(c1 - c0), st));
      }
      CK(cudaStreamSynchronize(st));  // `div` is a host buffer of the async copy
    }
  }
  // (4) midpoint integration; the solution warm-starts the next step
  vfpi::launch_fem_advance(fb->n, q.dt, P<double>(fb->vhat), P<double>(fb->x), P<double>(fb->v),
                           P<double>(fb->warm), st);
  ++h->launches;
  CK(cudaGetLastError());
  CK(cudaEventRecord(fb->e1, st));
  CK(cudaEventSynchronize(fb->e1));
  int64_t ci = 0, it = 0;
  int mx = 0, dv = 0;
  for (int k = 0; k < fb->S; ++k) {
    const vfpi::SolveStatus& s = fb->stat[k];
    ci += (int64_t)(fb->h_cts[k + 1] - fb->h_cts[k]) * s.iterations;
    it += s.iterations;
    mx = std::max(mx, s.iterations);
    dv += s.diverged ? 1 : 0;
    if (iterations_per_scene) iterations_per_scene[k] = s.iterations;
  }
  float step = 0.f;
  cudaEventElapsedTime(&step, fb->e0, fb->e1);
  stats->contacts = d.n_c;
  stats->contact_iterations = ci;
  stats->iterations = it;
  stats->max_iterations = mx;
  stats->diverged_scenes = dv;
  stats->setup_ms = su;
  stats->loop_ms = lo;
  stats->step_ms = step;
  return VFPI_OK;
}

int vfpi_fem_run(vfpi_fem_batch* fb, const vfpi_config* cfg, int32_t steps, vfpi_fem_run_stats* stats,
                 int32_t* iterations, int32_t* contacts) {
  if (!fb || !cfg || !stats || steps < 0) return VFPI_BAD_ARGUMENT;
  vfpi_handle* h = fb->h;
  if (cfg->op < 0 || cfg->op > 2 || cfg->step_strategy < 0 || cfg->step_strategy > 4 || cfg->max_iters < 0) {
    h->err = "bad solver config";
    return VFPI_BAD_ARGUMENT;
  }
  std::memset(stats, 0, sizeof(*stats));
  const bool cheb = cfg->chebyshev != 0;
  const bool bb = cfg->step_strategy >= VFPI_STEP_BB1 && cfg->step_strategy <= VFPI_STEP_BB_ALTERNATING;
  const int nmode = fb->nb_ready && fb->nbd.cluster > 1 ? 2 : 0;
  if (!fb->nb_ready || bb || !h->node_kernel || vfpi::node_kernel_blocks_per_sm(cfg->op, cheb, 1, nmode) <= 0) {
    // the per-step path (host reads of the contact counts each step)
    for (int k = 0; k < steps; ++k) {
      vfpi_fem_step_stats s{};
      std::vector<int32_t> its(iterations ? (size_t)fb->S : 0);
      const int rc = vfpi_fem_step(fb, cfg, &s, iterations ? its.data() : nullptr);
      if (rc) return rc;
      if (iterations) std::memcpy(iterations + (size_t)k * fb->S, its.data(), 4 * (size_t)fb->S);
      if (contacts) contacts[k] = (int32_t)s.contacts;
      stats->contacts += s.contacts;
      stats->contact_iterations += s.contact_iterations;
      stats->iterations += s.iterations;
      stats->max_iterations = std::max(stats->max_iterations, s.max_iterations);
      stats->diverged_scene_steps += s.diverged_scenes;
      stats->loop_ms += s.loop_ms;
      stats->run_ms += s.step_ms;
    }
    stats->host_synced = 1;
    return VFPI_OK;
  }
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  cudaStream_t st = h->ws.stream;
  Workspace& ws = h->ws;
  const vfpi_fem_params& q = fb->prm;
  const int S = fb->S;
  const int n = (int)fb->n;
  const int ncmax = (int)fb->nodes;  // every node in contact: the upper bound the run sizes for
  int rc;
  if (fb->layout_epoch != ws.layout_epoch && (rc = fem_contact_free_layout(fb))) return rc;
  // everything the loop touches, sized once (no allocation, no host read inside the loop)
  const size_t tr = (size_t)std::max(cfg->max_iters, 1);
  const size_t npad = (((size_t)std::max(n, 1) + 3) / 4) * 4 + 4;
  CK(vfpi::ensure(ws.vbuf, 3 * 8 * npad));
  CK(vfpi::ensure(ws.lambuf, 2 * 24 * (size_t)ncmax));
  CK(vfpi::ensure(ws.status, sizeof(vfpi::SolveStatus) * (size_t)S));
  CK(vfpi::ensure(ws.b_trace, 8 * tr * (size_t)S));
  CK(vfpi::ensure(ws.cont_list, 4 * (size_t)ncmax));
  CK(vfpi::ensure(ws.blk_ct, 4 * ((size_t)S + 1)));
  CK(vfpi::ensure(ws.w, 8 * (size_t)n));
  CK(vfpi::ensure(ws.gamma, 8 * (size_t)ncmax));
  CK(vfpi::ensure(ws.w_mean, 16));
  CK(vfpi::ensure(ws.partials, 2 * 8 * (size_t)S * vfpi::kPartialStride));
  CK(vfpi::ensure(fb->cg_r, 8 * (size_t)n));
  CK(vfpi::ensure(fb->cg_p, 8 * (size_t)n));
  CK(vfpi::ensure(fb->cg_q, 8 * (size_t)n));
  CK(vfpi::ensure(fb->run_acc, 8 * 8));
  if (iterations) CK(vfpi::ensure(fb->run_its, 4 * (size_t)std::max(steps, 1) * S));
  if (contacts) CK(vfpi::ensure(fb->run_cts, 4 * (size_t)std::max(steps, 1)));
  while (fb->run_ev.size() < 2 * (size_t)steps + 2) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    fb->run_ev.push_back(e);
  }
  CK(cudaMemsetAsync(fb->run_acc.p, 0, 64, st));
  CK(cudaMemsetAsync(ws.flags.p, 0, 16, st));
  vfpi::launch_iota_int(ncmax, P<int>(ws.cont_list), st);  // contacts stay in scene order
  ++h->launches;
  double* vb = P<double>(ws.vbuf);
  double* lb = P<double>(ws.lambuf);
  vfpi_system d = fb->A;
  d.n_c = ncmax;
  d.b = P<double>(fb->b);
  d.col_i = P<int32_t>(fb->ci);
  d.col_j = P<int32_t>(fb->cj);
  d.frames = P<double>(fb->frames);
  d.mu = P<double>(fb->mu);
  d.mu2 = P<double>(fb->mu2);
  d.phi = P<double>(fb->phi);
  const int* d_nc = P<int>(fb->cts) + S;  // the step's contact count, on the device
  vfpi::IterParams p{};
  p.n = n;
  p.n_c = ncmax;  // upper bound; the kernels take each scene's range from blk_ct
  p.G = S;
  p.blk_ct = P<int>(ws.blk_ct);
  p.cont_list = P<int>(ws.cont_list);
  p.b = d.b;
  p.w = P<double>(ws.w);
  p.gamma = P<double>(ws.gamma);
  p.col_i = d.col_i;
  p.col_j = d.col_j;
  p.frames = d.frames;
  p.mu = d.mu;
  p.mu2 = d.mu2;
  p.phi = d.phi;
  p.w_mean = P<double>(ws.w_mean);
  p.diag = P<double>(ws.diag);
  p.fixed_alpha_default = (cfg->step_strategy == VFPI_STEP_FIXED_ALPHA && std::isnan(cfg->fixed_alpha)) ? 1 : 0;
  p.vbuf0 = vb;
  p.vbuf1 = vb + npad;
  p.vbuf2 = vb + 2 * npad;
  p.lam0 = lb;
  p.lam1 = lb + 3 * (size_t)ncmax;
  p.partials = P<double>(ws.partials);
  p.trace = P<double>(ws.b_trace);
  p.trace_stride = tr;
  p.status = P<vfpi::SolveStatus>(ws.status);
  p.out_v = P<double>(fb->vhat);
  p.out_lam = P<double>(fb->lam);
  p.max_iters = cfg->max_iters;
  p.cheby_start = cfg->cheby_start;
  p.step = cfg->step_strategy;
  p.tol = cfg->residual_tol;
  p.under_relax = cfg->under_relax;
  p.omega = cfg->omega;
  p.cfactor = cfg->consistency_factor;
  CK(cudaEventRecord(fb->run_ev[0], st));
  for (int k = 0; k < steps; ++k) {
    // (1) right-hand side, (2) node-plane contacts (as vfpi_fem_step)
    fem_rhs(fb, 2.0 / q.dt, st);
    if (vfpi::launch_fem_detect(fb->nodes, S, fb->Nn, P<double>(fb->x), P<double>(fb->v), q.margin, fb->tmp.p,
                                fb->tmp.cap, P<int>(fb->pos), P<int>(fb->cts), P<double>(fb->frame), q.mu,
                                -(q.beta_err / q.dt), q.e_rest, q.rest_threshold, P<int>(fb->ci), P<int>(fb->cj),
                                P<double>(fb->frames), P<double>(fb->mu), P<double>(fb->mu2), P<double>(fb->phi),
                                lb, lb + 3 * (size_t)ncmax, st)) {
      h->err = "node-plane detection launch failed";
      return VFPI_CUDA_ERROR;
    }
    // (3) W, gamma and the solve of every scene (counts read on the device)
    CK(cudaMemcpyAsync(ws.blk_ct.p, fb->cts.p, 4 * ((size_t)S + 1), cudaMemcpyDeviceToDevice, st));
    rc = vfpi::setup_step_matrix(ws, d, *cfg, nullptr, st, h->err, h->launches, d_nc);
    if (rc) return rc;
    // (v ring: buffers 0 and 2 get the warm start, buffer 1 is written before it is read;
    // impulses and J_c^T lam slots of the live contacts are zeroed by the contact kernels)
    CK(cudaMemcpyAsync(vb, fb->warm.p, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(vb + 2 * npad, fb->warm.p, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(ws.status.p, 0, sizeof(vfpi::SolveStatus) * (size_t)S, st));
    if (vfpi::node_slots_refresh(fb->nbd, S, ncmax, d.col_i, d.col_j, d_nc, st)) {
      h->err = "node slot refresh failed";
      return VFPI_CUDA_ERROR;
    }
    CK(cudaEventRecord(fb->run_ev[2 + 2 * k], st));
    rc = vfpi::launch_iterate_nodes(p, fb->nbd, cfg->op, cheb, 1, st, h->err, nmode);
    if (rc) return rc;
    CK(cudaEventRecord(fb->run_ev[3 + 2 * k], st));
    // (3b) diverged scenes: the flagged contact-free CG step, decided on the device
    const int64_t ns = 3 * (int64_t)fb->Nn;
    if (vfpi::launch_cg_scenes_status(S, ns, fb->A.indptr, fb->A.indices, fb->A.data, P<double>(fb->b),
                                      P<double>(fb->vhat), P<double>(fb->cg_r), P<double>(fb->cg_p),
                                      P<double>(fb->cg_q), 1e-10, 10 * ns, P<vfpi::SolveStatus>(ws.status),
                                      P<int>(fb->cts), P<double>(fb->lam), st)) {
      h->err = "fallback CG launch failed";
      return VFPI_CUDA_ERROR;
    }
    // (4) midpoint integration, warm start; (5) counters
    vfpi::launch_fem_advance(fb->n, q.dt, P<double>(fb->vhat), P<double>(fb->x), P<double>(fb->v),
                             P<double>(fb->warm), st);
    vfpi::launch_fem_run_stats(S, P<vfpi::SolveStatus>(ws.status), P<int>(fb->cts), k,
                               P<unsigned long long>(fb->run_acc), iterations ? P<int>(fb->run_its) : nullptr,
                               contacts ? P<int>(fb->run_cts) : nullptr, st,
                               const_cast<int*>(fb->nbd.scene_perm));  // + the next step's longest-first order
    h->launches += 12;  // rhs, scan x2, detection, W/tie/gamma x3, slots, kernel, CG, advance, stats + order
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(fb->run_ev[1], st));
  unsigned long long acc[8];
  CK(cudaMemcpyAsync(acc, fb->run_acc.p, 64, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->h_flags, ws.flags.p, 4, cudaMemcpyDeviceToHost, st));
  if (iterations && steps) CK(cudaMemcpyAsync(iterations, fb->run_its.p, 4 * (size_t)steps * S, cudaMemcpyDeviceToHost, st));
  if (contacts && steps) CK(cudaMemcpyAsync(contacts, fb->run_cts.p, 4 * (size_t)steps, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  rc = flags_to_code(h, *h->h_flags);
  if (rc) return rc;
  stats->contact_iterations = (int64_t)acc[0];
  stats->iterations = (int64_t)acc[1];
  stats->diverged_scene_steps = (int32_t)acc[2];
  stats->max_iterations = (int32_t)acc[3];
  stats->contacts = (int64_t)acc[4];
  float ms = 0.f;
  cudaEventElapsedTime(&ms, fb->run_ev[0], fb->run_ev[1]);
  stats->run_ms = ms;
  for (int k = 0; k < steps; ++k) {
    cudaEventElapsedTime(&ms, fb->run_ev[2 + 2 * k], fb->run_ev[3 + 2 * k]);
    stats->loop_ms += ms;
  }
  h->last_node_kernel = 1;
  return VFPI_OK;
}

int vfpi_fem_set_node_layout(vfpi_fem_batch* fb, int32_t nodes_per_scene, const int32_t* order, int32_t n_slices,
                             const int64_t* slice_off, const int32_t* block_cols) {
  if (!fb || !order || !slice_off || !block_cols || nodes_per_scene != fb->Nn || n_slices != (fb->Nn + 31) / 32)
    return VFPI_BAD_ARGUMENT;
  vfpi_handle* h = fb->h;
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  if (slice_off[0] != 0) return VFPI_BAD_ARGUMENT;
  for (int t = 0; t < n_slices; ++t)
    if (slice_off[t + 1] < slice_off[t] || slice_off[t + 1] - slice_off[t] > 32) {
      h->err = "node layout: slice widths must be 0..32 blocks";
      return VFPI_BAD_ARGUMENT;
    }
  std::vector<char> seen((size_t)fb->Nn, 0);
  for (int i = 0; i < fb->Nn; ++i) {
    if (order[i] < 0 || order[i] >= fb->Nn || seen[(size_t)order[i]]) {
      h->err = "node layout: order must be a permutation of the scene's nodes";
      return VFPI_BAD_ARGUMENT;
    }
    seen[(size_t)order[i]] = 1;
  }
  const int64_t K = slice_off[n_slices];
  for (int64_t e = 0; e < 32 * K; ++e)
    if (block_cols[e] < -1 || block_cols[e] >= fb->Nn) {
      h->err = "node layout: block column out of range";
      return VFPI_BAD_ARGUMENT;
    }
  if ((int64_t)fb->S * K * 32 * 9 >= ((int64_t)1 << 40)) return VFPI_UNSUPPORTED;
  vfpi::NodeLayoutHost& L = fb->nbh;
  L.nn = fb->Nn;
  L.nsl = n_slices;
  L.k_scene = K;
  int rc;
  if ((rc = fem_upload(h, L.t_order, order, 4 * (size_t)fb->Nn)) ||
      (rc = fem_upload(h, L.t_off, slice_off, 8 * ((size_t)n_slices + 1))) ||
      (rc = fem_upload(h, L.t_bcol, block_cols, 4 * 32 * (size_t)std::max<int64_t>(K, 1))))
    return rc;
  cudaStream_t st = h->ws.stream;
  CK(vfpi::ensure(h->ws.flags, 16));
  CK(cudaMemsetAsync(h->ws.flags.p, 0, 16, st));
  L.t_off_host.assign(slice_off, slice_off + n_slices + 1);
  int cl = h->node_cluster ? vfpi::node_cluster_size(fb->S, n_slices, h->ws.num_sms) : 1;
  if (h->node_cluster_force > 0) cl = std::min(h->node_cluster_force, std::max(1, n_slices / 2));
  if (vfpi::node_layout_build(L, fb->S, fb->A.indptr, fb->A.indices, fb->A.data, fb->nbd, (int*)h->ws.flags.p, st,
                              cl, L.t_off_host)) {
    h->err = "node layout build failed";
    return VFPI_CUDA_ERROR;
  }
  h->launches += 2;
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, h->ws.flags.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (flag) {
    h->err = "node layout: A has entries outside the block template";
    fb->nb_ready = false;
    return VFPI_UNSUPPORTED;
  }
  fb->nb_ready = true;
  // K on the same template: the right-hand side streams node blocks too
  CK(cudaMemsetAsync(h->ws.flags.p, 0, 16, st));
  fb->kn_ready = false;
  if (vfpi::node_fill_matrix(L, fb->S, P<int64_t>(fb->krp), P<int>(fb->kc), P<double>(fb->kv), fb->kn_desc, fb->kn_val,
                             (int*)h->ws.flags.p, st) == 0) {
    CK(cudaMemcpyAsync(&flag, h->ws.flags.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fb->kn_ready = flag == 0;
  }
  return VFPI_OK;
}

int vfpi_fem_layout_info(vfpi_fem_batch* fb, int32_t* cluster, int64_t* bytes_per_scene_iteration) {
  if (!fb || !cluster || !bytes_per_scene_iteration) return VFPI_BAD_ARGUMENT;
  if (!fb->nb_ready) return VFPI_UNSUPPORTED;
  const int64_t ks = fb->nbd.k_scene;
  const bool nodesc = fb->nbd.tcol != nullptr;  // block columns from the template (no descriptor stream)
  *cluster = fb->nbd.cluster;
  // per k-step 32 lanes x (9 values [+ 1 descriptor]); per row b, w, v^(l-1), v^(l); per node its list entry and slot
  *bytes_per_scene_iteration = 32 * ks * (72 + (nodesc ? 0 : 4)) + 32 * 3 * (int64_t)fb->Nn + 8 * (int64_t)fb->Nn;
  return VFPI_OK;
}

int vfpi_fem_reset(vfpi_fem_batch* fb) {
  if (!fb) return VFPI_BAD_ARGUMENT;
  vfpi_handle* h = fb->h;
  if (cudaSetDevice(h->ws.device) != cudaSuccess) return VFPI_CUDA_ERROR;
  cudaStream_t st = h->ws.stream;
  const size_t n = (size_t)fb->n;
  CK(cudaMemcpyAsync(fb->x.p, fb->x0.p, 8 * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(fb->v.p, fb->v0.p, 8 * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(fb->warm.p, 0, 8 * n, st));
  return VFPI_OK;
}

int vfpi_fem_state_device(vfpi_fem_batch* fb, const double** x, const double** v) {
  if (!fb) return VFPI_BAD_ARGUMENT;
  if (x) *x = (const double*)fb->x.p;
  if (v) *v = (const double*)fb->v.p;
  return VFPI_OK;
}

int vfpi_fem_state(vfpi_fem_batch* fb, double* x, double* v) {
  if (!fb) return VFPI_BAD_ARGUMENT;
  vfpi_handle* h = fb->h;
  cudaSetDevice(h->ws.device);
  CK(cudaStreamSynchronize(h->ws.stream));
  if (x) CK(cudaMemcpy(x, fb->x.p, 8 * (size_t)fb->n, cudaMemcpyDeviceToHost));
  if (v) CK(cudaMemcpy(v, fb->v.p, 8 * (size_t)fb->n, cudaMemcpyDeviceToHost));
  return VFPI_OK;
}

void vfpi_fem_destroy(vfpi_fem_batch* fb) {
  if (!fb) return;
  cudaSetDevice(fb->h->ws.device);
  for (Workspace::Buf* b : {&fb->a_indptr, &fb->a_indices, &fb->a_data, &fb->krp, &fb->kc, &fb->kv, &fb->m, &fb->g,
                            &fb->X, &fb->x, &fb->v, &fb->warm, &fb->vhat, &fb->lam, &fb->b, &fb->ci, &fb->cj,
                            &fb->frames, &fb->mu, &fb->mu2, &fb->phi, &fb->flag, &fb->pos, &fb->cts, &fb->rows,
                            &fb->frame, &fb->tmp, &fb->zero_cts, &fb->ks_off, &fb->ks_val, &fb->ks_col, &fb->cg_r,
                            &fb->cg_p, &fb->cg_q, &fb->cg_list, &fb->x0, &fb->v0, &fb->nbh.t_order,
                            &fb->nbh.t_off, &fb->nbh.t_bcol, &fb->nbh.desc, &fb->nbh.val, &fb->nbh.slice_off,
                            &fb->nbh.node_list, &fb->nbh.node_slot, &fb->nbh.blk_slice, &fb->nbh.blk_pos, &fb->nbh.vs,
                            &fb->nbh.jt, &fb->nbh.perm, &fb->run_acc, &fb->run_its, &fb->run_cts})
    if (b->p) vfpi::dev_free(b->p);
  for (cudaEvent_t e : fb->run_ev) cudaEventDestroy(e);
  if (fb->e0) cudaEventDestroy(fb->e0);
  if (fb->e1) cudaEventDestroy(fb->e1);
  delete fb;
}

}  // extern "C"


// ---- virtual-node augmentation ----------------------------------------------
namespace {
int augment_common(vfpi_handle* h, const vfpi_augment_input* in, const vfpi_augment_input& dev, cudaStream_t st,
                   vfpi::AugmentOut& o) {
  vfpi::AugmentIn ai;
  ai.n_o = (int)in->n_o;
  ai.n_v3 = (int)in->n_v3;
  ai.a_nnz = in->a_nnz;
  ai.jv_nnz = in->jv_nnz;
  ai.a_indptr = dev.a_indptr;
  ai.a_indices = dev.a_indices;
  ai.a_data = dev.a_data;
  ai.jv_indptr = dev.jv_indptr;
  ai.jv_indices = dev.jv_indices;
  ai.jv_data = dev.jv_data;
  ai.k_v = in->k_v;
  return vfpi::augment_device(h->aug, ai, st, o, h->err, h->launches);
}
bool augment_args_ok(vfpi_handle* h, const vfpi_augment_input* in) {
  if (!in || in->n_o < 0 || in->n_v3 < 0 || in->n_v3 % 3 || in->a_nnz < 0 || in->jv_nnz < 0 ||
      in->n_o + in->n_v3 > INT32_MAX || in->a_nnz > INT32_MAX || in->jv_nnz > INT32_MAX) {
    h->err = "augment: bad sizes";
    return false;
  }
  return true;
}
}  // namespace

int vfpi_augment_device(vfpi_handle* h, const vfpi_augment_input* in, vfpi_augmented* out, void* stream) {
  if (!h || !out) return VFPI_BAD_ARGUMENT;
  if (!augment_args_ok(h, in)) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::AugmentOut o;
  const int rc = augment_common(h, in, *in, st, o);
  if (rc != VFPI_OK) return rc;
  out->n = o.n;
  out->nnz = o.nnz;
  out->indptr = o.indptr;
  out->indices = o.indices;
  out->data = o.data;
  return VFPI_OK;
}

int vfpi_augment(vfpi_handle* h, const vfpi_augment_input* in, vfpi_augmented* out) {
  if (!h || !out) return VFPI_BAD_ARGUMENT;
  if (!augment_args_ok(h, in)) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = h->ws.stream;
  Workspace& ws = h->ws;
  const int64_t n_o = in->n_o, rows = in->n_v3;
  CK(vfpi::ensure(ws.b_indptr, sizeof(int) * (size_t)(n_o + 1 + rows + 1)));
  CK(vfpi::ensure(ws.b_indices, sizeof(int) * (size_t)std::max<int64_t>(in->a_nnz + in->jv_nnz, 1)));
  CK(vfpi::ensure(ws.b_data, sizeof(double) * (size_t)std::max<int64_t>(in->a_nnz + in->jv_nnz, 1)));
  vfpi_augment_input dev = *in;
  int* dp = P<int>(ws.b_indptr);
  int* di = P<int>(ws.b_indices);
  double* dx = P<double>(ws.b_data);
  dev.a_indptr = dp;
  dev.jv_indptr = dp + n_o + 1;
  dev.a_indices = di;
  dev.jv_indices = di + in->a_nnz;
  dev.a_data = dx;
  dev.jv_data = dx + in->a_nnz;
  CK(cudaMemcpyAsync(dp, in->a_indptr, sizeof(int) * (size_t)(n_o + 1), cudaMemcpyHostToDevice, st));
  if (rows) CK(cudaMemcpyAsync(dp + n_o + 1, in->jv_indptr, sizeof(int) * (size_t)(rows + 1), cudaMemcpyHostToDevice, st));
  if (in->a_nnz) {
    CK(cudaMemcpyAsync(di, in->a_indices, sizeof(int) * (size_t)in->a_nnz, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dx, in->a_data, sizeof(double) * (size_t)in->a_nnz, cudaMemcpyHostToDevice, st));
  }
  if (in->jv_nnz) {
    CK(cudaMemcpyAsync(di + in->a_nnz, in->jv_indices, sizeof(int) * (size_t)in->jv_nnz, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dx + in->a_nnz, in->jv_data, sizeof(double) * (size_t)in->jv_nnz, cudaMemcpyHostToDevice, st));
  }
  vfpi::AugmentOut o;
  const int rc = augment_common(h, in, dev, st, o);
  if (rc != VFPI_OK) return rc;
  if (o.nnz > out->nnz) {
    h->err = "augment: output capacity too small (need " + std::to_string(o.nnz) + ")";
    out->nnz = o.nnz;
    return VFPI_BAD_ARGUMENT;
  }
  CK(cudaMemcpyAsync(out->indptr, o.indptr, sizeof(int) * (size_t)(o.n + 1), cudaMemcpyDeviceToHost, st));
  if (o.nnz) {
    CK(cudaMemcpyAsync(out->indices, o.indices, sizeof(int) * (size_t)o.nnz, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->data, o.data, sizeof(double) * (size_t)o.nnz, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  out->n = o.n;
  out->nnz = o.nnz;
  return VFPI_OK;
}

// ---- step-pipeline primitives (device pointers, caller stream) --------------
int vfpi_fem_rhs_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, const int32_t* k_indices,
                        const double* k_data, const double* x, const double* X, const double* v, const double* m,
                        const double* g, double dt, double* b, void* stream) {
  if (!h || n < 0) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::launch_fem_rhs(n, k_indptr, k_indices, k_data, x, X, v, m, g, 2.0 / dt, b, st);
  h->launches += n > 0;
  CK(cudaGetLastError());
  return VFPI_OK;
}

int vfpi_csr_matvec_device(vfpi_handle* h, int64_t rows, const int32_t* indptr, const int32_t* indices,
                           const double* data, const double* x, double* y, void* stream) {
  if (!h || rows < 0) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::launch_csr_matvec(rows, indptr, indices, data, x, y, st);
  h->launches += rows > 0;
  CK(cudaGetLastError());
  return VFPI_OK;
}

int vfpi_advance_device(vfpi_handle* h, int64_t n, double dt, const double* v_hat, double* x, double* v,
                        void* stream) {
  if (!h || n < 0) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::launch_fem_advance(n, dt, v_hat, x, v, nullptr, st);
  h->launches += n > 0;
  CK(cudaGetLastError());
  return VFPI_OK;
}

int vfpi_pile_contacts_device(vfpi_handle* h, const vfpi_pile_geometry* g, const double* x, const double* v,
                              vfpi_pile_contacts* out, void* stream) {
  if (!h || !g || !out || g->nodes < 0 || g->n_surf < 0 || g->n_tris < 0 || 3 * g->nodes > INT32_MAX ||
      !(g->cell > 0.0))
    return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::PileGeometry pg;
  pg.nodes = g->nodes;
  pg.n_surf = g->n_surf;
  pg.n_tris = g->n_tris;
  pg.n_o = (int)(3 * g->nodes);
  pg.surf = g->surf;
  pg.tris = g->tris;
  pg.node_body = g->node_body;
  pg.tri_body = g->tri_body;
  pg.reach = g->reach;
  pg.cell = g->cell;
  pg.neg_half_h = g->neg_half_h;
  pg.margin = g->margin;
  pg.mu = g->mu;
  pg.neg_beta_dt = g->neg_beta_dt;
  pg.e_rest = g->e_rest;
  pg.rest_threshold = g->rest_threshold;
  vfpi::PileContactsOut o;
  const int rc = vfpi::pile_contacts_device(h->pile, pg, x, v, st, o, h->err, h->launches);
  if (rc != VFPI_OK) return rc;
  out->n_c = o.n_ground + o.n_face;
  out->n_ground = o.n_ground;
  out->n_face = o.n_face;
  out->n_virtual = o.n_virtual;
  out->jv_nnz = o.jv_nnz;
  out->col_i = o.col_i;
  out->col_j = o.col_j;
  out->frames = o.frames;
  out->mu = o.mu;
  out->phi = o.phi;
  out->jv_indptr = o.jv_indptr;
  out->jv_indices = o.jv_indices;
  out->jv_data = o.jv_data;
  return VFPI_OK;
}

int vfpi_heightfield_contacts_device(vfpi_handle* h, const vfpi_heightfield_params* p, int64_t nodes,
                                     const double* x, vfpi_heightfield_contacts* out, void* stream) {
  if (!h || !p || !out || nodes < 0 || 3 * nodes > INT32_MAX || (nodes > 0 && !x)) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::HfParams hp{p->amp, p->freq, p->slope, p->margin, p->mu, p->neg_beta_dt};
  vfpi::HfContactsOut o;
  const int rc = vfpi::heightfield_contacts_device(h->hf, hp, nodes, x, st, o, h->err, h->launches);
  if (rc != VFPI_OK) return rc;
  out->n_c = o.n_c;
  out->col_i = o.col_i;
  out->col_j = o.col_j;
  out->frames = o.frames;
  out->mu = o.mu;
  out->phi = o.phi;
  return VFPI_OK;
}

int vfpi_add_device(vfpi_handle* h, int64_t n, const double* f, double* b, void* stream) {
  if (!h || n < 0 || (n > 0 && (!f || !b))) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::launch_add_inplace(n, f, b, st);
  h->launches += n > 0;
  CK(cudaGetLastError());
  return VFPI_OK;
}

int vfpi_memcpy_d2d(void* dst, const void* src, int64_t bytes) {
  if (bytes < 0) return VFPI_BAD_ARGUMENT;
  if (bytes == 0) return VFPI_OK;
  return cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice) == cudaSuccess ? VFPI_OK : VFPI_CUDA_ERROR;
}

int vfpi_nodalize_device(vfpi_handle* h, const vfpi_nodalize_input* in, vfpi_nodal_contacts* out, void* stream) {
  if (!h || !in || !out || in->n_c < 0 || in->n_c > INT32_MAX / 2 || in->n_o < 0 || in->n_o > INT32_MAX / 2)
    return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::NodalizeIn ni;
  ni.n_c = in->n_c;
  ni.n_o = (int)in->n_o;
  ni.n_bodies = (int)in->n_bodies;
  ni.n_q = in->n_q;
  ni.first_kind = in->first_kind;
  ni.first_ref = in->first_ref;
  ni.second_kind = in->second_kind;
  ni.second_ref = in->second_ref;
  ni.point = in->point;
  ni.normal = in->normal;
  ni.depth = in->depth;
  ni.q = in->q;
  ni.v = in->v;
  ni.body_q = in->body_q;
  ni.body_v = in->body_v;
  ni.mu = in->mu;
  ni.mu2 = std::isnan(in->mu2) ? in->mu : in->mu2;
  ni.neg_beta_dt = -(in->beta_err / in->dt);
  ni.e_rest = in->e_rest;
  ni.rest_threshold = in->rest_threshold;
  vfpi::NodalizeOut o;
  const int rc = vfpi::nodalize_device(h->nod, ni, st, o, h->err, h->launches);
  if (rc != VFPI_OK) return rc;
  out->n_c = in->n_c;
  out->n_virtual = o.n_virtual;
  out->jv_nnz = o.jv_nnz;
  out->col_i = o.col_i;
  out->col_j = o.col_j;
  out->frames = o.frames;
  out->phi = o.phi;
  out->mu = o.mu;
  out->mu2 = o.mu2;
  out->jv_indptr = o.jv_indptr;
  out->jv_indices = o.jv_indices;
  out->jv_data = o.jv_data;
  return VFPI_OK;
}

// ---- SELL-32 packing of a CSR matrix (step-pipeline right-hand sides) -------
int vfpi_sell_layout_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, int64_t* slice_off,
                            int64_t* elems) {
  if (!h || n < 0 || !elems) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = h->ws.stream;
  const int64_t nsl = (n + 31) / 32;
  CK(vfpi::ensure(h->ws.y, 8 * (size_t)(nsl + 1)));
  vfpi::launch_fem_sell_width(n, k_indptr, P<int64_t>(h->ws.y), st);
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, P<int64_t>(h->ws.y), slice_off, (int)(nsl + 1), st));
  CK(vfpi::ensure(h->ws.cub_tmp, tb));
  CK(cub::DeviceScan::ExclusiveSum(h->ws.cub_tmp.p, tb, P<int64_t>(h->ws.y), slice_off, (int)(nsl + 1), st));
  CK(cudaMemcpyAsync(elems, slice_off + nsl, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->launches += 2;
  return VFPI_OK;
}

int vfpi_sell_pack_device(vfpi_handle* h, int64_t n, const int64_t* k_indptr, const int32_t* k_indices,
                          const double* k_data, const int64_t* slice_off, double* sell_val, int32_t* sell_col) {
  if (!h || n < 0) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = h->ws.stream;
  vfpi::launch_fem_sell_pack(n, k_indptr, k_indices, k_data, slice_off, sell_val, sell_col, st);
  CK(cudaStreamSynchronize(st));
  h->launches += n > 0;
  return VFPI_OK;
}

int vfpi_fem_rhs_sell_device(vfpi_handle* h, int64_t n, const int64_t* slice_off, const double* sell_val,
                             const int32_t* sell_col, const double* x, const double* X, const double* v,
                             const double* m, const double* g, double dt, double* b, void* stream) {
  if (!h || n < 0) return VFPI_BAD_ARGUMENT;
  CK(cudaSetDevice(h->ws.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->ws.stream;
  vfpi::launch_fem_rhs_sell(n, slice_off, sell_val, sell_col, x, X, v, m, g, 2.0 / dt, b, st);
  h->launches += n > 0;
  CK(cudaGetLastError());
  return VFPI_OK;
}
