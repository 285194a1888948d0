"""FEM scene batches stepped entirely on the device (configs[0]/[2]; SURVEY
§8(f) item 1): ``FemBatch`` uploads the block-diagonal A and K and the state
of a list of ``scenes.FemCube`` once; every ``step`` then assembles b, detects
node-plane contacts, solves all scenes (``vfpi_solve_scenes`` semantics, warm
start = previous solution) and integrates on the GPU through ``vfpi_fem_step``
(include/vfpi.h). The host pipeline (``FemCube.system`` -> ``solve_scenes`` ->
``FemCube.advance``) is its restatement; both give identical bits
(tests/test_gpu_fem.py)."""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from ._lib import VfpiConfig, as_f64, as_i32, ptr
from .contacts import contact_frame
from .solver import SolverConfig, _c_config, _raise_for
from .system import make_packed


class _Params(C.Structure):
    _fields_ = [("dt", C.c_double), ("margin", C.c_double), ("beta_err", C.c_double), ("e_rest", C.c_double),
                ("rest_threshold", C.c_double), ("mu", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("contacts", C.c_int64), ("contact_iterations", C.c_int64), ("iterations", C.c_int64),
                ("max_iterations", C.c_int32), ("diverged_scenes", C.c_int32), ("setup_ms", C.c_double),
                ("loop_ms", C.c_double), ("step_ms", C.c_double)]


class _RunStats(C.Structure):
    _fields_ = [("contacts", C.c_int64), ("contact_iterations", C.c_int64), ("iterations", C.c_int64),
                ("max_iterations", C.c_int32), ("diverged_scene_steps", C.c_int32), ("loop_ms", C.c_double),
                ("run_ms", C.c_double), ("host_synced", C.c_int32), ("reserved", C.c_int32)]


def _bind():
    L = _lib.lib()
    if not hasattr(L, "_fem_bound"):
        i64p = C.POINTER(C.c_int64)
        L.vfpi_fem_create.restype = C.c_int
        L.vfpi_fem_create.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_lib.VfpiSystem), i64p,
                                      _lib._i32p, _lib._f64p, _lib._f64p, _lib._f64p, _lib._f64p, _lib._f64p,
                                      _lib._f64p, _lib._f64p, C.POINTER(_Params), C.POINTER(C.c_void_p)]
        L.vfpi_fem_step.restype = C.c_int
        L.vfpi_fem_step.argtypes = [C.c_void_p, C.POINTER(VfpiConfig), C.POINTER(_Stats), _lib._i32p]
        L.vfpi_fem_state.restype = C.c_int
        L.vfpi_fem_state.argtypes = [C.c_void_p, _lib._f64p, _lib._f64p]
        L.vfpi_fem_set_node_layout.restype = C.c_int
        L.vfpi_fem_set_node_layout.argtypes = [C.c_void_p, C.c_int32, _lib._i32p, C.c_int32, C.POINTER(C.c_int64),
                                               _lib._i32p]
        L.vfpi_fem_run.restype = C.c_int
        L.vfpi_fem_run.argtypes = [C.c_void_p, C.POINTER(VfpiConfig), C.c_int32, C.POINTER(_RunStats), _lib._i32p,
                                   _lib._i32p]
        L.vfpi_fem_layout_info.restype = C.c_int
        L.vfpi_fem_layout_info.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.vfpi_fem_reset.restype = C.c_int
        L.vfpi_fem_reset.argtypes = [C.c_void_p]
        L.vfpi_fem_state_device.restype = C.c_int
        L.vfpi_fem_state_device.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.vfpi_fem_destroy.restype = None
        L.vfpi_fem_destroy.argtypes = [C.c_void_p]
        L._fem_bound = True
    return L


def _block_diag(mats):
    """Compressed arrays (CSC or CSR alike) of the block-diagonal stack, entries
    of each block kept exactly as stored (order, explicit zeros)."""
    ptrs, idx, val = [np.zeros(1, dtype=np.int64)], [], []
    nnz = 0
    off = 0
    for m in mats:
        ptrs.append(m.indptr[1:].astype(np.int64) + nnz)
        idx.append(m.indices.astype(np.int64) + off)
        val.append(m.data)
        nnz += m.nnz
        off += m.shape[0]
    return np.concatenate(ptrs), np.concatenate(idx), np.concatenate(val)


def node_block_template(indptr, indices, n):
    """Node-block SELL template of one scene (``vfpi_fem_set_node_layout``) from
    the CSC pattern of its K (every scene of a batch shares it): per node the
    ascending list of 3x3 block columns its rows touch, nodes ordered by
    decreasing block count (stable) in slices of 32, each slice as wide as its
    busiest node. Returns (order, slice_off, block_cols)."""
    nn = n // 3
    indptr = np.asarray(indptr, dtype=np.int64)
    col = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    key = np.unique((col // 3) * nn + np.asarray(indices, dtype=np.int64) // 3)  # (node, block column), sorted
    node, bcol = key // nn, key % nn
    cnt = np.bincount(node, minlength=nn)
    order = np.argsort(-cnt, kind="stable").astype(np.int32)
    nsl = (nn + 31) // 32
    pcnt = np.zeros(nsl * 32, dtype=np.int64)
    pcnt[:nn] = cnt[order]
    width = pcnt.reshape(nsl, 32).max(axis=1)
    slice_off = np.zeros(nsl + 1, dtype=np.int64)
    np.cumsum(width, out=slice_off[1:])
    pos = np.empty(nn, dtype=np.int64)
    pos[order] = np.arange(nn)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    k = np.arange(key.shape[0]) - start[node]
    p = pos[node]
    block_cols = np.full(32 * slice_off[-1], -1, dtype=np.int32)
    block_cols[32 * slice_off[p // 32] + 32 * k + p % 32] = bcol
    return order, slice_off, block_cols


def fem_batch_arrays(plan, X, kd, ad, m3, dt=1e-3, margin=1e-4, beta_err=0.2, e_rest=0.0, rest_threshold=0.01,
                     mu=0.5, gravity=-9.81, x=None, v=None):
    """The host arrays ``vfpi_fem_create`` uploads, in their final dtypes, built
    from ``scenes.fem_assemble``'s batched output without per-scene objects: A
    drops exact zeros per scene like the scipy sum ``FemCube`` uses; K is
    bitwise symmetric, so its CSC arrays are its CSR arrays."""
    S, nk = kd.shape
    n = plan["n"]
    keep = ad != 0
    cnt = np.add.reduceat(keep.astype(np.int64), plan["indptr"][:-1], axis=1)     # (S, n)
    a_ptr = np.zeros(S * n + 1, dtype=np.int64)
    np.cumsum(cnt.ravel(), out=a_ptr[1:])
    if a_ptr[-1] >= 2 ** 31 or S * nk >= 2 ** 31:
        raise ValueError("FemBatch: more than 2^31 stored entries; split the batch")
    off = (n * np.arange(S, dtype=np.int64))[:, None]
    a_idx = (plan["indices"][None, :] + off)[keep].astype(np.int32)
    a_val = ad[keep]
    k_ptr = (plan["indptr"][None, :-1] + nk * np.arange(S, dtype=np.int64)[:, None]).ravel()
    k_ptr = np.concatenate([k_ptr, [S * nk]])
    k_idx = (plan["indices"][None, :] + off).ravel().astype(np.int32)
    grav = np.zeros((S, n))
    grav[:, 2::3] = gravity
    Xf = np.ascontiguousarray(X.reshape(-1))
    prm = _Params(dt, margin, beta_err, e_rest, rest_threshold, mu)
    return (S, n, (a_ptr.astype(np.int32), a_idx, a_val), (k_ptr, k_idx, kd.reshape(-1)), m3.reshape(-1),
            grav.reshape(-1), Xf, Xf.copy() if x is None else x.reshape(-1),
            np.zeros(S * n) if v is None else v.reshape(-1), prm)


class FemBatch:
    """Device-resident batch of FemCube scenes (same node count, same dt/margin/mu).

    ``FemBatch(cubes, device)`` takes ``scenes.FemCube`` objects;
    ``FemBatch.assembled(...)`` takes ``scenes.fem_assemble``'s batched arrays
    directly (configs[2]'s 1024 scenes without per-scene objects)."""

    def __init__(self, cubes, device=None, _arrays=None, node_layout=True):
        if _arrays is None:
            c0 = cubes[0]
            for c in cubes:
                if (c.n, c.dt, c.margin, c.beta, c.e_rest, c.thr, c.mu) != (c0.n, c0.dt, c0.margin, c0.beta,
                                                                            c0.e_rest, c0.thr, c0.mu):
                    raise ValueError("scenes of a FemBatch share node count, dt, margin and contact parameters")
            a_ptr, a_idx, a_val = _block_diag([c.A for c in cubes])
            ks = [c.K.tocsr() for c in cubes]
            for km in ks:
                km.sort_indices()
            k_ptr, k_idx, k_val = _block_diag(ks)
            cat = lambda f: as_f64(np.concatenate([np.asarray(f(c), float).ravel() for c in cubes]))  # noqa: E731
            m, g, X, x, v = (cat(lambda c: c.m), cat(lambda c: c.gravity), cat(lambda c: c.X), cat(lambda c: c.x),
                             cat(lambda c: c.v))
            S, n_scene = len(cubes), c0.n
            prm = _Params(c0.dt, c0.margin, c0.beta, c0.e_rest, c0.thr, c0.mu)
        else:
            S, n_scene, (a_ptr, a_idx, a_val), (k_ptr, k_idx, k_val), m, g, X, x, v, prm = _arrays
        self.S, self.n_scene = S, n_scene
        self.h = _lib.handle(device)
        self.device = self.h.device
        self.L = _bind()
        ntot = self.S * self.n_scene
        self._a = make_packed(ntot, a_ptr, a_idx, a_val, np.zeros(ntot), [], [], [], [])
        self._k = (np.ascontiguousarray(k_ptr, dtype=np.int64), as_i32(k_idx), as_f64(k_val))
        self._m, self._g, self._X = as_f64(m), as_f64(g), as_f64(X)
        x, v = as_f64(x), as_f64(v)
        self.h2d_bytes = int(sum(a.nbytes for a in (self._a.indptr, self._a.indices, self._a.data, *self._k, self._m,
                                                     self._g, self._X, x, v)))
        frame = as_f64(contact_frame(np.array([0.0, 0.0, 1.0])).ravel())
        t0 = time.perf_counter()
        out = C.c_void_p()
        i64p = C.POINTER(C.c_int64)
        code = self.L.vfpi_fem_create(self.h.h, self.S, self.n_scene // 3, self._a.c_struct(), ptr(self._k[0], i64p),
                                      ptr(self._k[1], _lib._i32p), ptr(self._k[2]), ptr(self._m), ptr(self._g),
                                      ptr(self._X), ptr(x), ptr(v), ptr(frame), C.byref(prm), C.byref(out))
        _raise_for(code, self.h)
        self.fb = out
        t1 = time.perf_counter()
        self.node_kernel = False
        self.cluster = 1
        # bytes one iteration of one scene streams with the row-SELL layout: 12 per
        # stored entry + the row operands (the SURVEY §8(d) per-iteration count)
        self.layout_bytes_per_scene_iter = None
        if node_layout:
            # K's CSC pattern of scene 0 (all scenes share it)
            kp = self._k[0]
            n0 = self.n_scene
            order, soff, bcols = node_block_template(kp[: n0 + 1], self._k[1][: kp[n0]], n0)
            if soff.shape[0] > 1 and int(np.diff(soff).max(initial=0)) <= 32:
                rc = self.L.vfpi_fem_set_node_layout(self.fb, n0 // 3, ptr(order, _lib._i32p), soff.shape[0] - 1,
                                                     ptr(soff, C.POINTER(C.c_int64)), ptr(bcols, _lib._i32p))
                if rc not in (_lib.OK, _lib.UNSUPPORTED):
                    _raise_for(rc, self.h)
                self.node_kernel = rc == _lib.OK
                if self.node_kernel:
                    # the bytes the layout streams per scene and iteration (vfpi_fem_layout_info)
                    cl, by = C.c_int32(), C.c_int64()
                    _raise_for(self.L.vfpi_fem_layout_info(self.fb, C.byref(cl), C.byref(by)), self.h)
                    self.cluster = int(cl.value)
                    self.layout_bytes_per_scene_iter = int(by.value)
        # wall-clock split of the construction (vfpi_fem_create: uploads + K's row
        # SELL; vfpi_fem_set_node_layout with the host template)
        self.timings = {"create_s": t1 - t0, "node_layout_s": time.perf_counter() - t1}

    @classmethod
    def assembled(cls, plan, X, kd, ad, m3, device=None, node_layout=True, **params):
        """Batch straight from ``scenes.fem_assemble(nx, Es, drops, yaws)``: scene k is
        bit-identical to ``FemCube.batch(...)[k]``."""
        return cls(None, device=device, _arrays=fem_batch_arrays(plan, X, kd, ad, m3, **params),
                   node_layout=node_layout)

    def reset(self):
        """Back to the creation state (device to device, on the handle's stream)."""
        _raise_for(self.L.vfpi_fem_reset(self.fb), self.h)

    def state_device_ptrs(self):
        """(x, v) device pointers of the batch state (scene-major, n doubles each)."""
        x, v = C.c_void_p(), C.c_void_p()
        _raise_for(self.L.vfpi_fem_state_device(self.fb, C.byref(x), C.byref(v)), self.h)
        return int(x.value), int(v.value)

    def step(self, cfg: SolverConfig, per_scene=False):
        """One step of every scene; ``node_kernel`` in the result says whether the
        node-block iteration kernel ran (vs the row-SELL scene kernel)."""
        st = _Stats()
        its = np.zeros(self.S, dtype=np.int32) if per_scene else None
        code = self.L.vfpi_fem_step(self.fb, _c_config(cfg), C.byref(st),
                                    ptr(its, _lib._i32p) if its is not None else None)
        _raise_for(code, self.h)
        out = {f: getattr(st, f) for f, _ in _Stats._fields_}
        out["node_kernel"] = bool(self.L.vfpi_set_tuning(self.h.h, 7, 0))
        if its is not None:
            out["iterations_per_scene"] = its
        return out

    def run(self, cfg: SolverConfig, steps: int, per_step=False):
        """``steps`` steps of every scene back to back on the device (``vfpi_fem_run``:
        contact counts, the fallback and the counters stay on the device, one
        synchronisation at the end); identical results to ``steps`` calls of
        ``step``. ``per_step``: also the [steps, scenes] iteration counts and the
        per-step contact counts."""
        st = _RunStats()
        its = np.zeros((steps, self.S), dtype=np.int32) if per_step else None
        cts = np.zeros(steps, dtype=np.int32) if per_step else None
        code = self.L.vfpi_fem_run(self.fb, _c_config(cfg), int(steps), C.byref(st),
                                   ptr(its, _lib._i32p) if its is not None else None,
                                   ptr(cts, _lib._i32p) if cts is not None else None)
        _raise_for(code, self.h)
        out = {f: getattr(st, f) for f, _ in _RunStats._fields_ if f != "reserved"}
        if per_step:
            out["iterations_per_step"] = its
            out["contacts_per_step"] = cts
        return out

    def state(self):
        x = np.empty(self.S * self.n_scene)
        v = np.empty(self.S * self.n_scene)
        _raise_for(self.L.vfpi_fem_state(self.fb, ptr(x), ptr(v)), self.h)
        return x.reshape(self.S, -1, 3), v.reshape(self.S, -1, 3)

    def state_into(self, x: np.ndarray, v: np.ndarray):
        """Copy the device state into caller-owned (e.g. pinned) float64 host arrays."""
        _raise_for(self.L.vfpi_fem_state(self.fb, ptr(x), ptr(v)), self.h)

    def close(self):
        if getattr(self, "fb", None):
            self.L.vfpi_fem_destroy(self.fb)
            self.fb = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
