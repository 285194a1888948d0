"""ctypes binding of libvfpi.so (include/vfpi.h). Fails loudly if the
library or a CUDA device is missing — there is no CPU fallback."""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VFPI_LIB") or os.path.join(HERE, "libvfpi.so")

OK, DIVERGED, INVALID_MATRIX, TIE_VIOLATION, DIM_MISMATCH, CUDA_ERROR, UNSUPPORTED, BAD_ARGUMENT = range(8)
OPERATORS = {"strict": 0, "proximal": 1, "strict-anisotropic": 2}
STRATEGIES = {"frobenius": 0, "bb1": 1, "bb2": 2, "bb-alternating": 3, "fixed-alpha": 4}

_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


class VfpiSystem(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("n_c", C.c_int64), ("nnz", C.c_int64),
        ("indptr", _i32p), ("indices", _i32p), ("data", _f64p), ("b", _f64p),
        ("col_i", _i32p), ("col_j", _i32p), ("frames", _f64p),
        ("mu", _f64p), ("mu2", _f64p), ("phi", _f64p),
    ]


class VfpiConfig(C.Structure):
    _fields_ = [
        ("op", C.c_int32), ("step_strategy", C.c_int32), ("max_iters", C.c_int32),
        ("chebyshev", C.c_int32), ("cheby_start", C.c_int32), ("reserved", C.c_int32),
        ("residual_tol", C.c_double), ("under_relax", C.c_double), ("omega", C.c_double),
        ("fixed_alpha", C.c_double), ("consistency_factor", C.c_double),
    ]


class VfpiResult(C.Structure):
    _fields_ = [
        ("v", _f64p), ("lam", _f64p), ("residual_trace", _f64p), ("scc", _f64p), ("w", _f64p),
        ("iterations", C.c_int32), ("converged", C.c_int32), ("diverged", C.c_int32), ("status", C.c_int32),
        ("consistency", C.c_double), ("setup_ms", C.c_double), ("loop_ms", C.c_double),
    ]


class VfpiAugmentInput(C.Structure):
    _fields_ = [
        ("n_o", C.c_int64), ("n_v3", C.c_int64), ("a_nnz", C.c_int64),
        ("a_indptr", _i32p), ("a_indices", _i32p), ("a_data", _f64p),
        ("jv_nnz", C.c_int64), ("jv_indptr", _i32p), ("jv_indices", _i32p), ("jv_data", _f64p),
        ("k_v", C.c_double),
    ]


class VfpiAugmented(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("indptr", _i32p), ("indices", _i32p), ("data", _f64p)]


class VfpiPileGeometry(C.Structure):
    _fields_ = [
        ("nodes", C.c_int64), ("n_surf", C.c_int64), ("n_tris", C.c_int64),
        ("surf", C.c_void_p), ("tris", C.c_void_p), ("node_body", C.c_void_p), ("tri_body", C.c_void_p),
        ("reach", C.c_double), ("cell", C.c_double), ("neg_half_h", C.c_double), ("margin", C.c_double),
        ("mu", C.c_double), ("neg_beta_dt", C.c_double), ("e_rest", C.c_double), ("rest_threshold", C.c_double),
    ]


class VfpiPileContacts(C.Structure):
    _fields_ = [
        ("n_c", C.c_int64), ("n_ground", C.c_int64), ("n_face", C.c_int64), ("n_virtual", C.c_int64),
        ("jv_nnz", C.c_int64), ("col_i", _i32p), ("col_j", _i32p), ("frames", _f64p), ("mu", _f64p),
        ("phi", _f64p), ("jv_indptr", _i32p), ("jv_indices", _i32p), ("jv_data", _f64p),
    ]


class VfpiNodalizeInput(C.Structure):
    _fields_ = [
        ("n_c", C.c_int64), ("n_o", C.c_int64),
        ("first_kind", C.c_void_p), ("first_ref", C.c_void_p), ("second_kind", C.c_void_p),
        ("second_ref", C.c_void_p), ("point", C.c_void_p), ("normal", C.c_void_p), ("depth", C.c_void_p),
        ("q", C.c_void_p), ("v", C.c_void_p), ("body_q", C.c_void_p), ("body_v", C.c_void_p),
        ("mu", C.c_double), ("mu2", C.c_double), ("beta_err", C.c_double), ("dt", C.c_double),
        ("e_rest", C.c_double), ("rest_threshold", C.c_double), ("n_bodies", C.c_int64), ("n_q", C.c_int64),
    ]


class VfpiNodalContacts(C.Structure):
    _fields_ = [
        ("n_c", C.c_int64), ("n_virtual", C.c_int64), ("jv_nnz", C.c_int64),
        ("col_i", C.c_void_p), ("col_j", C.c_void_p), ("frames", C.c_void_p), ("phi", C.c_void_p),
        ("mu", C.c_void_p), ("mu2", C.c_void_p), ("jv_indptr", C.c_void_p), ("jv_indices", C.c_void_p),
        ("jv_data", C.c_void_p),
    ]


class VfpiHeightfieldParams(C.Structure):
    _fields_ = [("amp", C.c_double), ("freq", C.c_double), ("slope", C.c_double), ("margin", C.c_double),
                ("mu", C.c_double), ("neg_beta_dt", C.c_double)]


class VfpiHeightfieldContacts(C.Structure):
    _fields_ = [("n_c", C.c_int64), ("col_i", _i32p), ("col_j", _i32p), ("frames", _f64p), ("mu", _f64p),
                ("phi", _f64p)]


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libvfpi.so (raise if absent: the product has no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is not built; run `python -m paper_2201_09212_b200.build` "
                    "(the V-FPI solver has no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            H = C.c_void_p
            sysp, cfgp, resp = C.POINTER(VfpiSystem), C.POINTER(VfpiConfig), C.POINTER(VfpiResult)
            sig = {
                "vfpi_create": (C.c_int, [C.c_int, C.POINTER(H)]),
                "vfpi_destroy": (None, [H]),
                "vfpi_last_error": (C.c_char_p, [H]),
                "vfpi_version": (C.c_int, []),
                "vfpi_solve": (C.c_int, [H, sysp, cfgp, _f64p, _f64p, resp]),
                "vfpi_solve_device": (C.c_int, [H, sysp, cfgp, _f64p, _f64p, resp, C.c_void_p]),
                "vfpi_wait": (C.c_int, [H, resp]),
                "vfpi_launch_count": (C.c_int64, [H]),
                "vfpi_stream": (C.c_void_p, [H]),
                "vfpi_cg_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_double, C.c_int64, C.POINTER(C.c_int32), C.c_void_p]),
                "vfpi_last_layout": (C.c_int, [H, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
                "vfpi_set_kernel": (C.c_int, [H, C.c_int]),
                "vfpi_set_profile": (C.c_int, [H, C.c_int]),
                "vfpi_set_tuning": (C.c_int, [H, C.c_int, C.c_int]),
                "vfpi_augment": (C.c_int, [H, C.POINTER(VfpiAugmentInput), C.POINTER(VfpiAugmented)]),
                "vfpi_augment_device": (C.c_int, [H, C.POINTER(VfpiAugmentInput), C.POINTER(VfpiAugmented),
                                                  C.c_void_p]),
                "vfpi_get_profile": (C.c_int, [H, C.POINTER(C.c_longlong), C.c_int64]),
                "vfpi_fem_rhs_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                                  C.c_void_p, C.c_void_p]),
                "vfpi_csr_matvec_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                     C.c_void_p, C.c_void_p]),
                "vfpi_pile_contacts_device": (C.c_int, [H, C.POINTER(VfpiPileGeometry), C.c_void_p, C.c_void_p,
                                                        C.POINTER(VfpiPileContacts), C.c_void_p]),
                "vfpi_memcpy_d2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
                "vfpi_heightfield_contacts_device": (C.c_int, [H, C.POINTER(VfpiHeightfieldParams), C.c_int64,
                                                               C.c_void_p, C.POINTER(VfpiHeightfieldContacts),
                                                               C.c_void_p]),
                "vfpi_add_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
                "vfpi_sell_layout_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p,
                                                      C.POINTER(C.c_int64)]),
                "vfpi_sell_pack_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                    C.c_void_p, C.c_void_p]),
                "vfpi_fem_rhs_sell_device": (C.c_int, [H, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                                       C.c_void_p, C.c_void_p]),
                "vfpi_nodalize_device": (C.c_int, [H, C.POINTER(VfpiNodalizeInput), C.POINTER(VfpiNodalContacts),
                                                   C.c_void_p]),
                "vfpi_advance_device": (C.c_int, [H, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p]),
                "vfpi_host_alloc": (C.c_void_p, [C.c_int64]),
                "vfpi_host_free": (None, [C.c_void_p]),
                "vfpi_spmv": (C.c_int, [H, sysp, _f64p, _f64p]),
                "vfpi_row_norms_sq": (C.c_int, [H, sysp, _f64p]),
                "vfpi_diagonal": (C.c_int, [H, sysp, _f64p]),
                "vfpi_step_matrix_frobenius": (C.c_int, [H, sysp, C.c_int, _f64p]),
                "vfpi_surrogate_gamma": (C.c_int, [H, sysp, _f64p, C.c_double, _f64p]),
                "vfpi_apply_jc": (C.c_int, [H, sysp, _f64p, _f64p]),
                "vfpi_apply_jc_t": (C.c_int, [H, sysp, _f64p, _f64p]),
                "vfpi_contact_solve_oneshot": (C.c_int, [H, C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p, C.c_int,
                                                         _f64p]),
                "vfpi_scc_residual": (C.c_int, [H, C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p]),
                "vfpi_inverse_contact": (C.c_int, [H, sysp, _f64p, C.c_double, C.c_int, _f64p]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def ptr(a, typ=_f64p):
    if a is None:
        return None
    return a.ctypes.data_as(typ)


class Handle:
    """One device stream + workspace (vfpi_handle). One per thread."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        rc = self.L.vfpi_create(int(device), C.byref(h))
        if rc != OK:
            raise RuntimeError(f"vfpi_create(device={device}) failed with code {rc}: no usable CUDA device")
        self.h = h
        self.device = device

    def error(self) -> str:
        msg = self.L.vfpi_last_error(self.h)
        return msg.decode() if msg else ""

    def launches(self) -> int:
        return int(self.L.vfpi_launch_count(self.h))

    def stream_ptr(self) -> int:
        """The handle's own cudaStream_t (the FEM batch pipeline and NULL-stream
        calls enqueue there): record timing events on it."""
        return int(self.L.vfpi_stream(self.h) or 0)

    def torch_stream(self):
        import torch

        return torch.cuda.ExternalStream(self.stream_ptr(), device=torch.device("cuda", self.device))

    def set_kernel(self, mode: str):
        """'auto' | 'resident' | 'streaming' for later solves on this handle
        ('streaming' = a global-memory kernel: node-block when eligible, see
        ``set_node_kernel``, else row-SELL)."""
        code = {"auto": 0, "resident": 1, "streaming": 2}[mode]
        self.L.vfpi_set_kernel(self.h, code)

    def last_layout(self):
        r, g = C.c_int(), C.c_int()
        self.L.vfpi_last_layout(self.h, C.byref(r), C.byref(g))
        return {"resident": bool(r.value), "ctas": int(g.value),
                "node_kernel": bool(self.L.vfpi_set_tuning(self.h, 7, 0))}

    def set_node_cluster(self, on: bool):
        """FEM batches created afterwards: one thread-block cluster per scene when the
        batch is too small to fill the GPU (default on)."""
        self.L.vfpi_set_tuning(self.h, 8, 1 if on else 0)

    def set_node_kernel(self, on: bool):
        """Use the node-block kernels (FEM batches, single systems) when eligible (default on)."""
        self.L.vfpi_set_tuning(self.h, 6, 1 if on else 0)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.vfpi_destroy(self.h)
                self.h = None
        except Exception:
            pass


_tls = threading.local()


def default_device() -> int:
    """The device a handle binds to when none is given: torch's current CUDA
    device when torch is imported and sees a GPU (a rank that called
    ``torch.cuda.set_device(local_rank)``), else ``VFPI_DEVICE``, else
    ``LOCAL_RANK`` (one process per GPU under torchrun), else 0."""
    import sys

    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized() or torch.cuda.is_available():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    for var in ("VFPI_DEVICE", "LOCAL_RANK"):
        val = os.environ.get(var)
        if val not in (None, ""):
            return int(val)
    return 0


def handle(device: int | None = None) -> Handle:
    """Thread-local handle for ``device`` (default: ``default_device()``)."""
    if device is None:
        device = default_device()
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    h = hs.get(device)
    if h is None:
        h = hs[device] = Handle(device)
    return h


def as_i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.float64)


def device_to_numpy(src, count: int, dtype, device: int = 0) -> np.ndarray:
    """Copy ``count`` elements at a device pointer (e.g. a handle-owned output
    buffer) into a new host array."""
    import torch

    tdt = {np.dtype(np.int32): torch.int32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    t = torch.empty(max(int(count), 1), dtype=tdt, device=torch.device("cuda", device))
    if count:
        nbytes = int(count) * t.element_size()
        rc = lib().vfpi_memcpy_d2d(C.c_void_p(t.data_ptr()), C.cast(src, C.c_void_p), C.c_int64(nbytes))
        if rc != OK:
            raise RuntimeError(f"device copy failed with code {rc}")
    return t.cpu().numpy()[: int(count)]
