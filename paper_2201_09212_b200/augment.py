"""Virtual-node augmentation on the GPU.

``augment_dynamics`` mirrors ``condsim.contacts.augment_dynamics``
(``contacts.py:343-375``): it appends the virtual-node coordinates of a
``NodalContactSet`` and the viscous tie blocks

    A = [[A_o + k_v J_vᵀ J_v, -k_v J_vᵀ], [-k_v J_v, k_v I]],   b = [b_o; 0]

computed by ``vfpi_augment`` (``csrc/vfpi_augment.cu``) with the reference's
scipy arithmetic and stored-entry rules, so the CSC arrays are bit-identical to
the reference's ``SparseSymmetric.from_scipy(sp.bmat(...))``
(``tests/test_gpu_augment.py`` against ``tests/golden/aug_*.npz``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import VfpiAugmented, VfpiAugmentInput, as_f64, as_i32, ptr
from .errors import DimensionMismatchError
from .solver import _raise_for
from .system import AugmentedDynamics, SparseSymmetric


def _canonical_csr(jv, n_o: int):
    import scipy.sparse as sp

    m = sp.csr_matrix(jv)
    if m.shape[1] != n_o:
        raise DimensionMismatchError(f"J_v has {m.shape[1]} columns, A_o has {n_o}")
    if not m.has_canonical_format:
        m = m.copy()
        m.sum_duplicates()  # sorts too (what scipy's COO -> CSR gives nodalize)
    return m


def augment_arrays(n_o: int, a_indptr, a_indices, a_data, jv, k_v: float, device=None):
    """CSC arrays (indptr, indices, data) of the augmented matrix."""
    n_o = int(n_o)
    jv = _canonical_csr(jv, n_o)
    ap, ai, ax = as_i32(a_indptr), as_i32(a_indices), as_f64(a_data)
    if ap.shape[0] != n_o + 1 or ai.shape[0] != ax.shape[0] or ai.shape[0] != int(ap[-1]):
        raise DimensionMismatchError("augment: A_o arrays do not match its dimension")
    jp, ji, jx = as_i32(jv.indptr), as_i32(jv.indices), as_f64(jv.data)
    rows = jv.shape[0]
    row_of = np.repeat(np.arange(rows), np.diff(jp))
    nz = np.bincount(row_of[jx != 0.0], minlength=rows).astype(np.int64)
    cap = int(ai.shape[0] + int((nz * nz).sum()) + 2 * jx.shape[0] + rows) if rows else int(ai.shape[0])
    n = n_o + rows
    out_p = np.empty(n + 1, dtype=np.int32)
    out_i = np.empty(max(cap, 1), dtype=np.int32)
    out_x = np.empty(max(cap, 1), dtype=np.float64)
    h = _lib.handle(device)
    inp = VfpiAugmentInput(n_o, rows, ai.shape[0], ptr(ap, _lib._i32p), ptr(ai, _lib._i32p), ptr(ax),
                           jx.shape[0], ptr(jp, _lib._i32p), ptr(ji, _lib._i32p), ptr(jx), float(k_v))
    out = VfpiAugmented(0, cap, ptr(out_p, _lib._i32p), ptr(out_i, _lib._i32p), ptr(out_x))
    _raise_for(h.L.vfpi_augment(h.h, C.byref(inp), C.byref(out)), h)
    nnz = int(out.nnz)
    return out_p, out_i[:nnz].copy(), out_x[:nnz].copy()


def _slot_col(slot, n_orig: int) -> int:
    """``contacts.py:378-381``."""
    if slot[0] == "orig":
        return int(slot[1])
    return n_orig + 3 * int(slot[1])


def augment_dynamics(a_o, b_o, nodal, device=None) -> AugmentedDynamics:
    """``contacts.py:343-375`` with the matrix work on the GPU."""
    n_o = int(a_o.dim)
    b_o = np.asarray(b_o, dtype=float)
    if b_o.shape[0] != n_o:
        raise DimensionMismatchError("augment_dynamics: b length mismatch")
    if nodal.n_virtual == 0:
        aug = AugmentedDynamics(a_o, b_o.copy(), n_o, n_o, nodal)
    else:
        p, i, x = augment_arrays(n_o, a_o.indptr, a_o.indices, a_o.data, nodal.jv, nodal.k_v, device)
        nv3 = 3 * nodal.n_virtual
        b = np.concatenate([b_o, np.zeros(nv3)])
        aug = AugmentedDynamics(SparseSymmetric(n_o + nv3, p, i, x), b, n_o + nv3, n_o, nodal)
    cs = nodal.contacts
    n_c = len(cs)
    col_i = np.zeros(n_c, dtype=int)
    col_j = np.full(n_c, -1, dtype=int)
    frames = np.zeros((n_c, 3, 3))
    for m, c in enumerate(cs):
        col_i[m] = _slot_col(c.slot_i, n_o)
        if c.slot_j is not None:
            col_j[m] = _slot_col(c.slot_j, n_o)
        frames[m] = c.frame
    aug.col_i, aug.col_j, aug.frames = col_i, col_j, frames
    return aug
