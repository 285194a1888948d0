"""Device SpMV and squared row norms (mirror of ``condsim/sparse.py:97-108``)."""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import as_f64, ptr
from .errors import DimensionMismatchError
from .solver import _raise_for
from .system import SparseSymmetric, make_packed


def _packed_matrix(a: SparseSymmetric):
    return make_packed(a.dim, a.indptr, a.indices, a.data, np.zeros(a.dim), [], [], [], [])


def spmv(a: SparseSymmetric, x) -> np.ndarray:
    """A @ x (``sparse.py:97-102``), bit-identical to scipy's CSC matvec."""
    x = as_f64(x)
    if x.shape != (a.dim,):
        raise DimensionMismatchError(f"spmv: x has shape {x.shape}, expected ({a.dim},)")
    h = _lib.handle()
    y = np.empty(a.dim)
    _raise_for(h.L.vfpi_spmv(h.h, _packed_matrix(a).c_struct(), ptr(x), ptr(y)), h)
    return y


def row_norms_sq(a: SparseSymmetric) -> np.ndarray:
    """Squared 2-norm of each row (``sparse.py:105-108``)."""
    h = _lib.handle()
    out = np.empty(a.dim)
    _raise_for(h.L.vfpi_row_norms_sq(h.h, _packed_matrix(a).c_struct(), ptr(out)), h)
    return out


def diagonal(a: SparseSymmetric) -> np.ndarray:
    """``SparseSymmetric.diagonal`` (``sparse.py:67-68``)."""
    h = _lib.handle()
    out = np.empty(a.dim)
    _raise_for(h.L.vfpi_diagonal(h.h, _packed_matrix(a).c_struct(), ptr(out)), h)
    return out
