"""Flat-array system container consumed by the C-ABI (``vfpi_system``).

``PackedSystem`` is the device-ready view of the reference's
``AugmentedDynamics`` (``contacts.py:118-128``): the CSC arrays of
``SparseSymmetric`` (``sparse.py:30-54``), ``b``, nodal contact columns,
frames and per-contact ``mu``/``mu2``/``phi``. ``pack(aug)`` accepts the
reference object (duck-typed) or one of this package's own.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import VfpiSystem, as_f64, as_i32, ptr, _i32p
from .errors import DimensionMismatchError


@dataclass
class SparseSymmetric:
    """Symmetric CSC matrix, both triangles stored (``sparse.py:30-54``)."""

    dim: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray

    @classmethod
    def from_scipy(cls, m) -> "SparseSymmetric":
        import scipy.sparse as sp

        csc = sp.csc_matrix(m)
        csc.sum_duplicates()
        return cls(csc.shape[0], csc.indptr, csc.indices, csc.data)

    @classmethod
    def from_dense(cls, m) -> "SparseSymmetric":
        import scipy.sparse as sp

        return cls.from_scipy(sp.csc_matrix(np.asarray(m, dtype=float)))

    @classmethod
    def identity(cls, n: int) -> "SparseSymmetric":
        import scipy.sparse as sp

        return cls.from_scipy(sp.identity(n, format="csc"))

    def as_scipy(self):
        import scipy.sparse as sp

        return sp.csc_matrix((self.data, self.indices, self.indptr), shape=(self.dim, self.dim))

    def to_dense(self) -> np.ndarray:
        return self.as_scipy().toarray()


@dataclass
class Contact:
    """One nodalized contact (``contacts.py:86-99``)."""

    kind: str
    slot_i: tuple
    frame: np.ndarray
    mu: float
    depth: float
    phi_n: float = 0.0
    slot_j: tuple | None = None
    mu2: float | None = None
    warm_impulse: np.ndarray | None = None
    key: tuple | None = None  # provenance (first side, second side)


@dataclass
class NodalContactSet:
    contacts: list
    n_virtual: int = 0
    jv: object = None
    k_v: float = 0.0


@dataclass
class AugmentedDynamics:
    """Same fields as the reference (``contacts.py:118-128``)."""

    a: SparseSymmetric
    b: np.ndarray
    n: int
    n_orig: int
    contacts: NodalContactSet | None = None
    col_i: np.ndarray | None = None
    col_j: np.ndarray | None = None
    frames: np.ndarray | None = None


@dataclass
class PackedSystem:
    """Contiguous arrays in the exact dtypes of ``vfpi_system``."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    b: np.ndarray
    col_i: np.ndarray
    col_j: np.ndarray
    frames: np.ndarray
    mu: np.ndarray
    mu2: np.ndarray
    phi: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_c(self) -> int:
        return int(self.col_i.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.data.shape[0])

    def c_struct(self) -> VfpiSystem:
        s = VfpiSystem()
        s.n, s.n_c, s.nnz = self.n, self.n_c, self.nnz
        s.indptr, s.indices = ptr(self.indptr, _i32p), ptr(self.indices, _i32p)
        s.data, s.b = ptr(self.data), ptr(self.b)
        s.col_i, s.col_j = ptr(self.col_i, _i32p), ptr(self.col_j, _i32p)
        s.frames, s.mu, s.mu2, s.phi = ptr(self.frames), ptr(self.mu), ptr(self.mu2), ptr(self.phi)
        return s


def make_packed(n, indptr, indices, data, b, col_i, col_j, frames, mu, mu2=None, phi=None) -> PackedSystem:
    n = int(n)
    col_i = as_i32(col_i).reshape(-1)
    n_c = col_i.shape[0]
    mu = as_f64(mu).reshape(-1) if n_c else np.zeros(0)
    ps = PackedSystem(
        n=n, indptr=as_i32(indptr), indices=as_i32(indices), data=as_f64(data),
        b=as_f64(b).reshape(-1), col_i=col_i, col_j=as_i32(col_j).reshape(-1),
        frames=as_f64(frames).reshape(-1),
        mu=mu, mu2=as_f64(mu2).reshape(-1) if mu2 is not None else mu.copy(),
        phi=as_f64(phi).reshape(-1) if phi is not None else np.zeros(n_c),
    )
    if ps.indptr.shape[0] != n + 1 or ps.b.shape[0] != n:
        raise DimensionMismatchError(f"system arrays do not match n={n}")
    if ps.col_j.shape[0] != n_c or ps.frames.shape[0] != 9 * n_c:
        raise DimensionMismatchError("contact arrays do not match n_c")
    return ps


def pack(aug) -> PackedSystem:
    """``AugmentedDynamics`` (reference or local) -> ``PackedSystem``.

    Per-contact parameters follow ``_contact_params`` (``solver.py:337-342``):
    ``mu2`` falls back to ``mu`` when ``None``.
    """
    if isinstance(aug, PackedSystem):
        return aug
    a = aug.a
    cs = aug.contacts.contacts if getattr(aug, "contacts", None) is not None else []
    n_c = len(cs)
    if n_c:
        mu = np.fromiter((c.mu for c in cs), dtype=float, count=n_c)
        mu2 = np.fromiter((c.mu2 if c.mu2 is not None else c.mu for c in cs), dtype=float, count=n_c)
        phi = np.fromiter((c.phi_n for c in cs), dtype=float, count=n_c)
        col_i, col_j, frames = aug.col_i, aug.col_j, aug.frames
    else:
        mu = mu2 = phi = np.zeros(0)
        col_i = col_j = np.zeros(0, dtype=np.int32)
        frames = np.zeros(0)
    return make_packed(aug.n, a.indptr, a.indices, a.data, aug.b, col_i, col_j, frames, mu, mu2, phi)
