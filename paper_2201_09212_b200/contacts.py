"""Device contact-Jacobian gather/scatter (mirror of ``condsim/contacts.py:402-423``)."""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import as_f64, ptr
from .solver import _raise_for
from .system import AugmentedDynamics, Contact, NodalContactSet, pack  # noqa: F401  (re-exported)


def contact_frame(normal) -> np.ndarray:
    """Orthonormal frame with rows (n, t1, t2) (``contacts.py:131-149``).
    Host geometry helper used to build inputs; not on the iteration path."""
    n = np.asarray(normal, dtype=float)
    norm = np.linalg.norm(n)
    if norm < 1e-12:
        raise ValueError("contact normal is zero")
    if abs(norm - 1.0) > 1e-9:
        n = n / norm
    e = np.zeros(3)
    e[int(np.argmin(np.abs(n)))] = 1.0
    t1 = np.cross(np.cross(n, e), n)
    t1 /= np.linalg.norm(t1)
    return np.vstack([n, t1, np.cross(n, t1)])


def apply_jc(aug, v) -> np.ndarray:
    """J_c v as (n_c, 3) contact-frame velocities."""
    ps = pack(aug)
    h = _lib.handle()
    out = np.empty((ps.n_c, 3))
    _raise_for(h.L.vfpi_apply_jc(h.h, ps.c_struct(), ptr(as_f64(v)), ptr(out)), h)
    return out


def apply_jc_t(aug, lam, n: int | None = None) -> np.ndarray:
    """J_c^T lam over the augmented coordinates (``np.add.at`` semantics)."""
    ps = pack(aug)
    h = _lib.handle()
    out = np.empty(ps.n)
    _raise_for(h.L.vfpi_apply_jc_t(h.h, ps.c_struct(), ptr(as_f64(lam).reshape(-1)), ptr(out)), h)
    if n is not None and n != ps.n:
        res = np.zeros(n)
        res[: min(n, ps.n)] = out[: min(n, ps.n)]
        return res
    return out
