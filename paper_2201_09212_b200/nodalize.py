"""Contact nodalization on the GPU.

``nodalize`` mirrors ``condsim.contacts.nodalize`` (``contacts.py:271-321``):
the reference's raw contacts (``RawContact`` with ``node`` / ``rigid`` /
``static`` sides), ``SystemState`` and ``Body`` list in, a ``NodalContactSet``
out (``Contact`` objects with the same slots, frames, ``phi_n``, ``mu``,
``mu2`` and keys, ``n_virtual``, the CSR ``J_v`` and ``k_v``), computed by
``vfpi_nodalize_device`` bit for bit like the reference
(``tests/test_nodalize.py`` against ``tests/golden/nodalize_mixed.npz``).
``nodalize_arrays`` is the flat-array form. Together with
``augment.augment_dynamics`` this is the reference's per-step contact
restructuring (``nodalize`` -> ``augment_dynamics``) on the device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib
from .solver import _raise_for
from .system import Contact, NodalContactSet

_KIND = {"node": 0, "rigid": 1, "static": -1}


def nodalize_arrays(first_kind, first_ref, second_kind, second_ref, point, normal, depth, q, v, body_q, body_v,
                    mu=0.5, mu2=None, beta_err=0.2, dt=0.01, e_rest=0.0, rest_threshold=0.01, device=None) -> dict:
    import torch

    h = _lib.handle(device)
    dev = torch.device("cuda", h.device)

    def up(a, dt_):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=dt_)).to(dev)

    n_c = int(np.asarray(first_kind).shape[0])
    n_o = int(np.asarray(v).shape[0])
    t = [up(first_kind, np.int32), up(first_ref, np.int32), up(second_kind, np.int32), up(second_ref, np.int32),
         up(np.asarray(point, float).reshape(-1), np.float64), up(np.asarray(normal, float).reshape(-1), np.float64),
         up(depth, np.float64), up(q, np.float64), up(v, np.float64), up(body_q, np.int32), up(body_v, np.int32)]
    inp = _lib.VfpiNodalizeInput(n_c, n_o, *[x.data_ptr() for x in t], float(mu),
                                 float("nan") if mu2 is None else float(mu2), float(beta_err), float(dt),
                                 float(e_rest), float(rest_threshold), int(np.asarray(body_q).shape[0]),
                                 int(np.asarray(q).shape[0]))
    out = _lib.VfpiNodalContacts()
    _raise_for(h.L.vfpi_nodalize_device(h.h, C.byref(inp), C.byref(out), None), h)
    d2h = lambda p, k, dt_: _lib.device_to_numpy(p, k, dt_, h.device)  # noqa: E731
    nv, nj = int(out.n_virtual), int(out.jv_nnz)
    jv = sp.csr_matrix((d2h(out.jv_data, nj, np.float64), d2h(out.jv_indices, nj, np.int32),
                        d2h(out.jv_indptr, 3 * nv + 1, np.int32)), shape=(3 * nv, n_o))
    return dict(col_i=d2h(out.col_i, n_c, np.int32).astype(np.int64),
                col_j=d2h(out.col_j, n_c, np.int32).astype(np.int64),
                frames=d2h(out.frames, 9 * n_c, np.float64).reshape(n_c, 3, 3),
                phi=d2h(out.phi, n_c, np.float64), mu=d2h(out.mu, n_c, np.float64),
                mu2=d2h(out.mu2, n_c, np.float64), jv=jv, n_virtual=nv)


def nodalize(raw_contacts, state, bodies, k_v: float, mu: float = 0.5, mu2: float | None = None, stab=None,
             device=None) -> NodalContactSet:
    """Drop-in for ``condsim.contacts.nodalize`` (``contacts.py:271-321``)."""
    beta, e_rest, thr = 0.2, 0.0, 0.01
    dt = getattr(state, "dt", 0.01)
    if stab is not None:
        beta, e_rest, thr, dt = stab.beta_err, stab.e_rest, stab.v_rest_threshold, stab.dt
    rc = list(raw_contacts)
    n_o = int(np.asarray(state.v).shape[0])
    if not rc:
        return NodalContactSet([], 0, None, k_v)
    for r in rc:
        for side in (r.first, r.second):
            if side[0] not in _KIND or (r.first is side and side[0] == "static"):
                raise ValueError(f"cannot nodalize side {side!r}")
    fk = [_KIND[r.first[0]] for r in rc]
    fr = [r.first[1] for r in rc]
    sk = [_KIND[r.second[0]] for r in rc]
    sr = [r.second[1] if len(r.second) > 1 else -1 for r in rc]
    out = nodalize_arrays(fk, fr, sk, sr, [r.point for r in rc], [r.normal for r in rc], [r.depth for r in rc],
                          state.q, state.v, [b.q_offset for b in bodies], [b.v_offset for b in bodies], mu, mu2,
                          beta, dt, e_rest, thr, device)

    def slot(col):
        return ("orig", int(col)) if col < n_o else ("virt", int(col - n_o) // 3)

    contacts = []
    for m, r in enumerate(rc):
        static = r.second[0] == "static"
        contacts.append(Contact(kind="S" if static else "D", slot_i=slot(out["col_i"][m]), frame=out["frames"][m],
                                mu=mu, depth=r.depth, phi_n=float(out["phi"][m]),
                                slot_j=None if static else slot(out["col_j"][m]), mu2=mu2,
                                key=(r.first, r.second)))
    return NodalContactSet(contacts, out["n_virtual"], out["jv"] if out["n_virtual"] else None, k_v)
