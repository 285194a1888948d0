"""Host restatement of the configs[4] pile step pieces -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (and the digest generator under ``tests/golden/``) import
this module. The product steps a pile on the device (``pile.PileStepper``:
``vfpi_pile_contacts_device``, ``vfpi_fem_rhs_sell_device``,
``vfpi_augment_device``, ``vfpi_solve_device``, ``vfpi_advance_device``);
these functions are the restatement those kernels are checked against bit
for bit, written over a ``pile.CubePile``'s arrays:

* ``rhs`` -- b = (2/dt) M v - K (x - X) + M g;
* ``detect`` -- plane contacts + the spatial-hash broad phase and the
  node-to-face narrow phase (``pile`` module docstring);
* ``nodalize`` -- ``contacts.py:271-321`` with the ``face`` side kind;
* ``system`` / ``warm`` / ``advance`` -- ``augment_dynamics``
  (``contacts.py:343-375``), ``harness._warm_velocity`` (``harness.py:502-512``),
  midpoint integration (``dynamics.py:237-255``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from paper_2201_09212_b200.pile import PileContacts
from paper_2201_09212_b200.system import PackedSystem, make_packed

from . import vfpi_oracle as O

# Row-wise 3-vector products with their evaluation order spelled out (the
# device kernels in csrc/vfpi_pile.cu use exactly these expressions).
def _dot3(a, b):
    return a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1] + a[:, 2] * b[:, 2]


def _cross3(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


def contact_frames(normals: np.ndarray) -> np.ndarray:
    """``contact_frame`` (``contacts.py:131-149``) for many normals at once."""
    n = np.asarray(normals, dtype=float).reshape(-1, 3)
    norm = np.sqrt(_dot3(n, n))
    fix = np.abs(norm - 1.0) > 1e-9
    n = np.where(fix[:, None], n / norm[:, None], n)
    e = np.zeros_like(n)
    e[np.arange(n.shape[0]), np.argmin(np.abs(n), axis=1)] = 1.0
    t1 = _cross3(_cross3(n, e), n)
    t1 = t1 / np.sqrt(_dot3(t1, t1))[:, None]
    return np.stack([n, t1, _cross3(n, t1)], axis=1)


def _cell_key(c: np.ndarray) -> np.ndarray:
    c = c + (1 << 20)
    return (c[:, 0] << 42) | (c[:, 1] << 21) | c[:, 2]


def _ragged_arange(cnt: np.ndarray) -> np.ndarray:
    """concatenate(arange(k) for k in cnt)."""
    tot = int(cnt.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.cumsum(cnt) - cnt
    return np.arange(tot) - np.repeat(starts, cnt)



# ---- right-hand side ----
def rhs(pile) -> np.ndarray:
    """b = (2/dt) M v - K (x - X) + M g (scenes.FemCube.system), per row in
    increasing column order (scipy's CSC/CSR matvec order)."""
    K = sp.csr_matrix((pile.k_data, pile.k_indices, pile.k_indptr), shape=(pile.n, pile.n))
    u = (pile.x - pile.X).ravel()
    return (2.0 / pile.dt) * pile.m * pile.v.ravel() - K @ u + pile.m * pile.gravity

# ---- detection ----------------------------------------------------------
def detect(pile):
    """Raw contacts of the current state: plane contacts (all nodes with
    z < margin, node order), then node-to-face contacts (node order)."""
    x = pile.x
    ground = np.nonzero(x[:, 2] < pile.margin)[0]
    reach = max(0.5 * pile.h, pile.margin)
    cell = 2.0 * pile.h
    tri = pile.tris
    P = x[tri]                                    # (T, 3, 3)
    lo = np.floor((P.min(axis=1) - reach) / cell).astype(np.int64)
    hi = np.floor((P.max(axis=1) + reach) / cell).astype(np.int64)
    span = hi - lo
    smax = int(span.max(initial=0))
    if smax > 7:
        raise ValueError("pile: a surface triangle spans more than 8 hash cells (mesh too deformed)")
    keys, owner = [], []
    for dx in range(smax + 1):
        for dy in range(smax + 1):
            for dz in range(smax + 1):
                ok = (dx <= span[:, 0]) & (dy <= span[:, 1]) & (dz <= span[:, 2])
                c = lo[ok] + np.array([dx, dy, dz])
                keys.append(_cell_key(c))
                owner.append(np.nonzero(ok)[0])
    keys, owner = np.concatenate(keys), np.concatenate(owner)
    o = np.argsort(keys, kind="stable")
    keys, owner = keys[o], owner[o]
    s = pile.surf
    nk = _cell_key(np.floor(x[s] / cell).astype(np.int64))
    beg, end = np.searchsorted(keys, nk, "left"), np.searchsorted(keys, nk, "right")
    cnt = end - beg
    pn = np.repeat(s, cnt)
    pt = owner[np.repeat(beg, cnt) + _ragged_arange(cnt)]
    keep = pile.node_cube[pn] > pile.tri_cube[pt]  # one pass: nodes of the later body on faces of the earlier
    pn, pt = pn[keep], pt[keep]
    p = x[pn]
    a, b, c = x[tri[pt, 0]], x[tri[pt, 1]], x[tri[pt, 2]]
    nrm = _cross3(b - a, c - a)
    nrm = nrm / np.sqrt(_dot3(nrm, nrm))[:, None]
    d = _dot3(p - a, nrm)
    keep = (d > -0.5 * pile.h) & (d < pile.margin)
    pn, pt, p, a, b, c, nrm, d = pn[keep], pt[keep], p[keep], a[keep], b[keep], c[keep], nrm[keep], d[keep]
    q = p - d[:, None] * nrm
    v0, v1, v2 = b - a, c - a, q - a
    d00, d01, d11 = _dot3(v0, v0), _dot3(v0, v1), _dot3(v1, v1)
    d20, d21 = _dot3(v2, v0), _dot3(v2, v1)
    den = d00 * d11 - d01 * d01
    w1 = (d11 * d20 - d01 * d21) / den
    w2 = (d00 * d21 - d01 * d20) / den
    w0 = 1.0 - w1 - w2
    keep = (w0 >= 0.0) & (w1 >= 0.0) & (w2 >= 0.0)
    pn, pt, nrm, d = pn[keep], pt[keep], nrm[keep], d[keep]
    w = np.stack([w0[keep], w1[keep], w2[keep]], axis=1)
    o = np.lexsort((pt, -d, pn))                  # per node: largest d, then lowest triangle
    pn, pt, nrm, d, w = pn[o], pt[o], nrm[o], d[o], w[o]
    first = np.ones(pn.shape[0], dtype=bool)
    first[1:] = pn[1:] != pn[:-1]
    face = dict(node=pn[first], tri=tri[pt[first]], w=w[first], normal=nrm[first],
                depth=np.maximum(0.0, -d[first]))
    return ground, face

# ---- nodalize (contacts.py:271-321 with face sides) ----------------------
def nodalize(pile, ground, face) -> PileContacts:
    n_o = pile.n
    ng, nf = ground.shape[0], face["node"].shape[0]
    first_node = np.concatenate([ground, face["node"]])
    n_c = ng + nf
    # a node's first contact takes its own slot, later ones an identity virtual node
    _, first_idx = np.unique(first_node, return_index=True)
    own = np.zeros(n_c, dtype=bool)
    own[first_idx] = True
    needs = np.zeros((n_c, 2), dtype=bool)        # processing order: first side, second side
    needs[:, 0] = ~own
    needs[ng:, 1] = True
    vidx = (np.cumsum(needs.ravel()) - 1).reshape(n_c, 2)
    n_virtual = int(needs.sum())
    col_i = np.where(own, 3 * first_node, n_o + 3 * vidx[:, 0])
    col_j = np.full(n_c, -1, dtype=np.int64)
    col_j[ng:] = n_o + 3 * vidx[ng:, 1]
    # J_v blocks, every block entry stored (contacts.py:311-320)
    eye = np.eye(3).ravel()
    rr = np.repeat(np.arange(3), 3)
    cc = np.tile(np.arange(3), 3)
    ident = np.nonzero(~own)[0]
    r_id = (3 * vidx[ident, 0])[:, None] + rr[None, :]
    c_id = (3 * first_node[ident])[:, None] + cc[None, :]
    v_id = np.broadcast_to(eye, r_id.shape)
    fv = vidx[ng:, 1]
    r_f = (3 * fv)[:, None, None] + rr[None, None, :] + np.zeros((1, 3, 1), dtype=np.int64)
    c_f = (3 * face["tri"])[:, :, None] + cc[None, None, :]
    v_f = face["w"][:, :, None] * eye[None, None, :]
    rows = np.concatenate([r_id.ravel(), r_f.ravel()])
    cols = np.concatenate([c_id.ravel(), c_f.ravel()])
    vals = np.concatenate([np.asarray(v_id).ravel(), v_f.ravel()])
    jv = sp.csr_matrix((vals, (rows, cols)), shape=(3 * n_virtual, n_o))
    normals = np.concatenate([np.tile([0.0, 0.0, 1.0], (ng, 1)), face["normal"]])
    frames = contact_frames(normals) if n_c else np.zeros((0, 3, 3))
    depth = np.concatenate([np.maximum(0.0, -pile.x[ground, 2]), face["depth"]])
    vel = pile.v
    v_rel = vel[first_node].copy()
    if nf:
        w, vt = face["w"], vel[face["tri"]]
        v_rel[ng:] -= w[:, 0:1] * vt[:, 0] + w[:, 1:2] * vt[:, 1] + w[:, 2:3] * vt[:, 2]
    vn = _dot3(frames[:, 0, :], v_rel) if n_c else np.zeros(0)
    phi = -(pile.beta / pile.dt) * depth                 # stabilization_term (contacts.py:230-239)
    phi = np.where(np.abs(vn) > pile.thr, phi + pile.e_rest * np.minimum(0.0, vn), phi)
    return PileContacts(col_i, col_j, frames, phi, np.full(n_c, pile.mu), jv, ng, nf)


def contacts(pile) -> PileContacts:
    return nodalize(pile, *detect(pile))


# ---- the augmented system -------------------------------------------------
def system(pile, pc: PileContacts | None = None, b_o=None) -> PackedSystem:
    """The augmented system (``vfpi_oracle.augment``, the reference's ``augment_dynamics`` restated)."""
    pc = pc if pc is not None else contacts(pile)
    b_o = rhs(pile) if b_o is None else b_o
    nv3 = pc.jv.shape[0]
    ip, ix, dx, _ = O.augment(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, b_o, pc.jv, pile.k_v)
    b = np.concatenate([b_o, np.zeros(nv3)])
    return make_packed(pile.n + nv3, ip, ix, dx, b, pc.col_i, pc.col_j, pc.frames.reshape(-1), pc.mu, pc.mu,
                       pc.phi)


def warm(pile, prev_vhat, pc: PileContacts) -> np.ndarray:
    """``harness._warm_velocity`` (``harness.py:502-512``)."""
    n_o = pile.n
    v0 = np.zeros(n_o + pc.jv.shape[0])
    if prev_vhat is None:
        return v0
    v0[:n_o] = prev_vhat[:n_o]
    if pc.jv.shape[0]:
        v0[n_o:] = pc.jv @ v0[:n_o]
    return v0


def advance(pile, v_hat):
    """Midpoint integration (``dynamics.py:237-255``)."""
    vh = np.asarray(v_hat)[: pile.n].reshape(-1, 3)
    pile.x = pile.x + pile.dt * vh
    pile.v = 2.0 * vh - pile.v


