"""Seeded synthetic workloads at BASELINE.json's shapes (inputs to the hot path).

``rigid_contact_system`` builds configs[1]: ``n_bodies`` rigid bodies with a
block-diagonal SPD A_o of 3x3 blocks [m I, R diag(I) R^T] and ``n_contacts``
D-contacts between random body pairs, nodalized onto per-contact virtual nodes
tied to the bodies with gain ``k_v`` — the reference's ``nodalize``
(``contacts.py:271-321``, ``_slot_and_jv`` ``:242-268``) followed by
``augment_dynamics`` (``:343-375``). The draw order and every floating-point
operation match ``tests/golden/make_golden.py::rigid_pile_case`` (which runs
the reference itself), so the system is bit-identical to the reference's;
``tests/test_scenes.py`` checks that against the committed golden fixture.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .contacts import contact_frame
from .system import PackedSystem, make_packed


def _quat_to_rot(q):
    """``dynamics.py:150-158``."""
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def rigid_contact_system(n_bodies: int = 4096, n_contacts: int = 16384, seed: int = 2201, k_v: float = 1e5,
                         dt: float = 1e-3, beta_err: float = 0.2) -> PackedSystem:
    """configs[1]: 4096 rigid bodies, 16384 D-contacts (defaults)."""
    rng = np.random.default_rng(seed)
    mass = rng.uniform(0.5, 2.0, n_bodies)
    inert = rng.uniform(0.01, 0.1, (n_bodies, 3))
    quat = rng.standard_normal((n_bodies, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    pairs = rng.integers(0, n_bodies - 1, (n_contacts, 2))
    pairs[:, 1] += pairs[:, 1] >= pairs[:, 0]
    normals = rng.standard_normal((n_contacts, 3))
    levers = rng.uniform(-0.1, 0.1, (n_contacts, 3))
    mus = rng.uniform(0.2, 0.8, n_contacts)
    b_o = rng.standard_normal(6 * n_bodies)

    # A_o: per body the translational m*I and rotational R diag(I) R^T 3x3 blocks
    n_o = 6 * n_bodies
    blocks = np.empty((2 * n_bodies, 3, 3))
    eye = np.eye(3)
    for k in range(n_bodies):
        rot = _quat_to_rot(quat[k])
        blocks[2 * k] = mass[k] * eye
        blocks[2 * k + 1] = rot @ np.diag(inert[k]) @ rot.T
    offs = (3 * np.arange(2 * n_bodies))[:, None, None]
    ii = np.broadcast_to(offs + np.arange(3)[None, :, None], blocks.shape)
    jj = np.broadcast_to(offs + np.arange(3)[None, None, :], blocks.shape)
    a_o = sp.coo_matrix((blocks.ravel(), (ii.ravel(), jj.ravel())), shape=(n_o, n_o)).tocsc()
    a_o.sum_duplicates()

    # J_v rows of the two virtual nodes of every contact: [I, -[r]x]
    n_v = 2 * n_contacts
    blk = np.zeros((n_v, 3, 6))
    blk[:, :, :3] = eye
    lev = np.repeat(levers, 2, axis=0)
    lx = np.zeros((n_v, 3, 3))
    lx[:, 0, 1], lx[:, 0, 2] = -lev[:, 2], lev[:, 1]
    lx[:, 1, 0], lx[:, 1, 2] = lev[:, 2], -lev[:, 0]
    lx[:, 2, 0], lx[:, 2, 1] = -lev[:, 1], lev[:, 0]
    blk[:, :, 3:] = -lx
    body = pairs.reshape(-1)  # virtual node 2m -> first body, 2m+1 -> second
    rows = (3 * np.arange(n_v))[:, None, None] + np.arange(3)[None, :, None] + np.zeros((1, 1, 6), dtype=np.int64)
    cols = (6 * body)[:, None, None] + np.arange(6)[None, None, :] + np.zeros((1, 3, 1), dtype=np.int64)
    jv = sp.csr_matrix((blk.ravel(), (rows.ravel(), cols.ravel())), shape=(3 * n_v, n_o))

    frames = np.empty((n_contacts, 3, 3))
    for m in range(n_contacts):
        frames[m] = contact_frame(normals[m])
    phi = np.full(n_contacts, -(beta_err / dt) * 0.0)  # depth 0, bodies at rest

    top_left = a_o + k_v * (jv.T @ jv)
    a = sp.bmat([[top_left, -k_v * jv.T], [-k_v * jv, k_v * sp.identity(3 * n_v, format="csr")]], format="csc")
    a = sp.csc_matrix(a)
    a.sum_duplicates()
    b = np.concatenate([b_o, np.zeros(3 * n_v)])
    col_i = n_o + 6 * np.arange(n_contacts)
    col_j = col_i + 3
    return make_packed(n_o + 3 * n_v, a.indptr, a.indices, a.data, b, col_i, col_j, frames, mus, mus, phi)
