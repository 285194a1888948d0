"""Golden vectors of the virtual-node augmentation, from the REFERENCE.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_augment.py

Every case calls the reference's ``augment_dynamics`` (``contacts.py:343-375``)
and stores its input (A_o CSC arrays, b_o, J_v CSR arrays, k_v) and output
(the augmented CSC arrays and b):

* ``aug_rigid``: rigid bodies through the reference ``nodalize``
  (``contacts.py:271-321``, ``_slot_and_jv`` rigid sides: J_v blocks
  ``[I, -[r]x]``), including pairs of virtual nodes on one body with opposite
  levers (exact cancellations in J_vᵀJ_v) and explicit zeros stored in A_o;
* ``aug_face``: two FEM blocks with barycentric face-side virtual nodes
  (blocks ``w_k I`` on three nodes; some ``w_k`` exactly 0) and identity
  virtual nodes (a node's second contact, ``contacts.py:249-255``), J_v built
  the way ``nodalize`` builds it (COO of every block entry -> CSR);
* ``aug_none``: no virtual node (A_o returned unchanged, explicit zeros kept);
* ``metrics_ref.csv``: rows written by the reference's ``report_csv`` (harness.py:651-697);
* ``oneshot_aniso``: the reference strict-anisotropic one-shot with mu2 != mu
  (ellipse bisection, ``solver.py:103-141``);
* ``nodalize_mixed``: the reference ``nodalize`` (contacts.py:271-321) on mixed
  rigid / node / static sides with moving bodies and restitution.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from condsim.contacts import NodalContactSet, RawContact, augment_dynamics, nodalize  # noqa: E402
from condsim.dynamics import Body, SystemState, _quat_to_rot  # noqa: E402
from condsim.sparse import SparseSymmetric  # noqa: E402


def save(name, a_o, b_o, jv, k_v, aug):
    jv = sp.csr_matrix(jv) if jv is not None else sp.csr_matrix((0, a_o.dim))
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"), n_o=np.int64(a_o.dim), a_indptr=a_o.indptr.astype(np.int32),
        a_indices=a_o.indices.astype(np.int32), a_data=a_o.data, b_o=b_o, jv_rows=np.int64(jv.shape[0]),
        jv_indptr=jv.indptr.astype(np.int32), jv_indices=jv.indices.astype(np.int32), jv_data=jv.data,
        k_v=np.float64(k_v), out_indptr=aug.a.indptr.astype(np.int32), out_indices=aug.a.indices.astype(np.int32),
        out_data=aug.a.data, out_b=aug.b)
    print(name, "n", aug.n, "nnz", aug.a.data.shape[0], "zeros", int((aug.a.data == 0).sum()))


def rigid_case(rng, n_bodies=48, n_contacts=160, k_v=1e5):
    bodies, q, rows, cols, vals = [], [], [], [], []
    for k in range(n_bodies):
        m = rng.uniform(0.5, 2.0)
        inert = rng.uniform(0.01, 0.1, 3)
        quat = rng.standard_normal(4)
        quat /= np.linalg.norm(quat)
        bodies.append(Body("rigid6", float(m), 7 * k, 6 * k, np.diag(inert)))
        q += [np.zeros(3), quat]
        rot = _quat_to_rot(quat)
        for off, blk in ((6 * k, m * np.eye(3)), (6 * k + 3, rot @ np.diag(inert) @ rot.T)):
            ii, jj = np.meshgrid(range(off, off + 3), range(off, off + 3), indexing="ij")
            rows.append(ii.ravel())
            cols.append(jj.ravel())
            vals.append(blk.ravel())
        # explicit zeros between the translational and rotational blocks of some bodies
        if k % 3 == 0:
            rows.append(np.array([6 * k, 6 * k + 3]))
            cols.append(np.array([6 * k + 3, 6 * k]))
            vals.append(np.zeros(2))
    n_o = 6 * n_bodies
    a_o = SparseSymmetric.from_scipy(sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                                          np.concatenate(cols))),
                                                   shape=(n_o, n_o)).tocsc())
    b_o = rng.standard_normal(n_o)
    state = SystemState(np.concatenate(q), np.zeros(n_o), 0, 1e-3)
    raw = []
    for m in range(n_contacts):
        i, j = rng.choice(n_bodies - 2, 2, replace=False)
        lever = rng.uniform(-0.1, 0.1, 3)
        raw.append(RawContact(point=lever, normal=rng.standard_normal(3), depth=0.0,
                              first=("rigid", int(i), m), second=("rigid", int(j), m)))
        if m % 10 == 0:  # mirrored lever on the same bodies: J_v^T J_v cross terms cancel exactly
            raw.append(RawContact(point=-lever, normal=rng.standard_normal(3), depth=0.0,
                                  first=("rigid", int(i), m + 100000), second=("rigid", int(j), m + 100000)))
    if n_contacts:  # the last two bodies: only a mirrored pair -> exact zero sums in J_v^T J_v
        lever = np.array([0.0625, -0.03125, 0.0])
        for s, k in ((1.0, 0), (-1.0, 1)):
            raw.append(RawContact(point=s * lever, normal=np.array([0.0, 0.0, 1.0]), depth=0.0,
                                  first=("rigid", n_bodies - 2, -1 - k), second=("rigid", n_bodies - 1, -1 - k)))
    nodal = nodalize(raw, state, bodies, k_v, 0.5)
    return a_o, b_o, nodal


def face_case(rng, k_v=1e5):
    from paper_2201_09212_b200.scenes import FemCube

    blocks = [FemCube(nx=4).A, FemCube(nx=4, E=2e5).A]
    a = sp.block_diag(blocks, format="csc")
    a_o = SparseSymmetric.from_scipy(a)
    n_o = a_o.dim
    nn = n_o // 3
    b_o = rng.standard_normal(n_o)
    jv_rows = []
    nv = 0
    for f in range(40):  # face-side virtual nodes: w0 I, w1 I, w2 I on three nodes
        nodes = rng.choice(nn, 3, replace=False)
        w = rng.dirichlet(np.ones(3))
        if f % 7 == 0:
            w = np.array([0.25, 0.75, 0.0])
        for node, wk in zip(nodes, w):
            jv_rows.append((nv, 3 * int(node), wk * np.eye(3)))
        nv += 1
    for node in rng.choice(nn, 12, replace=False):  # identity virtual nodes
        jv_rows.append((nv, 3 * int(node), np.eye(3)))
        nv += 1
    r, c, v = [], [], []
    for virt, off, block in jv_rows:  # contacts.py:311-320
        for rr in range(3):
            for cc in range(block.shape[1]):
                r.append(3 * virt + rr)
                c.append(off + cc)
                v.append(block[rr, cc])
    jv = sp.csr_matrix((v, (r, c)), shape=(3 * nv, n_o))
    return a_o, b_o, NodalContactSet([], nv, jv, k_v)


def metrics_csv():
    """A CSV written by the reference's report_csv (harness.py:651-697)."""
    from condsim.harness import MetricsRow, report_csv

    rows = [MetricsRow(0, 0.123456789, 1.5, 12, 3.2e-9, 0.0, 0, 0.0),
            MetricsRow(1, 10.0, 0.1, 500, 1e-300, 1.4e-3, 60349, 1234.5678901234567, diverged=True),
            MetricsRow(2, 1.0 / 3.0, 2.0 ** -40, 7, 5e-324, 2.5e-17, 7, 1e22)]
    report_csv(rows, os.path.join(HERE, "metrics_ref.csv"))


def main():
    metrics_csv()
    rng = np.random.default_rng(91)
    a_o, b_o, nodal = rigid_case(rng)
    save("aug_rigid", a_o, b_o, nodal.jv, nodal.k_v, augment_dynamics(a_o, b_o, nodal))
    a_o, b_o, nodal = face_case(rng)
    save("aug_face", a_o, b_o, nodal.jv, nodal.k_v, augment_dynamics(a_o, b_o, nodal))
    a_o2, b_o2, _ = rigid_case(rng, n_bodies=6, n_contacts=0)
    save("aug_none", a_o2, b_o2, None, 1e5, augment_dynamics(a_o2, b_o2, NodalContactSet([], 0, None, 1e5)))



def nodalize_case(rng):
    """Mixed raw contacts through the reference ``nodalize`` (contacts.py:271-321):
    rigid-rigid, rigid-static, node-static, node-node, node-rigid, and nodes
    carrying a second contact (identity virtual nodes); moving bodies and a
    nonzero restitution so phi takes the v_n branch of stabilization_term."""
    from condsim.contacts import StabilizationParams

    n_rigid, n_part = 10, 14
    bodies, q, v = [], [], []
    qo = vo = 0
    for k in range(n_rigid):
        quat = rng.standard_normal(4)
        quat /= np.linalg.norm(quat)
        bodies.append(Body("rigid6", 1.0, qo, vo, np.eye(3)))
        q += [rng.uniform(-1, 1, 3), quat]
        v += [rng.standard_normal(6)]
        qo += 7
        vo += 6
    for k in range(n_part):
        bodies.append(Body("particle3", 0.1, qo, vo))
        q += [rng.uniform(-1, 1, 3)]
        v += [rng.standard_normal(3) * 0.05]
        qo += 3
        vo += 3
    state = SystemState(np.concatenate(q), np.concatenate(v), 0, 1e-3)
    node = lambda k: ("node", bodies[n_rigid + k].v_offset)  # noqa: E731
    raw = []
    for m in range(60):
        kind = m % 5
        if kind == 0:
            i, j = rng.choice(n_rigid, 2, replace=False)
            first, second = ("rigid", int(i), m), ("rigid", int(j), m)
        elif kind == 1:
            first, second = ("rigid", int(rng.integers(n_rigid)), m), ("static",)
        elif kind == 2:
            first, second = node(int(rng.integers(n_part))), ("static",)
        elif kind == 3:
            i, j = rng.choice(n_part, 2, replace=False)
            first, second = node(int(i)), node(int(j))
        else:
            first, second = node(int(rng.integers(n_part))), ("rigid", int(rng.integers(n_rigid)), m)
        nrm = rng.standard_normal(3)
        if m % 7 == 0:
            nrm = np.array([0.0, 0.0, 2.5])  # not unit: normalised inside contact_frame
        raw.append(RawContact(point=rng.uniform(-1, 1, 3), normal=nrm, depth=float(abs(rng.normal(0, 1e-3))),
                              first=first, second=second))
    stab = StabilizationParams(beta_err=0.2, e_rest=0.3, dt=1e-3, v_rest_threshold=0.01)
    nodal = nodalize(raw, state, bodies, 1e5, 0.45, 0.3, stab)
    slot = lambda s: -1 if s is None else (s[1] if s[0] == "orig" else state.v.shape[0] + 3 * s[1])  # noqa: E731
    kinds = {"node": 0, "rigid": 1, "static": -1}
    jv = sp.csr_matrix(nodal.jv)
    np.savez_compressed(
        os.path.join(HERE, "nodalize_mixed.npz"),
        q=state.q, v=state.v, body_q=np.array([b.q_offset for b in bodies], np.int32),
        body_v=np.array([b.v_offset for b in bodies], np.int32),
        first_kind=np.array([kinds[r.first[0]] for r in raw], np.int32),
        first_ref=np.array([r.first[1] for r in raw], np.int32),
        second_kind=np.array([kinds[r.second[0]] for r in raw], np.int32),
        second_ref=np.array([r.second[1] if len(r.second) > 1 else -1 for r in raw], np.int32),
        point=np.array([r.point for r in raw]), normal=np.array([r.normal for r in raw]),
        depth=np.array([r.depth for r in raw]), k_v=1e5, mu=0.45, mu2=0.3, beta=0.2, e_rest=0.3, dt=1e-3,
        thr=0.01, out_col_i=np.array([slot(c.slot_i) for c in nodal.contacts], np.int32),
        out_col_j=np.array([slot(c.slot_j) for c in nodal.contacts], np.int32),
        out_frames=np.array([c.frame for c in nodal.contacts]).reshape(-1),
        out_phi=np.array([c.phi_n for c in nodal.contacts]), out_mu=np.array([c.mu for c in nodal.contacts]),
        out_mu2=np.array([c.mu2 for c in nodal.contacts]), out_n_virtual=np.int64(nodal.n_virtual),
        out_jv_indptr=jv.indptr.astype(np.int32), out_jv_indices=jv.indices.astype(np.int32),
        out_jv_data=jv.data)
    print("nodalize_mixed n_c", len(nodal.contacts), "n_virtual", nodal.n_virtual, "jv nnz", jv.nnz)


def oneshot_aniso_case():
    """The reference one-shot with the strict-anisotropic operator and mu2 != mu
    (the ellipse bisection of solver.py:103-126, np.hypot included)."""
    from condsim.solver import SurrogateDelassus, contact_solve_oneshot

    g = np.random.default_rng(77)
    n = 3000
    eta = g.standard_normal((n, 3)) * 3.0
    eta[::17, 1:] *= 1e-6  # near-zero tangential parts
    gam = g.uniform(0.5, 2.0, n)
    phi = g.uniform(-1.0, 0.0, n)
    mu = g.uniform(0.1, 0.9, n)
    mu2 = g.uniform(0.1, 0.9, n)
    mu2[::11] = mu[::11]  # circle cases too
    lam = contact_solve_oneshot(SurrogateDelassus(gam), eta, phi, mu, "strict-anisotropic", mu2)
    np.savez_compressed(os.path.join(HERE, "oneshot_aniso.npz"), eta=eta, gamma=gam, phi=phi, mu=mu, mu2=mu2,
                        out_lam=np.asarray(lam))
    print("oneshot_aniso", n)


if __name__ == "__main__":
    main()
    nodalize_case(np.random.default_rng(5))
    oneshot_aniso_case()
