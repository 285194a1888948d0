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
                         dt: float = 1e-3, beta_err: float = 0.2, augment: str = "host") -> PackedSystem:
    """configs[1]: 4096 rigid bodies, 16384 D-contacts (defaults).

    ``augment="host"`` forms the augmented matrix with the reference's scipy
    expression (the fixture path), ``"device"`` with ``vfpi_augment`` on the
    GPU (bit-identical, ``tests/test_gpu_augment.py``)."""
    p = rigid_contact_parts(n_bodies, n_contacts, seed, k_v, dt, beta_err)
    if augment == "device":
        from .augment import augment_arrays

        ip, ix, dx = augment_arrays(p["n_o"], p["a_o"].indptr, p["a_o"].indices, p["a_o"].data, p["jv"], k_v)
    else:
        a_o, jv = p["a_o"], p["jv"]
        top_left = a_o + k_v * (jv.T @ jv)
        nv3 = jv.shape[0]
        a = sp.bmat([[top_left, -k_v * jv.T], [-k_v * jv, k_v * sp.identity(nv3, format="csr")]], format="csc")
        a = sp.csc_matrix(a)
        a.sum_duplicates()
        ip, ix, dx = a.indptr, a.indices, a.data
    b = np.concatenate([p["b_o"], np.zeros(p["jv"].shape[0])])
    return make_packed(p["n_o"] + p["jv"].shape[0], ip, ix, dx, b, p["col_i"], p["col_j"], p["frames"], p["mu"],
                       p["mu"], p["phi"])


def rigid_contact_parts(n_bodies: int = 4096, n_contacts: int = 16384, seed: int = 2201, k_v: float = 1e5,
                        dt: float = 1e-3, beta_err: float = 0.2) -> dict:
    """configs[1] before augmentation: A_o (CSC), b_o, J_v (CSR, nodalize's), contacts."""
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
    col_i = n_o + 6 * np.arange(n_contacts)
    return dict(n_o=n_o, a_o=a_o, b_o=b_o, jv=jv, col_i=col_i, col_j=col_i + 3, frames=frames, mu=mus, phi=phi)


# ---------------------------------------------------------------------------
# configs[0] / configs[2]: linear-tet FEM cube dropped on the plane z = 0
# ---------------------------------------------------------------------------
# The reference has no FEM; this is the linear small-strain
# assembly the SURVEY probe describes (Appendix C): 5 tets per hex with
# alternating parity, K_e = V B^T C B, lumped mass rho V / 4 per tet node,
# A = (2/dt) M + (dt/2) K, b = (2/dt) M v - K (x - X) + m g (Eq. 10 with the
# elastic potential). Node-plane contacts follow the reference's
# detect_contacts (contacts.py:159-200, NodeProxy radius 0, margin 1e-4) and
# nodalize (contacts.py:271-321): one S-contact per node below the margin,
# frame contact_frame(+z), phi = -(beta/dt) depth (+ restitution).

_EVEN = ((0, 1, 2, 4), (1, 3, 2, 7), (1, 4, 5, 7), (2, 4, 6, 7), (1, 2, 4, 7))
_ODD = ((1, 0, 3, 5), (0, 2, 3, 6), (0, 4, 5, 6), (3, 5, 6, 7), (0, 3, 5, 6))


def _tets(nx: int):
    tets = []
    idx = lambda i, j, k: i + nx * (j + nx * k)  # noqa: E731
    for k in range(nx - 1):
        for j in range(nx - 1):
            for i in range(nx - 1):
                c = [idx(i + (v & 1), j + ((v >> 1) & 1), k + ((v >> 2) & 1)) for v in range(8)]
                for t in (_EVEN if (i + j + k) % 2 == 0 else _ODD):
                    tets.append([c[a] for a in t])
    return np.array(tets, dtype=np.int64)


def _elasticity(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] += 2 * mu
    C[np.arange(3, 6), np.arange(3, 6)] = mu
    return C


class FemCube:
    """One deformable cube (configs[0] defaults; configs[2] varies E, drop, yaw)."""

    def __init__(self, nx=10, side=0.1, E=1e5, nu=0.3, rho=1000.0, drop=0.05, yaw=0.0, dt=1e-3, mu=0.5,
                 gravity=-9.81, margin=1e-4, beta_err=0.2, e_rest=0.0, rest_threshold=0.01):
        self.nx, self.dt, self.mu = nx, dt, mu
        self.margin, self.beta, self.e_rest, self.thr = margin, beta_err, e_rest, rest_threshold
        h = side / (nx - 1)
        g = np.arange(nx) * h - side / 2
        z, y, x = np.meshgrid(g, g, g, indexing="ij")
        X = np.stack([x.ravel(), y.ravel(), z.ravel() + side / 2], axis=1)
        cy, sy = np.cos(yaw), np.sin(yaw)
        X = X @ np.array([[cy, -sy, 0.0], [sy, cy, 0.0], [0.0, 0.0, 1.0]]).T
        X[:, 2] += drop
        self.X = X
        self.x = X.copy()
        self.v = np.zeros_like(X)
        tets = _tets(nx)
        C = _elasticity(E, nu)
        nn = X.shape[0]
        # all tets at once: D = [P1-P0, P2-P0, P3-P0] (columns), grad lambda_1..3 = rows of D^-1
        P = X[tets]                                   # (T, 4, 3)
        D = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], axis=2)
        V = np.abs(np.linalg.det(D)) / 6.0
        Gi = np.linalg.inv(D)                         # (T, 3, 3)
        grads = np.concatenate([-Gi.sum(axis=1, keepdims=True), Gi], axis=1)  # (T, 4, 3)
        T = tets.shape[0]
        B = np.zeros((T, 6, 12))
        for a in range(4):
            gx, gy, gz = grads[:, a, 0], grads[:, a, 1], grads[:, a, 2]
            c0 = 3 * a
            B[:, 0, c0], B[:, 1, c0 + 1], B[:, 2, c0 + 2] = gx, gy, gz
            B[:, 3, c0], B[:, 3, c0 + 1] = gy, gx
            B[:, 4, c0 + 1], B[:, 4, c0 + 2] = gz, gy
            B[:, 5, c0], B[:, 5, c0 + 2] = gz, gx
        Ke = V[:, None, None] * np.einsum("tji,jk,tkl->til", B, C, B)
        dof = (3 * tets[:, :, None] + np.arange(3)).reshape(T, 12)
        rows = [np.broadcast_to(dof[:, :, None], (T, 12, 12)).ravel()]
        cols = [np.broadcast_to(dof[:, None, :], (T, 12, 12)).ravel()]
        vals = [Ke.ravel()]
        mass = np.zeros(nn)
        np.add.at(mass, tets.ravel(), np.repeat(rho * V / 4.0, 4))
        n = 3 * nn
        K = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsc()
        K.sum_duplicates()
        self.K = K
        self.m = np.repeat(mass, 3)
        self.gravity = np.zeros(n)
        self.gravity[2::3] = gravity
        A = sp.diags((2.0 / dt) * self.m, format="csc") + (dt / 2.0) * K
        A = sp.csc_matrix(A)
        A.sum_duplicates()
        A.sort_indices()
        self.A = A
        self.n = n

    def contacts(self):
        """Node-plane contacts of the current configuration (reference detect + nodalize)."""
        z = self.x[:, 2]
        nodes = np.nonzero(z < self.margin)[0]
        depth = np.maximum(0.0, -z[nodes])
        phi = -(self.beta / self.dt) * depth
        vn = self.v[nodes, 2]
        rest = np.abs(vn) > self.thr
        phi = np.where(rest, phi + self.e_rest * np.minimum(0.0, vn), phi)
        frame = contact_frame(np.array([0.0, 0.0, 1.0]))
        return nodes, phi, depth, frame

    def system(self) -> PackedSystem:
        b = (2.0 / self.dt) * self.m * self.v.ravel() - self.K @ (self.x - self.X).ravel() + self.m * self.gravity
        nodes, phi, depth, frame = self.contacts()
        n_c = nodes.shape[0]
        mu = np.full(n_c, self.mu)
        return make_packed(self.n, self.A.indptr, self.A.indices, self.A.data, b, 3 * nodes,
                           np.full(n_c, -1), np.tile(frame.ravel(), n_c), mu, mu, phi)

    def advance(self, v_hat):
        """Midpoint integration (dynamics.py:237-255 for particles)."""
        vh = np.asarray(v_hat)[: self.n].reshape(-1, 3)
        self.x = self.x + self.dt * vh
        self.v = 2.0 * vh - self.v


# ---------------------------------------------------------------------------
# configs[3]: 64^3-node linear-tet block pressed onto a heightfield
# ---------------------------------------------------------------------------
# The reference has no heightfield detector (parity of the
# detection is unpinned; the solve itself is pinned like every other system).
# Parameters BASELINE leaves open are fixed here and recorded by the bench:
# side 0.1 m (cfg0's), E 1e6, nu 0.35, rho 1000, mu 0.4, dt 1e-3,
# heightfield z = 0.005 sin(40x) sin(40y), "pressed" = the bottom face conformed
# to the heightfield 0.1 mm deep, the layers above relaxing linearly to the flat
# rest shape, plus a 50 N downward load spread over the top face.

def _heightfield(x, y):
    return 0.005 * np.sin(40.0 * x) * np.sin(40.0 * y)


def _heightfield_normal(x, y):
    hx = 0.2 * np.cos(40.0 * x) * np.sin(40.0 * y)
    hy = 0.2 * np.sin(40.0 * x) * np.cos(40.0 * y)
    n = np.stack([-hx, -hy, np.ones_like(hx)], axis=-1)
    return n / np.linalg.norm(n, axis=-1, keepdims=True)


class HeightfieldBlock(FemCube):
    """configs[3] (nx=64); small nx for parity tests."""

    def __init__(self, nx=64, side=0.1, E=1e6, nu=0.35, rho=1000.0, dt=1e-3, mu=0.4, press=50.0,
                 depth=1e-4, margin=1e-4, beta_err=0.2):
        super().__init__(nx=nx, side=side, E=E, nu=nu, rho=rho, drop=0.0, dt=dt, mu=mu, margin=margin,
                         beta_err=beta_err)
        X = self.X
        k = np.round((X[:, 2] - X[:, 2].min()) / (side / (nx - 1))).astype(int)  # layer index
        bottom = _heightfield(X[:, 0], X[:, 1]) - depth
        frac = 1.0 - k / (nx - 1)
        self.x = X.copy()
        self.x[:, 2] = X[:, 2] + frac * bottom
        self.v = np.zeros_like(X)
        top = k == nx - 1
        self.f_ext = np.zeros(self.n)
        self.f_ext[3 * np.nonzero(top)[0] + 2] = -press / max(int(top.sum()), 1)

    def contacts(self):
        """Nodes within the margin of the heightfield: S-contacts along its normal."""
        x, y, z = self.x[:, 0], self.x[:, 1], self.x[:, 2]
        h = _heightfield(x, y)
        nodes = np.nonzero(z < h + self.margin)[0]
        depth = np.maximum(0.0, h[nodes] - z[nodes])
        phi = -(self.beta / self.dt) * depth
        normals = _heightfield_normal(x[nodes], y[nodes])
        frames = np.stack([contact_frame(nrm) for nrm in normals]) if len(nodes) else np.zeros((0, 3, 3))
        return nodes, phi, depth, frames

    def system(self) -> PackedSystem:
        b = ((2.0 / self.dt) * self.m * self.v.ravel() - self.K @ (self.x - self.X).ravel() + self.m * self.gravity
             + self.f_ext)
        nodes, phi, depth, frames = self.contacts()
        n_c = nodes.shape[0]
        mu = np.full(n_c, self.mu)
        return make_packed(self.n, self.A.indptr, self.A.indices, self.A.data, b, 3 * nodes, np.full(n_c, -1),
                           frames.reshape(-1), mu, mu, phi)
