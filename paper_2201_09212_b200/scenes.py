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

import math

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
# alternating parity, lumped mass rho V / 4 per tet node,
# A = (2/dt) M + (dt/2) K, b = (2/dt) M v - K (x - X) + m g (Eq. 10 with the
# elastic potential). Node-plane contacts follow the reference's
# detect_contacts (contacts.py:159-200, NodeProxy radius 0, margin 1e-4) and
# nodalize (contacts.py:271-321): one S-contact per node below the margin,
# frame contact_frame(+z), phi = -(beta/dt) depth (+ restitution).
#
# The element stiffness is the isotropic closed form of V B^T C B,
#   K_ab[p, q] = V (lam g_a[p] g_b[q] + mu (g_a[q] g_b[p] + delta_pq g_a . g_b)),
# with g_a the barycentric gradients (rows of D^-1 from explicit cross
# products), written as elementwise numpy only (no LAPACK/BLAS, whose kernels
# differ between hosts), so every host produces the same bits; duplicates are
# summed in element order into K's (column, row)-sorted pattern (np.add.at).
# The plan depends only on nx, so a batch of scenes (configs[2]) assembles all
# of them at once: ``fem_assemble`` vectorises over scenes and threads over
# scene chunks, and a single cube is the batch of one.

_EVEN = ((0, 1, 2, 4), (1, 3, 2, 7), (1, 4, 5, 7), (2, 4, 6, 7), (1, 2, 4, 7))
_ODD = ((1, 0, 3, 5), (0, 2, 3, 6), (0, 4, 5, 6), (3, 5, 6, 7), (0, 3, 5, 6))


def _tets(nx: int):
    """Tet connectivity of an nx^3-node grid, 5 tets per cell, parity-alternating split."""
    i, j, k = np.meshgrid(np.arange(nx - 1), np.arange(nx - 1), np.arange(nx - 1), indexing="ij")
    i, j, k = (a.transpose(2, 1, 0).ravel() for a in (i, j, k))  # i fastest, then j, then k
    v = np.arange(8)
    corners = ((i[:, None] + (v & 1)) + nx * ((j[:, None] + ((v >> 1) & 1)) + nx * (k[:, None] + ((v >> 2) & 1))))
    even = ((i + j + k) % 2 == 0)[:, None, None]
    loc = np.where(even, np.array(_EVEN)[None], np.array(_ODD)[None])  # (cells, 5, 4)
    return np.take_along_axis(corners[:, None, :], loc, axis=2).reshape(-1, 4).astype(np.int64)


def _elasticity(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return lam, mu


_PLANS: dict = {}


def _fem_plan(nx: int):
    """Sparsity plan of the nx^3 cube (cached): tets, K's CSC pattern (sorted
    by column, then row) and the slot of every element entry in it."""
    plan = _PLANS.get(nx)
    if plan is not None:
        return plan
    tets = _tets(nx)
    T = tets.shape[0]
    n = 3 * nx ** 3
    dof = (3 * tets[:, :, None] + np.arange(3)).reshape(T, 12)
    rows = np.broadcast_to(dof[:, :, None], (T, 12, 12)).ravel()
    cols = np.broadcast_to(dof[:, None, :], (T, 12, 12)).ravel()
    key = cols * n + rows
    uk, slot = np.unique(key, return_inverse=True)
    indices = (uk % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, (uk // n) + 1, 1)
    indptr = np.cumsum(indptr)
    diag = (uk % n) == (uk // n)
    plan = dict(tets=tets, slot=slot.astype(np.int32).reshape(T, 144), indices=indices, indptr=indptr, diag=diag,
                n=n, nnz=int(uk.shape[0]))
    _PLANS[nx] = plan
    return plan


def fem_rest_positions(nx, side, drops, yaws):
    """(S, nx^3, 3) rest positions: grid centred in x/y, bottom at z = 0, yawed
    by ``yaws`` about z, lifted by ``drops``."""
    h = side / (nx - 1)
    g = np.arange(nx) * h - side / 2
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel() + side / 2
    # glibc's cos/sin (math), not numpy's CPU-dispatched SIMD kernels: the same
    # bits on every host of this image
    yaws = [float(t) for t in np.atleast_1d(yaws)]
    cy = np.array([math.cos(t) for t in yaws])[:, None]
    sy = np.array([math.sin(t) for t in yaws])[:, None]
    drops = np.asarray(drops, dtype=np.float64)[:, None]
    X = np.empty((cy.shape[0], x.shape[0], 3))
    X[:, :, 0] = cy * x - sy * y
    X[:, :, 1] = sy * x + cy * y
    X[:, :, 2] = z[None, :] + drops
    return X


def _element_stiffness(X, tets, E, nu):
    """Element matrices (S, T, 144) (rows 3a+p, columns 3b+q) and volumes (S, T)."""
    S = X.shape[0]
    P = X[:, tets]                                            # (S, T, 4, 3)
    c0, c1, c2 = P[:, :, 1] - P[:, :, 0], P[:, :, 2] - P[:, :, 0], P[:, :, 3] - P[:, :, 0]

    def cross(a, b):
        return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                         a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                         a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)

    x12, x20, x01 = cross(c1, c2), cross(c2, c0), cross(c0, c1)
    det = (c0[..., 0] * x12[..., 0] + c0[..., 1] * x12[..., 1]) + c0[..., 2] * x12[..., 2]
    V = np.abs(det) / 6.0
    r = np.stack([x12, x20, x01], axis=2) / det[..., None, None]   # rows of D^-1: grad lambda_1..3
    g = np.concatenate([-((r[:, :, 0:1] + r[:, :, 1:2]) + r[:, :, 2:3]), r], axis=2)  # (S, T, 4, 3)
    lam, mu = _elasticity(np.asarray(E, dtype=np.float64), nu)
    lam = lam.reshape(S, 1, 1, 1, 1, 1)
    mu = mu.reshape(S, 1, 1, 1, 1, 1)
    gg = g[:, :, :, None, :, None] * g[:, :, None, :, None, :]           # [a, b, p, q] = g_a[p] g_b[q]
    dot = (gg[..., 0, 0] + gg[..., 1, 1]) + gg[..., 2, 2]                # g_a . g_b
    tr = gg.swapaxes(-1, -2).copy()                                      # g_a[q] g_b[p]
    idx = np.arange(3)
    tr[..., idx, idx] += dot[..., None]
    ke = V[:, :, None, None, None, None] * (lam * gg + mu * tr)          # (S, T, a, b, p, q)
    return ke.transpose(0, 1, 2, 4, 3, 5).reshape(S, tets.shape[0], 144), V


def _assemble_chunk(X, E, nu, rho, plan, tet_block=1 << 17):
    """K values (S, nnz_K) on the plan's pattern and lumped nodal masses
    (S, nodes): element entries added into their slots with ``np.add.at``
    (unbuffered, in element order -- the sum order is the tet order whatever
    the blocking)."""
    tets, slot, nk = plan["tets"], plan["slot"], plan["nnz"]
    S, nn = X.shape[0], X.shape[1]
    kd = np.zeros(S * nk)
    mass = np.zeros(S * nn)
    soff = (nk * np.arange(S, dtype=np.int64))[:, None, None]
    noff = (nn * np.arange(S, dtype=np.int64))[:, None, None]
    step = max(1, tet_block // S)
    for t0 in range(0, tets.shape[0], step):
        t1 = min(t0 + step, tets.shape[0])
        ke, V = _element_stiffness(X, tets[t0:t1], E, nu)
        np.add.at(kd, (slot[None, t0:t1] + soff).ravel(), ke.ravel())
        np.add.at(mass, (tets[None, t0:t1] + noff).ravel(), np.repeat((rho * V / 4.0).ravel(), 4))
    return kd.reshape(S, nk), mass.reshape(S, nn)


def fem_assemble(nx, Es, drops, yaws, side=0.1, nu=0.3, rho=1000.0, dt=1e-3, chunk=8, threads=None):
    """Batched assembly of ``len(Es)`` cubes sharing nx: returns the plan, rest
    positions (S, nodes, 3), K values (S, nnz_K), A values on K's pattern
    (S, nnz_K; exact zeros are dropped per scene, as scipy's sparse sum does),
    masses (S, n). Threads over scene chunks (numpy releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    plan = _fem_plan(nx)
    Es = np.atleast_1d(np.asarray(Es, dtype=np.float64))
    S = Es.shape[0]
    X = fem_rest_positions(nx, side, np.broadcast_to(drops, (S,)), np.broadcast_to(yaws, (S,)))
    kd = np.empty((S, plan["nnz"]))
    mass = np.empty((S, X.shape[1]))

    def work(a):
        b = min(a + chunk, S)
        kd[a:b], mass[a:b] = _assemble_chunk(X[a:b], Es[a:b], nu, rho, plan)

    starts = list(range(0, S, chunk))
    if len(starts) == 1:
        work(0)
    else:
        import os

        with ThreadPoolExecutor(threads or min(len(starts), len(os.sched_getaffinity(0)))) as ex:
            list(ex.map(work, starts))
    m3 = np.repeat(mass, 3, axis=1)
    # A = diags((2/dt) m) + (dt/2) K, as scipy's sparse sum forms it (entrywise a + b)
    ad = (dt / 2.0) * kd
    ad[:, plan["diag"]] = (2.0 / dt) * m3 + ad[:, plan["diag"]]
    return plan, X, kd, ad, m3


class FemCube:
    """One deformable cube (configs[0] defaults; configs[2] varies E, drop, yaw):
    matrices A (CSC, exact zeros dropped) and K (CSC, bitwise symmetric), lumped
    masses, rest and current state. Stepped on the device by
    ``fembatch.FemBatch``; the host restatement of its step (right-hand side,
    node-plane contacts, integration -- the checker) is ``oracle/fem_host.py``."""

    def __init__(self, nx=10, side=0.1, E=1e5, nu=0.3, rho=1000.0, drop=0.05, yaw=0.0, dt=1e-3, mu=0.5,
                 gravity=-9.81, margin=1e-4, beta_err=0.2, e_rest=0.0, rest_threshold=0.01, _parts=None):
        self.nx, self.dt, self.mu = nx, dt, mu
        self.margin, self.beta, self.e_rest, self.thr = margin, beta_err, e_rest, rest_threshold
        if _parts is None:
            plan, X, kd, ad, m3 = fem_assemble(nx, [E], [drop], [yaw], side=side, nu=nu, rho=rho, dt=dt)
            _parts = (plan, X[0], kd[0], ad[0], m3[0])
        plan, X, kd, ad, m3 = _parts
        n = plan["n"]
        self.X = X
        self.x = X.copy()
        self.v = np.zeros_like(X)
        self.K = sp.csc_matrix((kd, plan["indices"], plan["indptr"]), shape=(n, n))
        keep = ad != 0  # the sparse sum drops exact zeros
        cnt = np.zeros(n + 1, dtype=np.int64)
        cnt[1:] = np.add.reduceat(keep.astype(np.int64), plan["indptr"][:-1])
        self.A = sp.csc_matrix((ad[keep], plan["indices"][keep], np.cumsum(cnt)), shape=(n, n))
        self.m = m3
        self.gravity = np.zeros(n)
        self.gravity[2::3] = gravity
        self.n = n

    @classmethod
    def batch(cls, nx, Es, drops, yaws, side=0.1, nu=0.3, rho=1000.0, dt=1e-3, **kw):
        """configs[2]: many cubes assembled in one vectorised pass (``fem_assemble``);
        cube k is bit-identical to ``FemCube(nx, E=Es[k], drop=drops[k], yaw=yaws[k])``."""
        plan, X, kd, ad, m3 = fem_assemble(nx, Es, drops, yaws, side=side, nu=nu, rho=rho, dt=dt)
        return [cls(nx=nx, side=side, nu=nu, rho=rho, dt=dt, _parts=(plan, X[k], kd[k], ad[k], m3[k]), **kw)
                for k in range(len(Es))]


# ---------------------------------------------------------------------------
# configs[3]: 64^3-node linear-tet block pressed onto a heightfield
# ---------------------------------------------------------------------------
# The reference has no heightfield detector (parity of the
# detection is unpinned; the solve itself is pinned like every other system).
# Parameters BASELINE leaves open are fixed here and recorded by the bench:
# side 0.1 m (cfg0's), E 1e6, nu 0.35, rho 1000, mu 0.4, dt 1e-3,
# heightfield z = 0.005 sin(40x) sin(40y); the block is moulded to the surface
# (rest shape: bottom face on the heightfield, layers relaxing linearly to the
# flat top) and "pressed" = started 0.1 mm into it, plus a 50 N downward load
# spread over the top face -- so the whole bottom face (64^2 = 4,096 nodes,
# BASELINE's "~4096 node contacts") stays in contact. (A flat block pressed by
# 50 N cannot conform to 5 mm bumps at E = 1e6: it springs off and keeps only
# a few hundred contacts.)

# Heightfield trigonometry with a fixed operation sequence (Cody-Waite
# reduction by pi/2, fdlibm's sin/cos kernel polynomials, no FMA), so numpy on
# any host and the CUDA detector (csrc/vfpi_heightfield.cu, hf_sincos) produce
# the same bits; accurate to ~1 ulp for the |t| <= 10 the block reaches.
_TWO_OVER_PI = 6.36619772367581382433e-01
_PIO2_1 = 1.57079632673412561417e+00     # first 33 bits of pi/2
_PIO2_1T = 6.07710050650619224932e-11    # pi/2 - _PIO2_1
_S = (-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
      2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10)
_C = (4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
      -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11)


def hf_sincos(t):
    """(sin t, cos t) elementwise, the heightfield's deterministic evaluation."""
    t = np.asarray(t, dtype=np.float64)
    k = np.rint(t * _TWO_OVER_PI)
    r = (t - k * _PIO2_1) - k * _PIO2_1T
    z = r * r
    s = r + (z * r) * (_S[0] + z * (_S[1] + z * (_S[2] + z * (_S[3] + z * (_S[4] + z * _S[5])))))
    c = 1.0 - (0.5 * z - z * (z * (_C[0] + z * (_C[1] + z * (_C[2] + z * (_C[3] + z * (_C[4] + z * _C[5])))))))
    q = np.mod(k, 4.0)
    sin = np.where(q == 0, s, np.where(q == 1, c, np.where(q == 2, -s, -c)))
    cos = np.where(q == 0, c, np.where(q == 1, -s, np.where(q == 2, -c, s)))
    return sin, cos


HF_AMP, HF_FREQ = 0.005, 40.0


def heightfield(x, y, amp=HF_AMP, freq=HF_FREQ):
    """z = amp sin(freq x) sin(freq y), evaluated as (amp sx) sy."""
    sx, _ = hf_sincos(freq * np.asarray(x, dtype=np.float64))
    sy, _ = hf_sincos(freq * np.asarray(y, dtype=np.float64))
    return (amp * sx) * sy


class HeightfieldBlock(FemCube):
    """configs[3] (nx=64); small nx for parity tests. Stepped on the device by
    ``heightfield.HeightfieldStepper``; the host restatement of its contacts
    and right-hand side (the checker) is ``oracle/fem_host.py``."""

    def __init__(self, nx=64, side=0.1, E=1e6, nu=0.35, rho=1000.0, dt=1e-3, mu=0.4, press=50.0,
                 depth=1e-4, margin=1e-4, beta_err=0.2):
        self.amp, self.freq = HF_AMP, HF_FREQ
        plan = _fem_plan(nx)
        X = fem_rest_positions(nx, side, [0.0], [0.0])[0]
        k = np.round(X[:, 2] / (side / (nx - 1))).astype(int)  # layer index, 0 = bottom
        frac = 1.0 - k / (nx - 1)
        # rest shape: the bottom face follows the heightfield, the layers above
        # relax linearly to the flat top (a block moulded to the surface)
        X[:, 2] = X[:, 2] + frac * heightfield(X[:, 0], X[:, 1], self.amp, self.freq)
        kd, mass = _assemble_chunk(X[None], np.array([E]), nu, rho, plan)
        m3 = np.repeat(mass, 3, axis=1)
        ad = (dt / 2.0) * kd
        ad[:, plan["diag"]] = (2.0 / dt) * m3 + ad[:, plan["diag"]]
        super().__init__(nx=nx, side=side, E=E, nu=nu, rho=rho, drop=0.0, dt=dt, mu=mu, margin=margin,
                         beta_err=beta_err, _parts=(plan, X, kd[0], ad[0], m3[0]))
        # pressed `depth` into the surface: the bottom layer displaced down, the top not
        self.x = X.copy()
        self.x[:, 2] = X[:, 2] - frac * depth
        self.v = np.zeros_like(X)
        top = k == nx - 1
        self.f_ext = np.zeros(self.n)
        self.f_ext[3 * np.nonzero(top)[0] + 2] = -press / max(int(top.sum()), 1)
