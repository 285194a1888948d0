"""Host restatements of the FEM step pipeline -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s CPU legs (``cpu_baseline`` /
``--impl reference``) import this module; the product path steps scenes on
the device (``fembatch.FemBatch`` / ``vfpi_fem_step``).

* ``fem_rhs`` / ``fem_contacts`` / ``fem_system`` / ``fem_advance`` and
  ``heightfield_*`` -- the host restatement of the device step pieces
  (``csrc/vfpi_fem.cu``, ``csrc/vfpi_heightfield.cu``) they are checked against;
* ``oracle_steps`` -- one ``scenes.FemCube`` advanced on the host with the
  oracle's ``solve`` (``vfpi_oracle.solve`` restating ``solver.py:345-461``)
  and the harness's contact-free CG fallback on divergence
  (``harness.py:586-593``), warm start = previous solution
  (``harness.py:502-512``; no virtual nodes here).
* ``reference_steps`` -- the same scene through the reference's OWN code:
  ``condsim.contacts.detect_contacts`` (plane vs radius-0 node proxies,
  ``contacts.py:159-227``), ``nodalize`` (``:271-321``), ``augment_dynamics``
  (``:343-375``), ``condsim.solver.solve_vfpi`` and the same fallback. The
  reference has no FEM, so A and b come from this repo's assembly
  (``FemCube``), exactly as ``tests/golden/make_golden.py::fem_cases`` feeds
  them. Needs ``condsim`` importable (``baseline/_ref`` or the reference tree).
"""

from __future__ import annotations

import numpy as np

from paper_2201_09212_b200.system import PackedSystem, make_packed

from . import vfpi_oracle as O


# ---- configs[0]/[2]: one FEM cube on the plane z = 0 -------------------------

def fem_rhs(cube) -> np.ndarray:
    """b = (2/dt) M v - K (x - X) + M g (scipy's CSC matvec: per row in
    increasing column order), the device's k_fem_rhs_sell."""
    return (2.0 / cube.dt) * cube.m * cube.v.ravel() - cube.K @ (cube.x - cube.X).ravel() + cube.m * cube.gravity


def fem_contacts(cube):
    """Node-plane contacts of the current state: the reference's
    detect_contacts (contacts.py:159-200, radius-0 node proxies, margin) +
    nodalize (:271-321) for S-contacts on nodes, frame contact_frame(+z),
    phi from stabilization_term (:230-239)."""
    from paper_2201_09212_b200.contacts import contact_frame

    z = cube.x[:, 2]
    nodes = np.nonzero(z < cube.margin)[0]
    depth = np.maximum(0.0, -z[nodes])
    phi = -(cube.beta / cube.dt) * depth
    vn = cube.v[nodes, 2]
    rest = np.abs(vn) > cube.thr
    phi = np.where(rest, phi + cube.e_rest * np.minimum(0.0, vn), phi)
    frame = contact_frame(np.array([0.0, 0.0, 1.0]))
    return nodes, phi, depth, frame


def fem_system(cube) -> PackedSystem:
    """The step's system (A, b, contacts) as ``solve_vfpi`` consumes it."""
    b = fem_rhs(cube)
    nodes, phi, depth, frame = fem_contacts(cube)
    n_c = nodes.shape[0]
    mu = np.full(n_c, cube.mu)
    return make_packed(cube.n, cube.A.indptr, cube.A.indices, cube.A.data, b, 3 * nodes,
                       np.full(n_c, -1), np.tile(frame.ravel(), n_c), mu, mu, phi)


def fem_advance(cube, v_hat):
    """Midpoint integration (dynamics.py:237-255 for particles)."""
    vh = np.asarray(v_hat)[: cube.n].reshape(-1, 3)
    cube.x = cube.x + cube.dt * vh
    cube.v = 2.0 * vh - cube.v


# ---- configs[3]: the block pressed onto the heightfield ----------------------

def heightfield_rhs(blk) -> np.ndarray:
    """fem_rhs + the top-face load (added last, as the device does)."""
    return fem_rhs(blk) + blk.f_ext


def heightfield_contacts(blk):
    """Nodes within the margin of z = amp sin(freq x) sin(freq y) (node order):
    depth max(0, h - z), phi = -(beta/dt) depth, normal (-hx, -hy, 1)/norm with
    hx = (amp freq) cos(freq x) sin(freq y), hy = (amp freq) sin(freq x) cos(freq y),
    frames contact_frame(normal) -- the device's k_hf_contacts operation for operation."""
    from paper_2201_09212_b200.scenes import hf_sincos

    from .pile_host import contact_frames

    x, y, z = blk.x[:, 0], blk.x[:, 1], blk.x[:, 2]
    sx, cx = hf_sincos(blk.freq * x)
    sy, cy = hf_sincos(blk.freq * y)
    h = (blk.amp * sx) * sy
    nodes = np.nonzero(z < h + blk.margin)[0]
    depth = np.maximum(0.0, h[nodes] - z[nodes])
    phi = -(blk.beta / blk.dt) * depth
    slope = blk.amp * blk.freq
    hx = (slope * cx[nodes]) * sy[nodes]
    hy = (slope * sx[nodes]) * cy[nodes]
    norm = np.sqrt((hx * hx + hy * hy) + 1.0)
    normals = np.stack([-hx / norm, -hy / norm, 1.0 / norm], axis=1)
    frames = contact_frames(normals) if len(nodes) else np.zeros((0, 3, 3))
    return nodes, phi, depth, frames


def heightfield_system(blk) -> PackedSystem:
    b = heightfield_rhs(blk)
    nodes, phi, depth, frames = heightfield_contacts(blk)
    n_c = nodes.shape[0]
    mu = np.full(n_c, blk.mu)
    return make_packed(blk.n, blk.A.indptr, blk.A.indices, blk.A.data, b, 3 * nodes, np.full(n_c, -1),
                       frames.reshape(-1), mu, mu, phi)


def _cg_fallback(cube, b):
    """harness.py:586-593: v_hat = cg(A, b, rtol=1e-10, maxiter=10 n)."""
    from scipy.sparse.linalg import cg

    v, _ = cg(cube.A, b, rtol=1e-10, maxiter=10 * cube.n)
    return v


def oracle_steps(cube, steps, residual_tol=1e-8, max_iters=500, chebyshev=False, record=None, **cfg_extra):
    """Advance ``cube`` ``steps`` times on the host; returns the summed
    contact-iterations. ``record`` (list) receives per-step dicts;
    ``cfg_extra`` are further ``Config`` fields (operator, step_strategy, ...)."""
    prev = None
    ci = 0
    cfg = O.Config(residual_tol=residual_tol, max_iters=max_iters, chebyshev=chebyshev, **cfg_extra)
    for _ in range(steps):
        ps = fem_system(cube)
        s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64),
                     ps.col_j.astype(np.int64), ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
        warm = np.zeros(ps.n) if prev is None else prev
        try:
            v, lam, rep = O.solve(s, cfg, warm)
            it, div = rep.iterations, False
        except O.OracleDivergence as e:
            v, lam = _cg_fallback(cube, ps.b), np.zeros(3 * ps.n_c)
            it, div = len(e.residual_trace), True
        ci += ps.n_c * it
        if record is not None:
            record.append(dict(n_c=ps.n_c, iterations=it, diverged=div, v=v.copy(), lam=lam.copy()))
        fem_advance(cube, v)
        prev = v
    return ci


def reference_steps(cube, steps, residual_tol=1e-8, max_iters=500, chebyshev=False, k_v=1e5, record=None):
    """Advance ``cube`` through the reference's own contact pipeline and
    solver; returns the summed contact-iterations (n_c x V-FPI iterations;
    a diverged solve counts the iterations its residual trace recorded)."""
    from condsim.contacts import Geometry, NodeProxy, Plane, StabilizationParams, augment_dynamics, \
        detect_contacts, nodalize
    from condsim.dynamics import Body, SystemState
    from condsim.errors import DivergenceError
    from condsim.solver import SolverConfig, solve_vfpi
    from condsim.sparse import SparseSymmetric

    nn = cube.n // 3
    bodies = [Body("particle3", float(cube.m[3 * k]), 3 * k, 3 * k) for k in range(nn)]
    geom = Geometry(planes=[Plane(np.zeros(3), np.array([0.0, 0.0, 1.0]))],
                    node_proxies=[NodeProxy(k, 3 * k, 0.0) for k in range(nn)])
    a_o = SparseSymmetric.from_scipy(cube.A)
    cfg = SolverConfig(residual_tol=residual_tol, max_iters=max_iters, chebyshev=chebyshev)
    prev = None
    ci = 0
    for step in range(steps):
        b = fem_rhs(cube)
        state = SystemState(cube.x.ravel().copy(), cube.v.ravel().copy(), step, cube.dt)
        raw = detect_contacts(state, bodies, geom)
        nodal = nodalize(raw, state, bodies, k_v, cube.mu, None, StabilizationParams(dt=cube.dt))
        aug = augment_dynamics(a_o, b, nodal)
        warm = np.zeros(aug.n)
        if prev is not None:  # harness._warm_velocity (no virtual nodes on FEM nodes)
            warm[: cube.n] = prev[: cube.n]
        n_c = len(nodal.contacts)
        try:
            v, lam, rep = solve_vfpi(aug, cfg, warm)
            it, div = rep.iterations, False
        except DivergenceError as e:
            v = np.concatenate([_cg_fallback(cube, b), np.zeros(aug.n - cube.n)])
            lam = np.zeros((n_c, 3))
            it, div = len(e.residual_trace or []), True
        ci += n_c * it
        if record is not None:
            record.append(dict(n_c=n_c, iterations=it, diverged=div, v=np.asarray(v).copy()))
        fem_advance(cube, v)
        prev = v
    return ci
