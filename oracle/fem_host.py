"""Host restatements of the FEM step pipeline -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s CPU legs (``cpu_baseline`` /
``--impl reference``) import this module; the product path steps scenes on
the device (``fembatch.FemBatch`` / ``vfpi_fem_step``).

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

from . import vfpi_oracle as O


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
        ps = cube.system()
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
        cube.advance(v)
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
        b = cube.rhs()
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
        cube.advance(v)
        prev = v
    return ci
