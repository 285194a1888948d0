"""Generate golden input/output vectors from the REFERENCE package.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each ``<case>.npz`` holds one augmented system exactly as the reference's
``solve_vfpi`` (``solver.py:345-461``) consumed it — the CSC arrays of
``aug.a``, ``aug.b``, ``col_i/col_j``, ``frames``, per-contact
``mu/mu2/phi``, the warm start and the ``SolverConfig`` — plus the reference's
outputs (``v``, ``lam``, iterations, residual trace, converged/diverged,
consistency, SCC residuals) and per-operator reference outputs on seeded
inputs (``spmv``, ``row_norms_sq``, ``step_matrix_frobenius``,
``surrogate_gamma``, ``apply_jc``, ``apply_jc_t``, ``contact_solve_oneshot``
for all three operators, ``inverse_contact``).

Systems come from the reference's own generators (``testing.py``), its
scenario pipeline (``harness.build_scene`` → ``assemble_step`` →
``detect_contacts`` → ``nodalize`` → ``augment_dynamics``, warm-started as
``harness._warm_velocity``), and a reduced configs[1] rigid-body system built
through the reference ``nodalize``/``augment_dynamics``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

import condsim.harness as H  # noqa: E402
from condsim.contacts import (  # noqa: E402
    Contact,
    RawContact,
    apply_jc,
    apply_jc_t,
    augment_dynamics,
    contact_frame,
    detect_contacts,
    nodalize,
)
from condsim.dynamics import Body, SystemState, assemble_step, integrate  # noqa: E402
from condsim.errors import DivergenceError  # noqa: E402
from condsim.solver import (  # noqa: E402
    SolverConfig,
    contact_solve_oneshot,
    inverse_contact,
    solve_vfpi,
    step_matrix_frobenius,
    surrogate_gamma,
)
from condsim.sparse import SparseSymmetric, row_norms_sq, spmv  # noqa: E402
from condsim.testing import build_augmented, random_contact_set, random_spd  # noqa: E402

CFG_KEYS = ("operator", "step_strategy", "residual_tol", "max_iters", "chebyshev", "cheby_start",
            "under_relax", "omega", "fixed_alpha", "consistency_factor")


def _params(aug):
    cs = aug.contacts.contacts if aug.contacts is not None else []
    mu = np.array([c.mu for c in cs], dtype=float)
    mu2 = np.array([c.mu2 if c.mu2 is not None else c.mu for c in cs], dtype=float)
    phi = np.array([c.phi_n for c in cs], dtype=float)
    return mu, mu2, phi


def save_case(name, aug, cfg: SolverConfig, warm, w_cached=None, seed=0, extra=None):
    a = aug.a
    n_c = len(aug.contacts.contacts) if aug.contacts is not None else 0
    mu, mu2, phi = _params(aug)
    rec = dict(
        n=np.int64(aug.n), indptr=a.indptr.astype(np.int32), indices=a.indices.astype(np.int32),
        data=a.data.astype(float), b=aug.b.astype(float),
        col_i=(aug.col_i if n_c else np.zeros(0)).astype(np.int32),
        col_j=(aug.col_j if n_c else np.zeros(0)).astype(np.int32),
        frames=(aug.frames if n_c else np.zeros((0, 3, 3))).reshape(-1).astype(float),
        mu=mu, mu2=mu2, phi=phi, warm=np.asarray(warm, dtype=float),
        cfg=json.dumps({k: getattr(cfg, k) for k in CFG_KEYS}),
    )
    if w_cached is not None:
        rec["w_cached"] = w_cached.w
    try:
        v, lam, rep = solve_vfpi(aug, cfg, warm, w_cached=w_cached)
        rec.update(
            out_v=v, out_lam=np.asarray(lam, dtype=float).reshape(-1), out_iterations=np.int64(rep.iterations),
            out_trace=np.array(rep.residual_trace, dtype=float), out_converged=np.int64(rep.converged),
            out_diverged=np.int64(0), out_consistency=np.float64(rep.consistency),
            out_scc=(rep.scc_residuals if rep.scc_residuals is not None else np.zeros(0)),
        )
    except DivergenceError as exc:
        rec.update(out_diverged=np.int64(1), out_trace=np.array(exc.residual_trace, dtype=float),
                   out_iterations=np.int64(len(exc.residual_trace)))
    # per-operator reference outputs on seeded inputs
    g = np.random.default_rng(seed + 7)
    x = g.standard_normal(aug.n)
    rec["op_x"] = x
    rec["op_spmv"] = spmv(a, x)
    rec["op_rns"] = row_norms_sq(a)
    rec["op_diag"] = a.diagonal()
    if np.all(rec["op_rns"] > 0):
        rec["op_w_strict"] = step_matrix_frobenius(a, aug, False).w
        rec["op_w_prox"] = step_matrix_frobenius(a, aug, True).w
    if n_c:
        w = step_matrix_frobenius(a, aug, cfg.operator == "proximal")
        gam = surrogate_gamma(w, aug, cfg.omega)
        rec["op_gamma"] = gam.gamma
        rec["op_jc"] = apply_jc(aug, x).reshape(-1)
        lam_r = g.standard_normal((n_c, 3))
        rec["op_lam"] = lam_r.reshape(-1)
        rec["op_jct"] = apply_jc_t(aug, lam_r)
        eta = g.standard_normal((n_c, 3)) * 3.0
        rec["op_eta"] = eta.reshape(-1)
        for op in ("strict", "proximal", "strict-anisotropic"):
            key = "op_oneshot_" + op.replace("-", "_")
            rec[key] = contact_solve_oneshot(gam, eta, phi, mu, op, mu2).reshape(-1)
        rec["op_inverse"] = inverse_contact(aug, x, 1e-3, "proximal").reshape(-1)
    if extra:
        rec.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    return rec


def random_cases():
    rng = np.random.default_rng(12345)
    out = []
    specs = [
        ("rand_strict_plain", dict(operator="strict", residual_tol=1e-8, max_iters=3000)),
        ("rand_strict_cheb", dict(operator="strict", residual_tol=1e-8, max_iters=3000, chebyshev=True)),
        ("rand_prox_cheb", dict(operator="proximal", residual_tol=1e-8, max_iters=3000, chebyshev=True)),
        ("rand_prox_plain", dict(operator="proximal", residual_tol=1e-6, max_iters=3000)),
        ("rand_aniso_cheb", dict(operator="strict-anisotropic", residual_tol=1e-8, max_iters=3000, chebyshev=True)),
        ("rand_bb1", dict(step_strategy="bb1", residual_tol=1e-8, max_iters=3000)),
        ("rand_bb2", dict(step_strategy="bb2", residual_tol=1e-8, max_iters=3000)),
        ("rand_bbalt", dict(step_strategy="bb-alternating", residual_tol=1e-8, max_iters=3000)),
        ("rand_fixed_default", dict(step_strategy="fixed-alpha", residual_tol=1e-6, max_iters=3000)),
        ("rand_omega_prox", dict(operator="proximal", residual_tol=1e-10, max_iters=5000, chebyshev=True, omega=1e-3)),
        ("rand_tol0_200", dict(operator="strict", residual_tol=0.0, max_iters=200)),
        ("rand_maxit0", dict(operator="strict", residual_tol=1e-8, max_iters=0)),
        ("rand_cheb_ls3", dict(operator="strict", residual_tol=1e-9, max_iters=3000, chebyshev=True,
                               cheby_start=3, under_relax=0.7)),
    ]
    for k, (name, kw) in enumerate(specs):
        n, contacts = random_contact_set(rng, n_nodes=int(rng.integers(6, 30)))
        if kw.get("operator") == "strict-anisotropic":
            for c in contacts:
                c.mu2 = float(rng.uniform(0.1, 1.0))
        for c in contacts:
            c.phi_n = float(-abs(rng.standard_normal()) * 0.05)
        a = random_spd(rng, n)
        b = rng.standard_normal(n) * 3.0
        aug = build_augmented(a, b, contacts)
        warm = rng.standard_normal(n) * 0.1 if k % 2 else np.zeros(n)
        save_case(name, aug, SolverConfig(**kw), warm, seed=k)
        out.append(name)
    # proximal at the TestSolveVfpi.test_consistency_at_convergence shape (phi = 0)
    for k in range(3):
        n, contacts = random_contact_set(rng)
        a = random_spd(rng, n)
        aug = build_augmented(a, rng.standard_normal(n), contacts)
        name = f"rand_prox_conv{k}"
        save_case(name, aug, SolverConfig(operator="proximal", residual_tol=1e-8, max_iters=3000,
                                          chebyshev=bool(k != 1)), np.zeros(n), seed=40 + k)
        out.append(name)
    # larger random system with many contacts (multi-block partition on GPU)
    n, contacts = random_contact_set(rng, n_nodes=600, n_contacts=250)
    a = random_spd(rng, n, density=0.0015)
    aug = build_augmented(a, rng.standard_normal(n), contacts)
    save_case("rand_large_strict", aug, SolverConfig(residual_tol=1e-9, max_iters=4000, chebyshev=True),
              np.zeros(n), seed=99)
    out.append("rand_large_strict")
    # contact-free (TestSolveVfpi.test_contact_free_matches_direct_solve shape)
    a = random_spd(rng, 20)
    aug = build_augmented(a, rng.standard_normal(20), [])
    save_case("free_cheb", aug, SolverConfig(residual_tol=1e-10, max_iters=5000, chebyshev=True), np.zeros(20))
    out.append("free_cheb")
    # divergence (fixed alpha far above 2/lambda_max)
    a = random_spd(rng, 6)
    aug = build_augmented(a, rng.standard_normal(6), [])
    with np.errstate(over="ignore", invalid="ignore"):
        save_case("diverge_fixed", aug, SolverConfig(step_strategy="fixed-alpha", fixed_alpha=1e3, max_iters=5000),
                  np.zeros(6))
    out.append("diverge_fixed")
    # divergence with contacts
    n, contacts = random_contact_set(rng, n_nodes=8, n_contacts=3)
    a = random_spd(rng, n)
    aug = build_augmented(a, rng.standard_normal(n), contacts)
    with np.errstate(over="ignore", invalid="ignore"):
        save_case("diverge_contacts", aug, SolverConfig(step_strategy="fixed-alpha", fixed_alpha=50.0,
                                                        max_iters=5000, chebyshev=True), np.zeros(n))
    out.append("diverge_contacts")
    # resting particle (TestSolveVfpi.test_resting_particle_equilibrium shape)
    a = SparseSymmetric.from_dense(200.0 * np.eye(3))
    frame = contact_frame(np.array([0.0, 0.0, 1.0]))
    aug = build_augmented(a, np.array([0.0, 0.0, -9.81]), [Contact("S", ("orig", 0), frame, 0.0, 0.0)])
    save_case("resting", aug, SolverConfig(residual_tol=1e-12, max_iters=200), np.zeros(3))
    out.append("resting")
    # cached step matrix
    n, contacts = random_contact_set(rng, n_nodes=10, n_contacts=4)
    a = random_spd(rng, n)
    aug = build_augmented(a, rng.standard_normal(n), contacts)
    w = step_matrix_frobenius(a, aug, False)
    w.w = w.w * 0.9
    save_case("w_cached", aug, SolverConfig(residual_tol=1e-8, max_iters=3000), np.zeros(n), w_cached=w)
    out.append("w_cached")
    return out


def scenario_cases():
    """Per-step systems from the reference scenario pipeline (``harness.run``
    ``harness.py:526-619``), at the acceptance configuration."""
    out = []
    picks = {
        "lattice_drag": [0, 3, 12],
        "box_slide": [0, 5],
        "particle_stack": [2, 20],
        "anisotropic_slide": [1, 10],
        "lattice_invertible": [2],
    }
    for name, steps in picks.items():
        s = H.load_scenario(os.path.join(REF, "scenarios", name + ".json"))
        op = "strict-anisotropic" if name == "anisotropic_slide" else "strict"
        rcfg = H.RunConfig(solver="cond", operator=op, residual_tol=1e-4 if name != "anisotropic_slide" else 1e-7,
                           chebyshev=True, kv=1e5 if name != "anisotropic_slide" else 1e3, max_iters=4000)
        scene = H.build_scene(s, rcfg)
        state, bodies = scene.state, scene.bodies
        n = state.v.shape[0]
        prev = None
        for step in range(max(steps) + 1):
            f_ext = H.external_force(scene, step * s.step_size, n)
            asm = assemble_step(state, bodies, scene.constraints, f_ext)
            raw = detect_contacts(state, bodies, scene.geometry)
            nodal = nodalize(raw, state, bodies, scene.k_v, scene.mu, scene.mu2, scene.stab)
            aug = augment_dynamics(asm.a, asm.b, nodal)
            warm = H._warm_velocity(prev, aug, asm.n)
            scfg = H._solver_cfg(rcfg)
            if step in steps:
                case = f"scn_{name}_s{step}"
                save_case(case, aug, scfg, warm, seed=step)
                out.append(case)
            v, lam, rep = solve_vfpi(aug, scfg, warm)
            state = integrate(state, v[: asm.n], bodies)
            prev = v[: asm.n]
    return out


def rigid_pile_case(n_bodies=256, n_contacts=1024, seed=2201, k_v=1e5):
    """configs[1] shape at reduced size, through the reference ``nodalize``
    (``contacts.py:271-321``) and ``augment_dynamics`` (``:343-375``).
    Draw order matches ``paper_2201_09212_b200.scenes.rigid_contact_system``."""
    rng = np.random.default_rng(seed)
    mass = rng.uniform(0.5, 2.0, n_bodies)
    inert = rng.uniform(0.01, 0.1, (n_bodies, 3))
    quat = rng.standard_normal((n_bodies, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    pairs = rng.integers(0, n_bodies - 1, (n_contacts, 2))
    pairs[:, 1] += pairs[:, 1] >= pairs[:, 0]  # distinct second body
    normals = rng.standard_normal((n_contacts, 3))
    levers = rng.uniform(-0.1, 0.1, (n_contacts, 3))
    mus = rng.uniform(0.2, 0.8, n_contacts)
    b_o = rng.standard_normal(6 * n_bodies)

    from condsim.dynamics import _quat_to_rot
    import scipy.sparse as sps

    bodies, q = [], []
    rows, cols, vals = [], [], []
    for k in range(n_bodies):
        bodies.append(Body("rigid6", float(mass[k]), 7 * k, 6 * k, np.diag(inert[k])))
        q.append(np.zeros(3))
        q.append(quat[k])
        rot = _quat_to_rot(quat[k])
        for off, blk in ((6 * k, mass[k] * np.eye(3)), (6 * k + 3, rot @ np.diag(inert[k]) @ rot.T)):
            ii, jj = np.meshgrid(range(off, off + 3), range(off, off + 3), indexing="ij")
            rows.append(ii.ravel())
            cols.append(jj.ravel())
            vals.append(blk.ravel())
    n_o = 6 * n_bodies
    a_o = sps.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n_o, n_o)).tocsc()
    a_o = SparseSymmetric.from_scipy(a_o)
    state = SystemState(np.concatenate(q), np.zeros(n_o), 0, 1e-3)
    raw = [RawContact(point=levers[m], normal=normals[m], depth=0.0,
                      first=("rigid", int(pairs[m, 0]), m), second=("rigid", int(pairs[m, 1]), m))
           for m in range(n_contacts)]
    nodal = nodalize(raw, state, bodies, k_v, 0.5)
    for m, c in enumerate(nodal.contacts):
        c.mu = float(mus[m])
    aug = augment_dynamics(a_o, b_o, nodal)
    return aug


def fem_cases():
    """configs[0]-shaped FEM cubes (the repo's own linear-tet assembly — the
    reference has none), stepped with the reference solve_vfpi; the contacts
    of the saved steps come from the reference detect_contacts / nodalize /
    augment_dynamics on the same state, so they pin oracle.fem_host.fem_contacts."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from condsim.contacts import Geometry, NodeProxy, Plane, StabilizationParams
    from oracle.fem_host import fem_advance, fem_system
    from paper_2201_09212_b200.scenes import FemCube

    out = []
    for tag, kw, picks in (("fem6", dict(nx=6, drop=0.01), (45, 47, 60)),
                           ("fem10", dict(nx=10), (101, 104))):
        cube = FemCube(**kw)
        nn = cube.n // 3
        bodies = [Body("particle3", float(cube.m[3 * k]), 3 * k, 3 * k) for k in range(nn)]
        geom = Geometry(planes=[Plane(np.zeros(3), np.array([0.0, 0.0, 1.0]))],
                        node_proxies=[NodeProxy(k, 3 * k, 0.0) for k in range(nn)])
        a_o = SparseSymmetric.from_scipy(cube.A)
        prev = None
        for step in range(max(picks) + 1):
            ps = fem_system(cube)
            state = SystemState(cube.x.ravel().copy(), cube.v.ravel().copy(), step, cube.dt)
            raw = detect_contacts(state, bodies, geom)
            nodal = nodalize(raw, state, bodies, 1e5, 0.5, None, StabilizationParams(dt=cube.dt))
            aug = augment_dynamics(a_o, ps.b.copy(), nodal)
            warm = np.zeros(aug.n) if prev is None else prev
            cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=(tag == "fem6"))
            if step in picks and aug.contacts.contacts:
                case = f"{tag}_s{step}"
                save_case(case, aug, cfg, warm, seed=step,
                          extra=dict(fem_x=cube.x.copy(), fem_v=cube.v.copy(),
                                     fem_kw=json.dumps(kw)))
                out.append(case)
            v, lam, rep = solve_vfpi(aug, cfg, warm)
            fem_advance(cube, v)
            prev = v
    return out


def main():
    names = fem_cases()
    names += random_cases()
    names += scenario_cases()
    aug = rigid_pile_case()
    save_case("rigid_pile_256", aug, SolverConfig(residual_tol=1e-8, max_iters=300), np.zeros(aug.n), seed=5)
    names.append("rigid_pile_256")
    save_case("rigid_pile_256_cheb", aug, SolverConfig(residual_tol=1e-8, max_iters=60, chebyshev=True),
              np.zeros(aug.n), seed=6)
    names.append("rigid_pile_256_cheb")
    with open(os.path.join(HERE, "INDEX.json"), "w") as f:
        json.dump(sorted(names), f, indent=1)
    print(len(names), "cases")


if __name__ == "__main__":
    main()
