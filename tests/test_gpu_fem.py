"""Multi-step parity on the FEM configs: the GPU solve and the CPU oracle are
stepped side by side through contact onset (configs[0] shape) and must take
the identical number of V-FPI iterations at every step, with final states
equal to 1e-9 relative (configs[0]/[2] are parity-friendly)."""

import numpy as np
import pytest

from oracle.fem_host import fem_advance, fem_system, heightfield_system

pytestmark = pytest.mark.gpu


def _oracle_step(ps, cfg, warm):
    from oracle import vfpi_oracle as O

    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, O.Config(**{k: getattr(cfg, k) for k in (
        "operator", "step_strategy", "residual_tol", "max_iters", "chebyshev", "cheby_start", "under_relax",
        "omega", "fixed_alpha", "consistency_factor")}), warm)


@pytest.mark.parametrize("cheb", [False, True])
def test_config0_cube_steps_match_oracle(cheb):
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=cheb)
    gpu, cpu = FemCube(), FemCube()
    wg = wc = None
    contact_steps = 0
    for step in range(125):
        pg, pc = fem_system(gpu), fem_system(cpu)
        assert pg.n_c == pc.n_c, step
        vg, lg, rg = solve_packed(pg, cfg, np.zeros(pg.n) if wg is None else wg)
        vc, lc, rc = _oracle_step(pc, cfg, np.zeros(pc.n) if wc is None else wc)
        assert rg.iterations == rc.iterations, (step, rg.iterations, rc.iterations)
        assert rg.converged == rc.converged
        contact_steps += pg.n_c > 0
        fem_advance(gpu, vg)
        fem_advance(cpu, vc)
        wg, wc = vg, vc
    assert contact_steps >= 20
    assert np.linalg.norm(gpu.x - cpu.x) <= 1e-9 * np.linalg.norm(cpu.x)


def test_config2_scene_batch_steps_match_oracle():
    from paper_2201_09212_b200.batch import solve_scenes
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    g = np.random.default_rng(22)
    params = [dict(nx=6, E=float(g.uniform(5e4, 2e5)), drop=float(g.uniform(0.002, 0.01)),
                   yaw=float(g.uniform(0, 2 * np.pi))) for _ in range(6)]
    gpu = [FemCube(**p) for p in params]
    cpu = [FemCube(**p) for p in params]
    cfg = SolverConfig(residual_tol=1e-8, max_iters=500)
    wg = [np.zeros(c.n) for c in gpu]
    wc = [np.zeros(c.n) for c in cpu]
    touched = 0
    for step in range(70):
        res, _ = solve_scenes([fem_system(c) for c in gpu], cfg, warms=wg)
        for k in range(len(gpu)):
            vc, lc, rc = _oracle_step(fem_system(cpu[k]), cfg, wc[k])
            v, lam, r = res[k]
            assert r.iterations == rc.iterations, (step, k)
            touched += lam.shape[0] > 0
            fem_advance(gpu[k], v)
            fem_advance(cpu[k], vc)
            wg[k], wc[k] = v, vc
    assert touched > 0
    for a, b in zip(gpu, cpu):
        assert np.linalg.norm(a.x - b.x) <= 1e-9 * np.linalg.norm(b.x)


@pytest.mark.parametrize("cheb", [False, True])
def test_config3_heightfield_block_matches_oracle(cheb):
    """configs[3]-shaped system (heightfield S-contacts with per-contact frames) at
    nx=8, through the single-system path: identical iterations, v bitwise (plain)."""
    from paper_2201_09212_b200.scenes import HeightfieldBlock
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = heightfield_system(HeightfieldBlock(nx=8))
    cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=cheb)
    v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
    vc, lc, rc = _oracle_step(ps, cfg, np.zeros(ps.n))
    assert rep.iterations == rc.iterations and rep.converged == rc.converged
    if cheb:
        assert np.allclose(v, vc, rtol=1e-9, atol=1e-12)
        assert np.allclose(lam, lc, rtol=1e-9, atol=1e-9)
    else:
        assert np.array_equal(v, vc)
        assert np.array_equal(lam, lc)


def test_device_fem_pipeline_matches_host_pipeline():
    """vfpi_fem_step (b, detection, solve, integration on the device) against the
    host pipeline (FemCube.system -> solve_scenes -> FemCube.advance): identical
    state bits after free fall, touchdown and contact steps."""
    from paper_2201_09212_b200.batch import solve_scenes
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    def make():
        return [FemCube(nx=5, E=e, drop=d, yaw=y) for e, d, y in ((6e4, 0.004, 0.3), (1.5e5, 0.006, 1.1),
                                                                  (1e5, 0.002, 2.0))]

    cfg = SolverConfig(residual_tol=1e-8, max_iters=200)
    host = make()
    dev = FemBatch(make())
    warms = [np.zeros(c.n) for c in host]
    saw_contacts = False
    for step in range(45):
        systems = [fem_system(c) for c in host]
        res, _ = solve_scenes(systems, cfg, warms=warms)
        st = dev.step(cfg, per_scene=True)
        assert st["contacts"] == sum(s.n_c for s in systems)
        saw_contacts |= st["contacts"] > 0
        for k, (c, r) in enumerate(zip(host, res)):
            v, lam, rep = r
            assert st["iterations_per_scene"][k] == rep.iterations
            fem_advance(c, v)
            warms[k] = v
        x, vel = dev.state()
        for k, c in enumerate(host):
            assert np.array_equal(x[k], c.x), f"step {step} scene {k}"
            assert np.array_equal(vel[k], c.v), f"step {step} scene {k}"
    assert saw_contacts
    dev.close()
