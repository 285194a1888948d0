"""Parity at BASELINE's full sizes (-m gpu; each case runs the CPU oracle for a
few iterations only, so the whole file takes about two minutes):

* configs[3]: the 64^3-node heightfield block (786,432 DOF, 24.6M entries,
  4,096 contacts), 4 plain V-FPI iterations, GPU == oracle bit for bit;
* configs[2]: a 1024-scene batch in contact, every distinct scene bit-equal
  to its oracle solve (iterations, v, lam);
* configs[4]: the 8x8x4 pile of 16^3-node cubes stacked in contact
  (3.1M DOF + 43k virtual nodes, 82M entries, 60k contacts): device
  detection/nodalization == host restatement, device augmentation == the
  reference's scipy expression, and 2 plain V-FPI iterations GPU == oracle,
  all bit for bit.
"""

import numpy as np
import pytest

from oracle import vfpi_oracle as O


def _oracle_solve(ps, iters):
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, O.Config(residual_tol=1e-8, max_iters=iters), np.zeros(ps.n))


@pytest.mark.gpu
def test_cfg3_full_size_bitwise():
    from oracle.fem_host import heightfield_system
    from paper_2201_09212_b200.scenes import HeightfieldBlock
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = heightfield_system(HeightfieldBlock(nx=64))
    assert ps.n == 786432 and ps.n_c > 3000
    v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-8, max_iters=4), np.zeros(ps.n))
    vo, lo, ro = _oracle_solve(ps, 4)
    assert rep.iterations == ro.iterations == 4
    assert np.array_equal(v, vo) and np.array_equal(lam, lo)


@pytest.mark.gpu
def test_cfg4_full_size_pipeline_bitwise():
    from paper_2201_09212_b200.pile import CubePile, PileStepper
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    pile = CubePile(gap=0.005, jitter=0.002, gap_z=0.0, jitter_z=0.0, k_v=100.0)  # layers stacked in contact
    stepper = PileStepper(pile)
    dc = stepper.device_contacts()
    from oracle import pile_host as H

    hc = H.contacts(pile)
    assert hc.n_ground == 16384 and hc.n_face > 40000
    assert (hc.n_ground, hc.n_face, hc.n_virtual) == (dc.n_ground, dc.n_face, dc.n_virtual)
    for name in ("col_i", "col_j", "frames", "phi"):
        assert np.array_equal(getattr(hc, name), getattr(dc, name)), name
    assert np.array_equal(hc.jv.indices, dc.jv.indices) and np.array_equal(hc.jv.data, dc.jv.data)
    from paper_2201_09212_b200.augment import augment_arrays

    b_o = H.rhs(pile)
    dp, di, dx = augment_arrays(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, hc.jv, pile.k_v)  # device
    p, i, x, b = O.augment(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, b_o, hc.jv, pile.k_v)
    assert np.array_equal(dp, p) and np.array_equal(di, i) and np.array_equal(dx, x)
    ps = H.system(pile, hc, b_o)
    v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-8, max_iters=2), np.zeros(ps.n))
    vo, lo, ro = _oracle_solve(ps, 2)
    assert rep.iterations == ro.iterations == 2
    assert np.array_equal(v, vo) and np.array_equal(lam, lo)


@pytest.mark.gpu
def test_cfg2_full_batch_bitwise():
    """configs[2]: a batch of 1024 FEM scenes (16 distinct cubes pressed into
    the plane and moving down, replicated) in one scene-batch solve; every
    distinct scene equals its oracle solve bit for bit with the same iteration
    count, and every replica equals its class."""
    from oracle.fem_host import fem_system
    from paper_2201_09212_b200.batch import solve_scenes
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    g = np.random.default_rng(7)
    base = []
    for _ in range(16):
        c = FemCube(E=float(g.uniform(5e4, 2e5)), drop=0.0, yaw=float(g.uniform(0, 2 * np.pi)))
        c.x = c.X.copy()
        c.x[:, 2] -= 5e-4
        c.v[:, 2] = -0.3
        base.append(fem_system(c))
    scenes = [base[k % 16] for k in range(1024)]
    res, rep = solve_scenes(scenes, SolverConfig(residual_tol=1e-8, max_iters=500))
    for k in range(16):
        vo, lo, ro = _oracle_solve(base[k], 500)
        v, lam, r = res[k]
        assert r.iterations == ro.iterations and r.converged == ro.converged, k
        assert np.array_equal(v, vo) and np.array_equal(lam, lo), k
    for k in range(16, 1024):
        assert np.array_equal(res[k][0], res[k % 16][0]) and res[k][2].iterations == res[k % 16][2].iterations
