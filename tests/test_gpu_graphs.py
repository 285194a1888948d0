"""Captured setup graphs (vfpi_api.cu run_setup_phase): the first solve of a
shape runs eagerly, the second is captured, later ones replay the graph. A
replay on new values (same structure, same staging buffers) must give the
oracle's answer bit for bit, and launch accounting must not change."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle(ps, cfg, warm):
    from oracle import vfpi_oracle as O

    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, O.Config(**{k: getattr(cfg, k) for k in (
        "operator", "step_strategy", "residual_tol", "max_iters", "chebyshev", "cheby_start", "under_relax",
        "omega", "fixed_alpha", "consistency_factor")}), warm)


def test_setup_graph_replay_matches_oracle():
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.scenes import rigid_contact_system
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed
    from paper_2201_09212_b200.system import make_packed

    base = rigid_contact_system(48, 160, 7)
    cfg = SolverConfig(residual_tol=1e-9, max_iters=80)
    h = _lib.handle(0)
    rng = np.random.default_rng(11)
    outs, launches = [], []
    for k in range(4):
        scale = 1.0 if k < 2 else 1.0 + 0.25 * k
        b = base.b if k < 2 else rng.standard_normal(base.n)
        ps = make_packed(base.n, base.indptr, base.indices, base.data * scale, b, base.col_i, base.col_j,
                         base.frames, base.mu, base.mu2, base.phi)
        l0 = h.launches()
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        launches.append(h.launches() - l0)
        vo, lo, ro = _oracle(ps, cfg, np.zeros(ps.n))
        assert rep.iterations == ro.iterations
        assert np.array_equal(v, vo), f"solve {k}"
        assert np.array_equal(lam, lo), f"solve {k}"
        outs.append(v)
    assert np.array_equal(outs[0], outs[1])
    assert len(set(launches)) == 1, launches
