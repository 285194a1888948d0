"""Error behaviour, edge cases, determinism, concurrency and full-size
properties of the CUDA path (reference semantics: solver.py, errors.py)."""

import threading

import numpy as np
import pytest

from gpu_util import relerr

pytestmark = pytest.mark.gpu


def _sys(a_dense, b, contacts=()):
    import scipy.sparse as sp

    from paper_2201_09212_b200.system import make_packed

    a = sp.csc_matrix(np.asarray(a_dense, float))
    a.sum_duplicates()
    n = a.shape[0]
    ci = [c[0] for c in contacts]
    cj = [c[1] for c in contacts]
    fr = [np.eye(3).ravel() for _ in contacts]
    mu = [0.5 for _ in contacts]
    return make_packed(n, a.indptr, a.indices, a.data, b, ci, cj, np.array(fr).reshape(-1), mu)


def test_resting_particle_equilibrium():
    from paper_2201_09212_b200.contacts import contact_frame
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed
    from paper_2201_09212_b200.system import make_packed
    import scipy.sparse as sp

    a = sp.csc_matrix(200.0 * np.eye(3))
    fr = contact_frame(np.array([0.0, 0.0, 1.0]))
    ps = make_packed(3, a.indptr, a.indices, a.data, [0.0, 0.0, -9.81], [0], [-1], fr.ravel(), [0.0])
    v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-12, max_iters=200), np.zeros(3))
    assert rep.converged
    assert np.allclose(v, 0.0, atol=1e-10)
    assert np.isclose(lam[0, 0], 9.81, atol=1e-8)


def test_zero_row_norm_raises_invalid_matrix():
    from paper_2201_09212_b200.errors import InvalidMatrixError
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    a = np.diag([1.0, 0.0, 2.0])
    with pytest.raises(InvalidMatrixError):
        solve_packed(_sys(a, np.ones(3)), SolverConfig(), np.zeros(3))
    # fixed-alpha never computes the Frobenius matrix (solver.py:367-369)
    solve_packed(_sys(a, np.ones(3)), SolverConfig(step_strategy="fixed-alpha", fixed_alpha=0.1, max_iters=5),
                 np.zeros(3))


def test_tie_violation_from_cached_w():
    from paper_2201_09212_b200.errors import InvalidMatrixError
    from paper_2201_09212_b200.solver import SolverConfig, StepMatrix, solve_vfpi, surrogate_gamma

    ps = _sys(np.eye(3), np.zeros(3), [(0, -1)])
    with pytest.raises(InvalidMatrixError):
        surrogate_gamma(StepMatrix(np.array([1.0, 2.0, 3.0])), ps)
    with pytest.raises(InvalidMatrixError):
        solve_vfpi(ps, SolverConfig(), np.zeros(3), w_cached=StepMatrix(np.array([1.0, 2.0, 3.0])))


def test_shared_node_column_rejected():
    from paper_2201_09212_b200.errors import UnsupportedInputError
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _sys(np.eye(9) * 4.0, np.ones(9), [(0, 3), (3, 6)])
    with pytest.raises(UnsupportedInputError):
        solve_packed(ps, SolverConfig(), np.zeros(9))


def test_overlapping_scatter_matches_add_at():
    from paper_2201_09212_b200.contacts import apply_jc_t

    ps = _sys(np.eye(9), np.zeros(9), [(0, 3), (3, 6), (0, -1)])
    lam = np.arange(9, dtype=float).reshape(3, 3) + 1.0
    ref = np.zeros(9)
    for m, (i, j) in enumerate([(0, 3), (3, 6), (0, -1)]):
        ref[i:i + 3] += lam[m]
    for m, (i, j) in enumerate([(0, 3), (3, 6), (0, -1)]):
        if j >= 0:
            ref[j:j + 3] -= lam[m]
    assert np.array_equal(apply_jc_t(ps, lam), ref)


def test_dimension_mismatch_and_override():
    from paper_2201_09212_b200.errors import DimensionMismatchError
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed, solve_vfpi

    ps = _sys(np.eye(3), np.zeros(3))
    with pytest.raises(DimensionMismatchError):
        solve_packed(ps, SolverConfig(), np.zeros(4))
    with pytest.raises(NotImplementedError):
        solve_vfpi(ps, SolverConfig(), np.zeros(3), project_override=lambda *a: a[0])


def test_empty_system_and_zero_iterations():
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _sys(np.eye(3) * 2.0, np.array([2.0, 4.0, 6.0]))
    v, lam, rep = solve_packed(ps, SolverConfig(max_iters=0), np.zeros(3))
    assert rep.iterations == 0 and not rep.converged
    assert np.array_equal(v, np.zeros(3))
    assert np.isclose(rep.consistency, np.linalg.norm([2.0, 4.0, 6.0]))


def _rigid(nb, nc, seed=7):
    from paper_2201_09212_b200.scenes import rigid_contact_system

    return rigid_contact_system(n_bodies=nb, n_contacts=nc, seed=seed)


def test_deterministic_bits():
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _rigid(512, 2048)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=200, chebyshev=True)
    v1, l1, r1 = solve_packed(ps, cfg, np.zeros(ps.n))
    v2, l2, r2 = solve_packed(ps, cfg, np.zeros(ps.n))
    assert np.array_equal(v1, v2) and np.array_equal(l1, l2)
    assert r1.residual_trace == r2.residual_trace


def test_concurrent_threads_independent_handles():
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _rigid(256, 1024)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=100)
    ref = solve_packed(ps, cfg, np.zeros(ps.n))[0]
    out = [None] * 4

    def work(k):
        out[k] = solve_packed(ps, cfg, np.zeros(ps.n))[0]

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for o in out:
        assert np.array_equal(o, ref)


@pytest.mark.parametrize("mode", ["auto", "streaming"])
def test_config1_full_size_matches_oracle_prefix(mode):
    """configs[1] at full size (122,880 DOF, 16,384 contacts): the first 40
    iterations bit-match the CPU oracle (plain V-FPI, no OpenBLAS-ordered
    decision involved), on both iteration kernels."""
    from oracle import vfpi_oracle as O
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _rigid(4096, 16384, seed=2201)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=40)
    h = _lib.handle()
    h.set_kernel(mode)
    try:
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        layout = h.last_layout()
    finally:
        h.set_kernel("auto")
    assert layout["resident"] == (mode == "auto")  # configs[1] fits on chip: the resident kernel is the default
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    vo, lo, ro = O.solve(s, O.Config(residual_tol=1e-8, max_iters=40), np.zeros(ps.n))
    assert rep.iterations == ro.iterations == 40
    assert np.array_equal(v, vo)
    assert np.array_equal(lam, lo)
    assert np.allclose(rep.residual_trace, ro.residual_trace, rtol=1e-12)


def test_config1_full_run_properties():
    """1000 iterations at configs[1]: never converges at k_v=1e5,
    finite, deterministic, impulses inside the friction cone, and bit-equal
    to the CPU oracle over the whole solve."""
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _rigid(4096, 16384, seed=2201)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
    v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
    assert rep.iterations == 1000 and not rep.converged
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(lam))
    assert np.all(lam[:, 0] >= 0.0)
    tn = np.sqrt(lam[:, 1] ** 2 + lam[:, 2] ** 2)
    assert np.all(tn <= ps.mu * lam[:, 0] * (1 + 1e-12) + 1e-300)
    v2, lam2, rep2 = solve_packed(ps, cfg, np.zeros(ps.n))
    assert np.array_equal(v, v2)
    # and the whole 1000-iteration solve equals the CPU oracle bit for bit
    from oracle import vfpi_oracle as O

    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    vo, lo, ro = O.solve(s, O.Config(residual_tol=1e-8, max_iters=1000), np.zeros(ps.n))
    assert ro.iterations == 1000
    assert np.array_equal(v, vo) and np.array_equal(lam, lo)
