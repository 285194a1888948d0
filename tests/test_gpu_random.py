"""Randomized parity of the V-FPI solve (-m gpu): seeded rigid-contact systems
of random size under random SolverConfigs (operator, step strategy,
Chebyshev, omega, under-relaxation, tolerance), both single-system kernels,
against the CPU oracle (itself pinned to the reference's golden vectors).
Bar: identical iteration counts and outcome; v and lam within 1e-9
relative (north_star); plain frobenius solves bit for bit.

Barzilai-Borwein steps take their scalar from three dot products that the
reference evaluates with OpenBLAS ddot; the GPU's fixed-order sums differ
in the last bit, and BB amplifies that chaotically (measured: 1e-16 after 10
iterations, 1e-13 after 80, 1e-10 after 140, `scripts/debug_bb.py`), so BB
cases run at most 40 iterations here."""

import numpy as np
import pytest

from oracle import vfpi_oracle as O
from paper_2201_09212_b200 import _lib
from paper_2201_09212_b200.scenes import rigid_contact_system
from paper_2201_09212_b200.solver import SolverConfig, solve_packed
from paper_2201_09212_b200.errors import DivergenceError


def _rel(a, b):
    a, b = np.asarray(a, float).ravel(), np.asarray(b, float).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("mode", ["resident", "streaming"])
def test_random_config_parity(seed, mode):
    g = np.random.default_rng(9000 + seed)
    nb = int(g.integers(8, 160))
    nc = int(g.integers(4, 3 * nb))
    ps = rigid_contact_system(nb, nc, seed=int(g.integers(1 << 30)), k_v=float(g.choice([1e2, 1e3, 1e5])))
    op = str(g.choice(["strict", "proximal", "strict-anisotropic"]))
    strategy = str(g.choice(["frobenius", "frobenius", "bb1", "bb2", "bb-alternating", "fixed-alpha"]))
    max_iters = int(g.integers(1, 200))
    if strategy.startswith("bb"):
        max_iters = 1 + max_iters % 40
    kw = dict(operator=op, step_strategy=strategy, residual_tol=float(g.choice([1e-6, 1e-8, 1e-10])),
              max_iters=max_iters, chebyshev=bool(g.random() < 0.4),
              cheby_start=int(g.integers(2, 15)), under_relax=float(g.choice([0.9, 0.7, 1.0])),
              omega=float(g.choice([0.0, 0.0, 1e-3])))
    if strategy == "fixed-alpha":
        kw["fixed_alpha"] = None if g.random() < 0.5 else float(g.uniform(1e-6, 1e-4))
    if op == "strict-anisotropic":
        ps.mu2[:] = g.uniform(0.1, 0.9, ps.n_c)
    warm = g.standard_normal(ps.n) * 0.01
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    try:
        with np.errstate(over="ignore", invalid="ignore"):
            vo, lo, ro = O.solve(s, O.Config(**kw), warm)
        odiv = None
    except O.OracleDivergence as e:
        odiv = e
    h = _lib.handle(0)
    h.set_kernel(mode)
    try:
        try:
            v, lam, rep = solve_packed(ps, SolverConfig(**kw), warm)
            gdiv = None
        except DivergenceError as e:
            gdiv = e
    finally:
        h.set_kernel("auto")
    assert (odiv is None) == (gdiv is None), (kw, odiv, gdiv)
    if odiv is not None:
        assert len(gdiv.residual_trace) == len(odiv.residual_trace)
        return
    assert rep.iterations == ro.iterations and rep.converged == ro.converged, kw
    if strategy == "frobenius" and not kw["chebyshev"]:
        assert np.array_equal(v, vo) and np.array_equal(lam, lo), kw
    else:
        assert _rel(v, vo) <= 1e-9 and _rel(lam, lo) <= 1e-9, kw


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_random_scene_batch_parity(seed):
    """A batch of random independent systems (different sizes and contact
    counts) in one scene-batch launch, random plain/Chebyshev configs: every
    scene equals its own oracle solve (iterations; bits for plain)."""
    from paper_2201_09212_b200.batch import solve_scenes

    g = np.random.default_rng(7000 + seed)
    scenes = [rigid_contact_system(int(g.integers(4, 40)), int(g.integers(1, 60)), seed=int(g.integers(1 << 30)),
                                   k_v=float(g.choice([1e2, 1e5]))) for _ in range(int(g.integers(2, 24)))]
    op = str(g.choice(["strict", "proximal", "strict-anisotropic"]))
    kw = dict(operator=op, residual_tol=1e-8, max_iters=int(g.integers(5, 150)),
              chebyshev=bool(seed % 2), cheby_start=int(g.integers(2, 10)))
    res, _ = solve_scenes(scenes, SolverConfig(**kw))
    for ps, r in zip(scenes, res):
        s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                     ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
        vo, lo, ro = O.solve(s, O.Config(**kw), np.zeros(ps.n))
        v, lam, rep = r
        assert rep.iterations == ro.iterations, kw
        if not kw["chebyshev"]:
            assert np.array_equal(v, vo) and np.array_equal(lam, lo), kw
        else:
            assert _rel(v, vo) <= 1e-9 and _rel(lam, lo) <= 1e-9, kw


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_random_wide_columns_per_op(seed):
    """Random symmetric matrices with columns of up to several hundred entries
    (numpy's pairwise blocking in row_norms_sq: 8 accumulators, 128-entry
    blocks) and random contacts: spmv, row norms, diagonal, Frobenius W (both
    tie rules), gamma, J_c / J_c^T, one-shots, inverse_contact -- bit for bit."""
    import scipy.sparse as sp

    from paper_2201_09212_b200 import contacts as GC
    from paper_2201_09212_b200 import solver as GS
    from paper_2201_09212_b200 import sparse as GP
    from paper_2201_09212_b200.system import SparseSymmetric, make_packed

    g = np.random.default_rng(3100 + seed)
    n = 3 * int(g.integers(40, 200))
    dens = float(g.uniform(0.05, 0.9))
    m = sp.random(n, n, density=dens, random_state=g, format="csc")
    m = (m + m.T + sp.identity(n) * n).tocsc()
    m.sort_indices()
    a = SparseSymmetric(n, m.indptr, m.indices, m.data)
    nodes = g.permutation(n // 3)
    n_c = int(g.integers(1, n // 6))
    ci = 3 * nodes[:n_c]
    cj = np.where(g.random(n_c) < 0.5, 3 * nodes[n_c:2 * n_c], -1)
    frames = np.stack([O.contact_frame(v) for v in g.standard_normal((n_c, 3))])
    mu, mu2 = g.uniform(0.1, 0.9, n_c), g.uniform(0.1, 0.9, n_c)
    phi = g.uniform(-1, 0, n_c)
    ps = make_packed(n, m.indptr, m.indices, m.data, g.standard_normal(n), ci, cj, frames.ravel(), mu, mu2, phi)
    s = O.System(n, m.indptr, m.indices, m.data, ps.b, ci.astype(np.int64), cj.astype(np.int64), frames, mu, mu2,
                 phi)
    x = g.standard_normal(n)
    assert np.array_equal(GP.spmv(a, x), O.spmv(s, x))
    assert np.array_equal(GP.row_norms_sq(a), O.row_norms_sq(s))
    assert np.array_equal(GP.diagonal(a), O.diagonal(s))
    for tie in (False, True):
        assert np.array_equal(GS.step_matrix_frobenius(a, ps, tie).w, O.step_matrix_frobenius(s, tie))
    w = O.step_matrix_frobenius(s, False)
    gam = GS.surrogate_gamma(GS.StepMatrix(w), ps, 1e-3)
    assert np.array_equal(gam.gamma, O.surrogate_gamma(s, w, 1e-3))
    assert np.array_equal(GC.apply_jc(ps, x), O.apply_jc(s, x))
    lam = g.standard_normal((n_c, 3))
    assert np.array_equal(GC.apply_jc_t(ps, lam), O.apply_jc_t(s, lam))
    eta = g.standard_normal((n_c, 3)) * 3
    for op in ("strict", "proximal", "strict-anisotropic"):
        got = GS.contact_solve_oneshot(gam, eta, phi, mu, op, mu2)
        assert np.array_equal(got, O.oneshot(gam.gamma, eta, phi, mu, mu2, op)), op
    assert np.array_equal(GS.inverse_contact(ps, x, 1e-3), O.inverse_contact(s, x, 1e-3, "proximal"))
