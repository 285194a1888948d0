"""Divergence fallback in the device step pipelines (harness.py:586-593): a
scene whose V-FPI solve diverges takes the flagged contact-free step
v_hat = cg(A, b, rtol=1e-10, maxiter=10 n), lam = 0, instead of integrating
the diverged iterate. Divergence is forced as the reference's own test does
(fixed_alpha = 1e3, test_solver_units.py:360-366). The CG result is
tolerance-equal to scipy's (both stop at ||r|| < 1e-10 ||b||)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pressed_cubes(nx=5, n=3):
    from paper_2201_09212_b200.scenes import FemCube

    cubes = []
    for k in range(n):
        c = FemCube(nx=nx, E=6e4 + 4e4 * k, drop=0.0, yaw=0.3 * k)
        c.x = c.X.copy()
        c.x[:, 2] -= 2e-4 * (k + 1)  # pressed below the plane: contacts from step 0
        c.v[:, 2] = -0.05
        cubes.append(c)
    return cubes


def test_fem_batch_diverged_scene_takes_contact_free_cg_step():
    from oracle import fem_host
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(residual_tol=1e-8, max_iters=200, step_strategy="fixed-alpha", fixed_alpha=1e3)
    gpu, cpu = _pressed_cubes(), _pressed_cubes()
    fb = FemBatch(gpu)
    st = fb.step(cfg)
    assert st["diverged_scenes"] == len(gpu)
    assert st["contacts"] > 0
    xg, vg = fb.state()
    for k, c in enumerate(cpu):
        rec = []
        fem_host.oracle_steps(c, 1, residual_tol=1e-8, max_iters=200, record=rec, step_strategy="fixed-alpha",
                              fixed_alpha=1e3)
        assert rec[0]["diverged"] and rec[0]["n_c"] > 0
        assert np.all(np.isfinite(xg[k])) and np.all(np.isfinite(vg[k]))
        dv = np.abs(vg[k] - c.v).max() / np.abs(c.v).max()
        assert dv < 1e-8, dv
        dx = np.abs(xg[k] - c.x).max()
        assert dx < 1e-12, dx
    fb.close()


def test_fem_batch_without_divergence_is_unchanged():
    """Converging solves never enter the fallback: the step stays bit-identical
    to the oracle pipeline."""
    from oracle import fem_host
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(residual_tol=1e-8, max_iters=300)
    gpu, cpu = _pressed_cubes(n=3), _pressed_cubes(n=3)
    fb = FemBatch(gpu)
    st = fb.step(cfg)
    assert st["diverged_scenes"] == 0
    xg, vg = fb.state()
    for k, c in enumerate(cpu):
        rec = []
        fem_host.oracle_steps(c, 1, residual_tol=1e-8, max_iters=300, record=rec)
        assert not rec[0]["diverged"]
        assert np.array_equal(xg[k], c.x) and np.array_equal(vg[k], c.v)
    fb.close()


def test_pile_stepper_diverged_step_takes_contact_free_cg_step():
    import scipy.sparse as sp

    from oracle import pile_host as H
    from paper_2201_09212_b200.pile import CubePile, PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    pile = CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, seed=3, gap=0.0, jitter=0.0, gap_z=-1e-4)
    x0, v0 = pile.x.copy(), pile.v.copy()
    b_o = H.rhs(pile)
    a_o = sp.csc_matrix((pile.a_data, pile.a_indices, pile.a_indptr), shape=(pile.n, pile.n))
    st = PileStepper(pile)
    r = st.step(SolverConfig(residual_tol=1e-8, max_iters=100, step_strategy="fixed-alpha", fixed_alpha=1e3))
    assert r["diverged"] and r["n_c"] > 0
    assert r["iterations"] == 0 and r["residual"] == 0.0 and not r["converged"]  # the harness row
    from scipy.sparse.linalg import cg

    vh, info = cg(a_o, b_o, rtol=1e-10, maxiter=10 * pile.n)
    assert info == 0
    xg, vg = st.state()
    x_ref = x0 + pile.dt * vh.reshape(-1, 3)
    v_ref = 2.0 * vh.reshape(-1, 3) - v0
    assert np.abs(vg - v_ref).max() <= 1e-8 * np.abs(v_ref).max()
    assert np.abs(xg - x_ref).max() <= 1e-12


def test_cg_device_matches_scipy_on_a_spd_system():
    import ctypes as C

    import scipy.sparse as sp
    import torch
    from scipy.sparse.linalg import cg

    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.scenes import FemCube

    c = FemCube(nx=8, E=1e5, yaw=0.4)
    a = c.A
    b = np.random.default_rng(5).standard_normal(c.n)
    h = _lib.handle()
    dev = torch.device("cuda", h.device)
    t = [torch.from_numpy(np.ascontiguousarray(z)).to(dev) for z in
         (a.indptr.astype(np.int32), a.indices.astype(np.int32), a.data, b)]
    x = torch.empty(c.n, dtype=torch.float64, device=dev)
    it = C.c_int32(0)
    rc = h.L.vfpi_cg_device(h.h, c.n, *(C.c_void_p(z.data_ptr()) for z in t), C.c_void_p(x.data_ptr()), 1e-10,
                            10 * c.n, C.byref(it), None)
    assert rc == 0, h.error()
    xr, info = cg(a, b, rtol=1e-10, maxiter=10 * c.n)
    xg = x.cpu().numpy()
    assert info == 0 and it.value > 0
    assert np.linalg.norm(xg - xr) <= 1e-8 * np.linalg.norm(xr)
    assert np.linalg.norm(a @ xg - b) <= 2e-10 * np.linalg.norm(b)
    # zero right-hand side: scipy returns b itself
    t[3].zero_()
    rc = h.L.vfpi_cg_device(h.h, c.n, *(C.c_void_p(z.data_ptr()) for z in t), C.c_void_p(x.data_ptr()), 1e-10,
                            10 * c.n, C.byref(it), None)
    assert rc == 0 and it.value == 0 and not torch.any(x != 0)
    _ = sp  # scipy.sparse imported for the matrix type
