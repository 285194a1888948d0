"""configs[3] device step pipeline (heightfield.HeightfieldStepper) against
the host restatement (oracle/fem_host: heightfield_rhs / heightfield_contacts
/ fem_advance, solved by the oracle): device detection equal bit for bit,
iteration counts equal and states bit-equal every step (plain V-FPI)."""

import numpy as np
import pytest

from oracle import fem_host as F
from oracle import vfpi_oracle as O

pytestmark = pytest.mark.gpu


def _oracle(ps, cfg, warm):
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, O.Config(residual_tol=cfg.residual_tol, max_iters=cfg.max_iters, chebyshev=cfg.chebyshev),
                   warm)


def test_heightfield_contacts_device_equal_host():
    from paper_2201_09212_b200.heightfield import HeightfieldStepper
    from paper_2201_09212_b200.scenes import HeightfieldBlock

    blk = HeightfieldBlock(nx=12)
    st = HeightfieldStepper(blk)
    d = st.contacts_device()
    nodes, phi, depth, frames = F.heightfield_contacts(blk)
    assert nodes.size > 10
    assert np.array_equal(d["col_i"], 3 * nodes) and (d["col_j"] == -1).all()
    assert np.array_equal(d["phi"], phi) and np.array_equal(np.signbit(d["phi"]), np.signbit(phi))
    assert np.array_equal(d["frames"], frames.reshape(-1))
    assert (d["mu"] == blk.mu).all()


@pytest.mark.parametrize("nx", [6, 10])
def test_heightfield_stepper_matches_host_pipeline(nx):
    from paper_2201_09212_b200.heightfield import HeightfieldStepper
    from paper_2201_09212_b200.scenes import HeightfieldBlock
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(residual_tol=1e-8, max_iters=300)
    host = HeightfieldBlock(nx=nx)
    st = HeightfieldStepper(HeightfieldBlock(nx=nx))
    prev = None
    for step in range(8):
        ps = F.heightfield_system(host)
        vo, lo, ro = _oracle(ps, cfg, np.zeros(ps.n) if prev is None else prev)
        r = st.step(cfg)
        assert r["n_c"] == ps.n_c and r["n_c"] > 0, step
        assert r["iterations"] == ro.iterations and r["converged"] == ro.converged, step
        assert np.array_equal(st.last["lam"].cpu().numpy(), lo.ravel()), step
        F.fem_advance(host, vo)
        prev = vo
        xg, vg = st.state()
        assert np.array_equal(xg, host.x) and np.array_equal(vg, host.v), step


def test_heightfield_rhs_device_equal_host():
    import ctypes as C

    import torch

    from paper_2201_09212_b200.heightfield import HeightfieldStepper
    from paper_2201_09212_b200.scenes import HeightfieldBlock

    blk = HeightfieldBlock(nx=9)
    blk.v = np.random.default_rng(3).standard_normal(blk.v.shape) * 1e-2
    st = HeightfieldStepper(blk)
    h = st.h
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    rc = h.L.vfpi_fem_rhs_sell_device(h.h, blk.n, P(st.k_off), P(st.k_val), P(st.k_col), P(st.x), P(st.X), P(st.v),
                                      P(st.m), P(st.g), blk.dt, P(st.b), None)
    assert rc == 0
    rc = h.L.vfpi_add_device(h.h, blk.n, P(st.f_ext), P(st.b), None)
    assert rc == 0
    torch.cuda.synchronize()
    b = st.b.cpu().numpy()
    assert np.array_equal(b, F.heightfield_rhs(blk))
