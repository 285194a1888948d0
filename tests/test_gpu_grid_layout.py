"""The single-system node-block grid layout (csrc/vfpi_nodes.cu,
node_grid_build) at small sizes, forced onto the streaming path: packed block
values (pack modes 0 / 1 / 2 / 3 = forced, tuning key 12) and the contact-weighted CTA
ranges (key 11) change how A streams and which CTA owns a node, never the
result -- every variant equals the CPU oracle bit for bit (plain strict V-FPI)."""

import numpy as np
import pytest

from oracle import pile_host as H
from oracle import vfpi_oracle as O

pytestmark = pytest.mark.gpu


def _pile_system(seed=5):
    from paper_2201_09212_b200.pile import CubePile

    # unrotated cubes: their 3x3 blocks store ~5.5 of 9 entries -> packed values
    pile = CubePile(nx_cubes=2, ny_cubes=2, layers=2, nodes=6, gap=0.0, jitter=0.00005, seed=seed, dt=5e-4)
    pc = H.contacts(pile)
    b_o = H.rhs(pile)
    return pile, pc, H.system(pile, pc, b_o)


def _oracle(ps, cfg_iters=120):
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, O.Config(residual_tol=1e-8, max_iters=cfg_iters), np.zeros(ps.n))


@pytest.mark.parametrize("pack", [0, 1, 2, 3])
@pytest.mark.parametrize("contact_cost", [0, 8, 64])
def test_grid_layout_variants_bitwise(pack, contact_cost):
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    _, pc, ps = _pile_system()
    assert pc.n_c > 0
    h = _lib.handle()
    try:
        h.set_kernel("streaming")
        h.L.vfpi_set_tuning(h.h, 12, pack)
        h.L.vfpi_set_tuning(h.h, 11, contact_cost)
        v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-8, max_iters=120), np.zeros(ps.n))
        assert h.last_layout()["node_kernel"]
        packed = bool(h.L.vfpi_set_tuning(h.h, 13, 0))
        if pack in (0, 3):  # off / forced (modes 1, 2 pack only where the slots fit tight)
            assert packed == (pack == 3)
    finally:
        h.set_kernel("auto")
        h.L.vfpi_set_tuning(h.h, 12, 2)
        h.L.vfpi_set_tuning(h.h, 11, 8)
    vo, lo, ro = _oracle(ps)
    assert rep.iterations == ro.iterations
    assert np.array_equal(v, vo), float(np.abs(v - vo).max())
    assert np.array_equal(lam, lo)
