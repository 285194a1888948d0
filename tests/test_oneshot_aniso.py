"""Strict-anisotropic one-shot with mu2 != mu (the ellipse bisection,
solver.py:103-141, np.hypot included): the oracle (CPU) and the device
(vfpi_contact_solve_oneshot, -m gpu) against the reference's own output
(tests/golden/oneshot_aniso.npz), bit for bit."""

import os

import numpy as np
import pytest

from oracle import vfpi_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oneshot_aniso.npz")


def test_oracle_aniso_oneshot_matches_reference():
    d = dict(np.load(GOLD))
    lam = O.oneshot(d["gamma"], d["eta"], d["phi"], d["mu"], d["mu2"], "strict-anisotropic")
    assert np.array_equal(lam, d["out_lam"])
    # the golden exercises the bisection: some outputs are strictly inside / on the ellipse
    assert (d["mu"] != d["mu2"]).mean() > 0.8


@pytest.mark.gpu
def test_device_aniso_oneshot_matches_reference():
    from paper_2201_09212_b200.solver import SurrogateDelassus, contact_solve_oneshot

    d = dict(np.load(GOLD))
    lam = contact_solve_oneshot(SurrogateDelassus(d["gamma"]), d["eta"], d["phi"], d["mu"], "strict-anisotropic",
                                d["mu2"])
    assert np.array_equal(lam, d["out_lam"])
