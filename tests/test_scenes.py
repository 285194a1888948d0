"""The configs[1] generator reproduces the reference's nodalize/augment output."""

import numpy as np

from oracle.fem_host import fem_system

from golden_cases import load
from paper_2201_09212_b200.scenes import rigid_contact_system


def test_rigid_system_bit_identical_to_reference_pipeline():
    d = load("rigid_pile_256")
    ps = rigid_contact_system(n_bodies=256, n_contacts=1024, seed=2201)
    assert ps.n == int(d["n"])
    for k in ("indptr", "indices", "data", "b", "col_i", "col_j", "frames", "mu", "phi"):
        got = getattr(ps, k)
        ref = d[k]
        assert got.shape == ref.shape, k
        assert np.array_equal(got, ref), k
        assert np.array_equal(np.signbit(got), np.signbit(ref)) if got.dtype.kind == "f" else True, k


def test_rigid_system_structure_at_config1_scale():
    ps = rigid_contact_system()  # 4096 bodies, 16384 contacts (BASELINE configs[1])
    assert ps.n == 6 * 4096 + 3 * 2 * 16384 == 122880
    assert ps.n_c == 16384
    assert np.all(ps.col_j == ps.col_i + 3)
    assert int(np.count_nonzero(ps.data)) == 786420  # SURVEY §8 sizing table
    assert ps.nnz == 1376244


def test_fem_cube_system_matches_reference_contact_pipeline():
    """FemCube's A, b and node-plane contacts equal what the reference's
    detect_contacts / nodalize / augment_dynamics built for the same state
    (golden fem*_s*: the FEM assembly itself has no reference and is the
    repo's own; the contact pipeline and the solve are pinned)."""
    import json

    from golden_cases import names

    from paper_2201_09212_b200.scenes import FemCube

    cases = [c for c in names() if c.startswith("fem")]
    assert len(cases) >= 3
    for c in cases:
        d = load(c)
        cube = FemCube(**json.loads(str(d["fem_kw"])))
        cube.x = d["fem_x"].copy()
        cube.v = d["fem_v"].copy()
        ps = fem_system(cube)
        for k in ("indptr", "indices", "data", "b", "col_i", "col_j", "frames", "mu", "phi"):
            assert np.array_equal(getattr(ps, k), d[k]), (c, k)
