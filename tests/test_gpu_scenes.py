"""Scene batches on the GPU: every scene of a heterogeneous batch matches the
reference's own result for that scene (solve_vfpi semantics per scene)."""

import numpy as np
import pytest

from golden_cases import load, names
from gpu_util import config, packed, relerr

pytestmark = pytest.mark.gpu


def _batch_by_cfg():
    groups = {}
    for nm in names():
        d = load(nm)
        if d["n"] > 5000 or d.get("w_cached") is not None:
            continue
        key = tuple(sorted(d["cfg"].items()))
        groups.setdefault(key, []).append(d)
    return groups


def test_scene_batches_match_reference_per_scene():
    from paper_2201_09212_b200.batch import solve_scenes
    from paper_2201_09212_b200.errors import DivergenceError

    checked = 0
    for key, ds in _batch_by_cfg().items():
        res, rep = solve_scenes([packed(d) for d in ds], config(ds[0]), warms=[d["warm"] for d in ds])
        for d, r in zip(ds, res):
            if d["out_diverged"]:
                assert isinstance(r, DivergenceError), d["name"]
                assert len(r.residual_trace) == int(d["out_iterations"])
                continue
            v, lam, srep = r
            assert srep.iterations == int(d["out_iterations"]), d["name"]
            assert srep.converged == bool(d["out_converged"]), d["name"]
            assert relerr(v, d["out_v"]) <= 1e-9, d["name"]
            if lam.size:
                assert relerr(lam, d["out_lam"]) <= 1e-9, d["name"]
            checked += 1
    assert checked >= 20


def test_rigid_scene_batch_equals_single_solves():
    from paper_2201_09212_b200.batch import solve_scenes
    from paper_2201_09212_b200.scenes import rigid_contact_system
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    scenes = [rigid_contact_system(n_bodies=16 + 8 * k, n_contacts=48 + 16 * k, seed=100 + k) for k in range(24)]
    cfg = SolverConfig(residual_tol=1e-9, max_iters=150)
    res, rep = solve_scenes(scenes, cfg)
    for s, r in zip(scenes, res):
        v1, l1, r1 = solve_packed(s, cfg, np.zeros(s.n))
        v, lam, rr = r
        assert rr.iterations == r1.iterations
        assert np.array_equal(v, v1) and np.array_equal(lam, l1)  # plain iteration: bit-identical
