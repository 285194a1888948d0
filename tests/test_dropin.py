"""dropin.install / uninstall patch every alias the reference imports by name
(CPU: fake condsim modules stand in for the reference package)."""

import sys
import types

from paper_2201_09212_b200 import augment, dropin, nodalize, solver


def _fake_condsim(monkeypatch):
    names = {"condsim": ["solve_vfpi"], "condsim.solver": ["solve_vfpi", "contact_solve_oneshot", "spmv"],
             "condsim.harness": ["solve_vfpi", "nodalize", "augment_dynamics"],
             "condsim.contacts": ["apply_jc", "apply_jc_t", "nodalize", "augment_dynamics"],
             "condsim.sparse": ["spmv", "row_norms_sq"]}
    mods = {}
    for mod, attrs in names.items():
        m = types.ModuleType(mod)
        for a in attrs:
            setattr(m, a, f"ref:{mod}.{a}")
        monkeypatch.setitem(sys.modules, mod, m)
        mods[mod] = m
    return mods


def test_install_patches_every_alias_and_uninstall_restores(monkeypatch):
    mods = _fake_condsim(monkeypatch)
    done = dropin.install()
    try:
        assert mods["condsim"].solve_vfpi is solver.solve_vfpi
        assert mods["condsim.harness"].solve_vfpi is solver.solve_vfpi
        assert mods["condsim.harness"].nodalize is nodalize.nodalize
        assert mods["condsim.harness"].augment_dynamics is augment.augment_dynamics
        assert mods["condsim.contacts"].augment_dynamics is augment.augment_dynamics
        assert "condsim.harness.nodalize" in done
    finally:
        dropin.uninstall()
    assert mods["condsim.harness"].nodalize == "ref:condsim.harness.nodalize"
    assert mods["condsim"].solve_vfpi == "ref:condsim.solve_vfpi"
