"""Swap the reference's V-FPI entry points for the CUDA ones in a running
``condsim`` process (the binding a condsim maintainer would add).

    import condsim
    from paper_2201_09212_b200 import dropin
    dropin.install()          # condsim.solve_vfpi & friends now run on the GPU

``solve_vfpi`` is imported *by name* in ``condsim.harness`` (harness.py:47)
and re-exported from ``condsim/__init__.py:18``, so every alias is patched;
``nodalize`` and ``augment_dynamics`` (imported by name in the harness,
harness.py:22-31) are patched too, so a harness step's contact restructuring
runs on the GPU as well.
"""

from __future__ import annotations

import sys

from . import augment as _augment
from . import contacts as _contacts
from . import nodalize as _nodalize
from . import solver as _solver
from . import sparse as _sparse

_PATCH = {
    "condsim.solver": {
        "solve_vfpi": _solver.solve_vfpi,
        "contact_solve_oneshot": _solver.contact_solve_oneshot,
        "step_matrix_frobenius": _solver.step_matrix_frobenius,
        "surrogate_gamma": _solver.surrogate_gamma,
        "scc_residual": _solver.scc_residual,
        "inverse_contact": _solver.inverse_contact,
        "apply_jc": _contacts.apply_jc,
        "apply_jc_t": _contacts.apply_jc_t,
        "spmv": _sparse.spmv,
        "row_norms_sq": _sparse.row_norms_sq,
    },
    # harness.run's per-step restructuring (harness.py:545-546) and solve (:557)
    "condsim.harness": {"solve_vfpi": _solver.solve_vfpi, "nodalize": _nodalize.nodalize,
                        "augment_dynamics": _augment.augment_dynamics},
    "condsim": {"solve_vfpi": _solver.solve_vfpi},
    "condsim.contacts": {"apply_jc": _contacts.apply_jc, "apply_jc_t": _contacts.apply_jc_t,
                         "nodalize": _nodalize.nodalize, "augment_dynamics": _augment.augment_dynamics},
    "condsim.sparse": {"spmv": _sparse.spmv, "row_norms_sq": _sparse.row_norms_sq},
}

_saved: dict = {}


def install() -> list:
    """Patch every loaded condsim module; returns the patched names."""
    import condsim  # noqa: F401  (raises if the reference is not installed)
    import condsim.harness  # noqa: F401
    import condsim.solver  # noqa: F401

    done = []
    for mod_name, attrs in _PATCH.items():
        mod = sys.modules.get(mod_name)
        if mod is None:
            continue
        for attr, fn in attrs.items():
            if hasattr(mod, attr):
                _saved.setdefault((mod_name, attr), getattr(mod, attr))
                setattr(mod, attr, fn)
                done.append(f"{mod_name}.{attr}")
    return done


def uninstall() -> None:
    for (mod_name, attr), fn in _saved.items():
        mod = sys.modules.get(mod_name)
        if mod is not None:
            setattr(mod, attr, fn)
    _saved.clear()
