"""Per-step metrics rows and the reference's CSV wire format (SURVEY §8(f)
item 4): ``MetricsRow`` mirrors ``condsim.harness.MetricsRow``
(``harness.py:211-223``), ``report_csv`` / ``parse_csv`` write and read the
same bytes as ``harness.report_csv`` / ``parse_csv`` (``harness.py:651-697``:
header ``step,dyn_ms,solve_ms,iters,residual,max_pen_m,contacts,ke_J``,
integers as integers, floats with 17 significant digits, booleans as 0/1),
so GPU runs feed the reference's CSV consumers unchanged
(``tests/test_metrics.py`` against a CSV written by the reference).

``kinetic_energy`` is ``0.5 vᵀ M v`` (``dynamics.py:258-265``) for a lumped
(diagonal) mass, evaluated on the device state."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CSV_HEADER = "step,dyn_ms,solve_ms,iters,residual,max_pen_m,contacts,ke_J"


class CsvFormatError(ValueError):
    """Unexpected CSV header (the reference raises ScenarioValidationError)."""


@dataclass
class MetricsRow:
    step: int
    dyn_ms: float
    solve_ms: float
    iters: int
    residual: float
    max_pen_m: float
    contacts: int
    ke_J: float
    diverged: bool = False
    # not part of the CSV contract, kept for in-process checks
    converged: bool = False
    consistency: float = float("nan")


def _fmt(x) -> str:
    if isinstance(x, (bool, np.bool_)):
        return "1" if x else "0"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return format(float(x), ".17g")


def report_csv(rows, path: str) -> None:
    lines = [CSV_HEADER]
    for r in rows:
        lines.append(",".join(_fmt(x) for x in (r.step, r.dyn_ms, r.solve_ms, r.iters, r.residual, r.max_pen_m,
                                                r.contacts, r.ke_J)))
    with open(path, "w", newline="") as fh:
        fh.write("\n".join(lines) + "\n")


def parse_csv(path: str):
    rows = []
    with open(path) as fh:
        header = fh.readline().strip()
        if header != CSV_HEADER:
            raise CsvFormatError(f"unexpected CSV header {header!r}")
        for line in fh:
            p = line.strip().split(",")
            rows.append(MetricsRow(step=int(p[0]), dyn_ms=float(p[1]), solve_ms=float(p[2]), iters=int(p[3]),
                                   residual=float(p[4]), max_pen_m=float(p[5]), contacts=int(p[6]),
                                   ke_J=float(p[7])))
    return rows


def kinetic_energy(m, v) -> float:
    """0.5 sum m_i v_i^2 for a lumped mass (device tensors or arrays)."""
    try:
        import torch

        if isinstance(v, torch.Tensor):
            return float(0.5 * torch.dot(m * v, v))
    except ImportError:  # pragma: no cover
        pass
    v = np.asarray(v, float)
    return float(0.5 * np.dot(np.asarray(m, float) * v, v))
