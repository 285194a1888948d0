"""Reference CSV wire format (harness.py:651-697): byte-identical output on
rows whose CSV the reference itself wrote (tests/golden/metrics_ref.csv), and
a round trip. A GPU pile run emits rows in that format (-m gpu)."""

import os

import numpy as np
import pytest

from paper_2201_09212_b200.metrics import CSV_HEADER, CsvFormatError, MetricsRow, kinetic_energy, parse_csv, report_csv

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metrics_ref.csv")

ROWS = [MetricsRow(0, 0.123456789, 1.5, 12, 3.2e-9, 0.0, 0, 0.0),
        MetricsRow(1, 10.0, 0.1, 500, 1e-300, 1.4e-3, 60349, 1234.5678901234567, diverged=True),
        MetricsRow(2, 1.0 / 3.0, 2.0 ** -40, 7, 5e-324, 2.5e-17, 7, 1e22)]


def test_csv_bytes_match_reference(tmp_path):
    out = tmp_path / "m.csv"
    report_csv(ROWS, str(out))
    assert out.read_bytes() == open(GOLD, "rb").read()


def test_csv_round_trip_and_header(tmp_path):
    rows = parse_csv(GOLD)
    assert [r.step for r in rows] == [0, 1, 2] and rows[1].contacts == 60349
    for a, b in zip(rows, ROWS):
        for f in ("dyn_ms", "solve_ms", "residual", "max_pen_m", "ke_J"):
            assert getattr(a, f) == getattr(b, f)
    bad = tmp_path / "bad.csv"
    bad.write_text("step,dyn\n")
    with pytest.raises(CsvFormatError):
        parse_csv(str(bad))
    assert open(GOLD).readline().strip() == CSV_HEADER


def test_kinetic_energy_lumped():
    m = np.array([1.0, 1.0, 1.0, 2.0, 2.0, 2.0])
    v = np.array([1.0, 0.0, 0.0, 0.0, 3.0, 0.0])
    assert kinetic_energy(m, v) == 0.5 * (1.0 + 18.0)


@pytest.mark.gpu
def test_gpu_pile_run_writes_reference_csv(tmp_path):
    from paper_2201_09212_b200.pile import CubePile, PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    st = PileStepper(CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, gap=0.0, jitter=0.00005, seed=5))
    rows = [st.metrics_row(k, st.step(SolverConfig(residual_tol=1e-8, max_iters=100))) for k in range(3)]
    out = tmp_path / "run.csv"
    report_csv(rows, str(out))
    back = parse_csv(str(out))
    assert [r.contacts for r in back] == [r.contacts for r in rows] and back[0].contacts > 0
    assert all(r.iters > 0 and r.ke_J > 0 for r in back)
