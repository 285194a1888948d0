"""Sweep of the partition cost model on configs[1] (tuning aid)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
h = _lib.handle(0)
cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
grid = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [(24, 40, 256), (24, 40, 512), (24, 40, 1024)]
for ec, rc, cc in grid:
    h.L.vfpi_set_tuning(h.h, 3, ec)
    h.L.vfpi_set_tuning(h.h, 4, rc)
    h.L.vfpi_set_tuning(h.h, 5, cc)
    best = 1e9
    for _ in range(3):
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        best = min(best, rep.timings["loop_s"] * 1e3)
    print(f"entry {ec:3d} row {rc:3d} contact {cc:5d}: {best:.3f} ms  resident={h.last_layout()['resident']}")
