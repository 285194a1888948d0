"""Sweep of the partition cost model on configs[1] (tuning aid)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
h = _lib.handle(0)
for a in sys.argv[1:]:  # key=value tuning knobs applied to every run
    if "=" in a:
        k_, v_ = a.split("=")
        h.L.vfpi_set_tuning(h.h, int(k_), int(v_))
cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
grid = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:] if "=" not in a] or [(24, 40, 256), (24, 40, 512), (24, 40, 1024)]
for g in grid:
    ec, rc, cc = g[:3]
    anchor = g[3] if len(g) > 3 else 0
    h.L.vfpi_set_tuning(h.h, 1, anchor)
    h.L.vfpi_set_tuning(h.h, 3, ec)
    h.L.vfpi_set_tuning(h.h, 4, rc)
    h.L.vfpi_set_tuning(h.h, 5, cc)
    best = 1e9
    for _ in range(3):
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        best = min(best, rep.timings["loop_s"] * 1e3)
    print(f"entry {ec:3d} row {rc:3d} contact {cc:5d} anchor {anchor}: {best:.3f} ms  resident={h.last_layout()['resident']}")
