"""configs[1] solves through the device path (ncu / tuning driver): 4096 rigid
bodies, 16,384 D-contacts, tol 1e-8, 1000 iterations; prints the kernel time.
usage: python scripts/cfg1_solve.py [solves=3] [key=value tuning knobs ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and "=" not in sys.argv[1] else 3
ps = rigid_contact_system(4096, 16384, 2201)
h = _lib.handle(0)
for a in sys.argv[1:]:
    if "=" in a:
        k, v = a.split("=")
        h.L.vfpi_set_tuning(h.h, int(k), int(v))
cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
loops = []
for _ in range(n):
    v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
    loops.append(rep.timings["loop_s"] * 1e3)
print("iterations", rep.iterations, "loop_ms", ["%.3f" % t for t in loops], "layout", h.last_layout())
