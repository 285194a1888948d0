"""One configs[1] solve (for profiler captures)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
cfg = SolverConfig(residual_tol=1e-8, max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 1000)
v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
print("iterations", rep.iterations, "loop_ms", rep.timings["loop_s"] * 1e3)
