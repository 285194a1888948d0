"""configs[1]: resident kernel free-row warp count (tuning key 7) and contact warps (key 0)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
h = _lib.handle(0)
cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
ref = None
for fw in [0, 2, 3, 4, 6, 8, 10, 0]:
    h.L.vfpi_set_tuning(h.h, 7, fw)
    best = 1e9
    for _ in range(4):
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        best = min(best, rep.timings["loop_s"] * 1e3)
    same = ref is None or (np.array_equal(v, ref[0]) and np.array_equal(lam, ref[1]))
    ref = ref or (v, lam)
    print(f"free warps {fw:2d}: loop {best:.3f} ms  same {same}", flush=True)
