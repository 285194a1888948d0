"""configs[1]: resident-kernel grid barrier variants (tuning key 6), timing + bitwise agreement."""
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
for mode in [int(a) for a in sys.argv[1:]] or [0, 1, 2, 0]:
    assert h.L.vfpi_set_tuning(h.h, 6, mode) == 0
    best = 1e9
    for _ in range(5):
        v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
        best = min(best, rep.timings["loop_s"] * 1e3)
    same = ref is None or (np.array_equal(v, ref[0]) and np.array_equal(lam, ref[1]))
    if ref is None:
        ref = (v, lam)
    print(f"bar_mode {mode}: loop {best:.3f} ms  iterations {rep.iterations}  bitwise_same {same}", flush=True)
