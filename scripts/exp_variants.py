"""Sensitivity experiments on configs[1] (tuning aid): loop time with and
without contacts, plain vs Chebyshev, resident vs streaming."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402
from paper_2201_09212_b200.system import make_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
nc = make_packed(ps.n, ps.indptr, ps.indices, ps.data, ps.b, [], [], [], [])
h = _lib.handle(0)


def t(sys_, cfg, mode="auto", reps=3):
    h.set_kernel(mode)
    best = 1e9
    for _ in range(reps):
        v, lam, rep = solve_packed(sys_, cfg, np.zeros(sys_.n))
        best = min(best, rep.timings["loop_s"] * 1e3)
    lay = h.last_layout()
    h.set_kernel("auto")
    return best, rep.iterations, lay["resident"]


cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
for anc in (0, 1):
    for ls in (0, 1):
        h.L.vfpi_set_tuning(h.h, 1, anc)
        h.L.vfpi_set_tuning(h.h, 2, ls)
        print(f"anchor={anc} lensort={ls}: contacts %.3f ms  no-contacts %.3f ms" % (
            t(ps, cfg)[0], t(nc, SolverConfig(residual_tol=0.0, max_iters=1000))[0]))
h.L.vfpi_set_tuning(h.h, 1, 0)
h.L.vfpi_set_tuning(h.h, 2, 1)
print("contacts, resident      %.3f ms (%d it, resident=%s)" % t(ps, cfg))
print("no contacts, resident   %.3f ms (%d it, resident=%s)" % t(nc, SolverConfig(residual_tol=0.0, max_iters=1000)))
print("contacts, streaming     %.3f ms (%d it, resident=%s)" % t(ps, cfg, "streaming"))
print("contacts, chebyshev     %.3f ms (%d it, resident=%s)" % t(ps, SolverConfig(residual_tol=0.0, max_iters=1000, chebyshev=True)))
cfg10 = SolverConfig(residual_tol=1e-8, max_iters=10)
print("contacts, 10 iters      %.3f ms (%d it, resident=%s)" % t(ps, cfg10))
