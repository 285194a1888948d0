"""Debug: growth of GPU-vs-oracle differences with iteration count for BB steps."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import vfpi_oracle as O
from paper_2201_09212_b200.scenes import rigid_contact_system
from paper_2201_09212_b200.solver import SolverConfig, solve_packed
g = np.random.default_rng(9002)
nb = int(g.integers(8, 160)); nc = int(g.integers(4, 3 * nb))
ps = rigid_contact_system(nb, nc, seed=int(g.integers(1 << 30)), k_v=float(g.choice([1e2, 1e3, 1e5])))
s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
             ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
warm = np.zeros(ps.n)
for strat in ("bb1", "bb2"):
    for it in (2, 3, 5, 10, 20, 40, 80, 140):
        kw = dict(operator="proximal", step_strategy=strat, residual_tol=1e-12, max_iters=it)
        vo, lo, ro = O.solve(s, O.Config(**kw), warm)
        v, lam, rep = solve_packed(ps, SolverConfig(**kw), warm)
        print(strat, it, "rel", np.linalg.norm(v - vo) / np.linalg.norm(vo), "bitwise", np.array_equal(v, vo))
