import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2201_09212_b200.fembatch import FemBatch
from paper_2201_09212_b200.scenes import FemCube
from paper_2201_09212_b200.solver import SolverConfig
g = np.random.default_rng(1)
cubes = [FemCube(E=float(g.uniform(5e4, 2e5)), drop=0.0005, yaw=float(g.uniform(0, 6.28))) for _ in range(256)]
for cheb in (False, True, False):
    fb = FemBatch(cubes)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=cheb)
    rows = []
    for k in range(12):
        t0 = time.perf_counter(); st = fb.step(cfg); w = time.perf_counter() - t0
        rows.append((round(st["setup_ms"], 3), round(st["loop_ms"], 3), round(st["step_ms"], 3), round(w * 1e3, 3), st["contacts"]))
    print("cheb", cheb, rows[-6:])
    fb.close()
