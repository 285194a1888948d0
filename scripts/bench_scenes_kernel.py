"""Lean timing of the scene-batch kernel on a configs[2]-shaped batch (tuning aid).

Builds D distinct FEM cubes pressed 0.5 mm into the plane (so every scene has
its bottom-layer contacts), replicates them to S scenes (each scene keeps its
own explicit A in the batch), and times repeated vfpi_solve_scenes calls.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_09212_b200.batch import solve_scenes  # noqa: E402
from paper_2201_09212_b200.scenes import FemCube  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scenes", type=int, default=1024)
ap.add_argument("--distinct", type=int, default=16)
ap.add_argument("--nx", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
g = np.random.default_rng(7)
base = []
for k in range(args.distinct):
    c = FemCube(nx=args.nx, E=float(g.uniform(5e4, 2e5)), drop=0.0, yaw=float(g.uniform(0, 2 * np.pi)))
    c.x = c.X.copy()
    c.x[:, 2] -= 5e-4
    c.v[:, 2] = -0.3
    base.append(c.system())
scenes = [base[k % args.distinct] for k in range(args.scenes)]
cfg = SolverConfig(residual_tol=1e-8, max_iters=500)
nnz_num = [int(np.count_nonzero(s.data)) for s in scenes]
best = None
for r in range(args.reps + 1):
    t0 = time.perf_counter()
    res, rep = solve_scenes(scenes, cfg)
    wall = time.perf_counter() - t0
    if r and (best is None or rep.loop_ms < best[0]):
        best = (rep.loop_ms, rep.setup_ms, wall, res)
loop_ms, setup_ms, wall, res = best
its = [r[2].iterations for r in res]
ci = sum(s.n_c * r[2].iterations for s, r in zip(scenes, res))
bytes_it = sum((12 * nz + 4 * (s.n + 1) + 32 * s.n + 128 * s.n_c) * it for s, nz, it in zip(scenes, nnz_num, its))
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
print(json.dumps({"scenes": args.scenes, "n": scenes[0].n, "n_c": scenes[0].n_c, "mean_iters": float(np.mean(its)),
                  "loop_ms": loop_ms, "setup_ms": setup_ms, "wall_ms": wall * 1e3,
                  "contact_iter_per_s_loop": ci / (loop_ms * 1e-3),
                  "achieved_GBps_loop": bytes_it / (loop_ms * 1e-3) / 1e9, "hbm_peak": peak,
                  "frac": bytes_it / (loop_ms * 1e-3) / 1e9 / peak}))
