"""configs[0] measurement: one FEM cube (10^3 nodes, E 1e5, nu 0.3, dropped
0.05 m) stepped 200 steps at dt 1e-3 through the device step pipeline
(FemBatch: b, node-plane detection, V-FPI solve, integration on the GPU),
and as a one-cube pile through the single-system kernel. Prints one JSON line
(the CPU reference path is timed by bench.py's reference arm).
usage: python scripts/bench_cfg0.py [--steps 200] [--chebyshev]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--chebyshev", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=a.chebyshev)
    runs = []
    for rep in range(2):  # the first run includes allocations and graph capture
        fb = FemBatch([FemCube()])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ci = its = 0
        loop_ms = setup_ms = 0.0
        per = []
        for _ in range(a.steps):
            st = fb.step(cfg)
            ci += st["contact_iterations"]
            its += st["iterations"]
            loop_ms += st["loop_ms"]
            setup_ms += st["setup_ms"]
            per.append((st["contacts"], st["iterations"]))
        torch.cuda.synchronize()
        runs.append((time.perf_counter() - t0, ci, its, loop_ms, setup_ms, per, fb.state()[0].copy()))
    wall, ci, its, loop_ms, setup_ms, per, x_dev = runs[-1]
    # the same cube as a one-cube CubePile through PileStepper: the single-system
    # (multi-CTA resident) kernel instead of the one-CTA scene kernel
    from paper_2201_09212_b200.pile import CubePile, PileStepper

    for rep in range(2):
        pst = PileStepper(CubePile(1, 1, 1, nodes=10, gap=0.0, jitter=0.0, gap_z=0.05, jitter_z=0.0, dt=1e-3,
                                   mu=0.5))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sci = 0
        sloop = 0.0
        for _ in range(a.steps):
            r = pst.step(cfg)
            sci += r["n_c"] * r["iterations"]
            sloop += r["loop_ms"]
        torch.cuda.synchronize()
        swall = time.perf_counter() - t0
    single = {"wall_s": swall, "sim_steps_per_s": a.steps / swall, "contact_iter_per_s": sci / swall,
              "loop_ms": sloop, "final_state_max_abs_diff_vs_batch_path":
                  float(np.abs(pst.state()[0] - x_dev.reshape(-1, 3)).max())}
    # roofline of the solve loops against the algorithmic bytes:
    # B_iter = 12 nnz_num + 4 (n+1) + 32 n (+8 n Chebyshev) + 128 n_c per iteration
    cube0 = FemCube()
    nnz_num = int(np.count_nonzero(cube0.A.data))
    n0 = cube0.n
    bytes_tot = sum((12 * nnz_num + 4 * (n0 + 1) + 32 * n0 + (8 * n0 if a.chebyshev else 0) + 128 * c) * i
                    for c, i in per)
    peak = 6650.0
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    gbs = bytes_tot / (loop_ms * 1e-3) / 1e9 if loop_ms > 0 else 0.0
    out = {"workload": "configs[0] single FEM cube 10^3 nodes, 200 steps", "steps": a.steps,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "note": "one-CTA scene kernel on a 1 MB system: latency-bound, cache-resident"},
           "chebyshev": a.chebyshev, "tol": 1e-8, "max_iters": 500, "operator": "strict", "mu": 0.5, "dt": 1e-3,
           "E": 1e5, "nu": 0.3, "drop_m": 0.05, "wall_s": wall,
           "sim_steps_per_s": a.steps / wall, "contact_iter_per_s": ci / wall, "contact_iterations": ci,
           "iterations": its, "loop_ms": loop_ms, "setup_ms": setup_ms,
           "contact_steps": sum(1 for c, _ in per if c > 0), "max_contacts": max(c for c, _ in per),
           "mean_iters_contact_steps": float(np.mean([i for c, i in per if c > 0])) if any(c for c, _ in per) else 0,
           "path": "FemBatch (scene kernel, one CTA)", "single_system_path": single}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
