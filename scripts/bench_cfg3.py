"""configs[3] to spec: the 64^3-node heightfield block (786,432 DOF) stepped
100 times on one GPU, every piece of the step on the device
(``heightfield.HeightfieldStepper``: right-hand side, heightfield detection,
V-FPI solve warm-started from the previous step, CG fallback, integration).
Prints one JSON line (sim steps/s, contact-iterations/s, per-launch roofline
of the single-system iteration kernel) and writes the per-step rows in the
reference's CSV format (``metrics.report_csv``).

usage: python scripts/bench_cfg3.py [--steps 100] [--max-iters 500] [--chebyshev] [--csv out.csv]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09212_b200.heightfield import HeightfieldStepper  # noqa: E402
from paper_2201_09212_b200.metrics import report_csv  # noqa: E402
from paper_2201_09212_b200.scenes import HeightfieldBlock  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--chebyshev", action="store_true")
    ap.add_argument("--csv", default=None)
    ap.add_argument("--tune", nargs="*", default=[], help="key=value tuning knobs of the handle (vfpi_set_tuning)")
    a = ap.parse_args()
    from paper_2201_09212_b200 import _lib

    for kv in a.tune:
        k, v = kv.split("=")
        _lib.handle().L.vfpi_set_tuning(_lib.handle().h, int(k), int(v))
    t0 = time.perf_counter()
    blk = HeightfieldBlock(nx=a.nx)
    t_build = time.perf_counter() - t0
    st = HeightfieldStepper(blk)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=a.max_iters, chebyshev=a.chebyshev)
    nnz = int(blk.A.nnz)  # A stores no zeros
    peak = 6650.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    rows, recs = [], []
    import torch

    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for k in range(a.steps):
        r = st.step(cfg)
        recs.append(r)
        rows.append(st.metrics_row(k, r))
    wall = time.perf_counter() - t1
    n = blk.n
    loop_ms = sum(r["loop_ms"] for r in recs)
    its = sum(r["vfpi_iterations"] for r in recs)
    ci = sum(r["n_c"] * r["vfpi_iterations"] for r in recs)
    bytes_total = sum((12 * nnz + 4 * (n + 1) + 32 * n + (8 * n if a.chebyshev else 0) + 128 * r["n_c"])
                      * r["vfpi_iterations"] for r in recs)
    out = {"workload": f"configs[3] heightfield block {a.nx}^3 nodes, {a.steps} steps on one GPU",
           "n": n, "nnz": nnz, "tol": 1e-8, "max_iters": a.max_iters, "chebyshev": a.chebyshev,
           "operator": "strict", "E": 1e6, "nu": 0.35, "mu": 0.4, "dt": 1e-3, "side_m": 0.1,
           "press": "bottom conformed 0.1 mm into the heightfield + 50 N on the top face",
           "build_s": t_build, "wall_s": wall, "sim_steps_per_s": a.steps / wall,
           "contact_iter_per_s": ci / wall, "mean_contacts": float(np.mean([r["n_c"] for r in recs])),
           "mean_iterations": its / a.steps, "converged_steps": sum(r["converged"] for r in recs),
           "diverged_steps": sum(r["diverged"] for r in recs),
           "loop_ms_total": loop_ms, "setup_ms_total": sum(r["setup_ms"] for r in recs),
           "kernel": {"achieved_gbs": bytes_total / (loop_ms * 1e-3) / 1e9, "peak_gbs": peak,
                      "frac": bytes_total / (loop_ms * 1e-3) / 1e9 / peak,
                      "note": "algorithmic bytes 12 nnz + 4(n+1) + 32 n (+8 n Chebyshev) + 128 n_c per iteration "
                              "over the summed iteration-kernel event time"},
           "final_ke_J": recs[-1]["ke_J"], "max_pen_m_last": recs[-1]["max_pen_m"]}
    if a.csv:
        report_csv(rows, a.csv)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
