"""configs[3] measurement: one V-FPI solve of the 64^3-node heightfield block
(786,432 DOF, ~24.6M stored nonzeros, ~4,096 S-contacts) on one GPU through
the single-system streaming kernel, against the algorithmic-byte roofline, and
a bounded CPU-oracle sample on the host. Prints one JSON line.
usage: python scripts/bench_cfg3.py [--nx 64] [--max-iters 500] [--cpu-iters 3] [--ncu]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import HeightfieldBlock  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402


def b_iter(n, nnz_num, n_c, cheb):
    return 12 * nnz_num + 4 * (n + 1) + 32 * n + (8 * n if cheb else 0) + 128 * n_c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--ncu", action="store_true", help="one short solve per variant (for a profiler capture)")
    a = ap.parse_args()
    t0 = time.perf_counter()
    blk = HeightfieldBlock(nx=a.nx)
    ps = blk.system()
    t_build = time.perf_counter() - t0
    nnz_num = int(np.count_nonzero(ps.data))
    peak = 6650.0
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    out = {"workload": f"configs[3] heightfield block {a.nx}^3 nodes", "n": ps.n, "n_c": ps.n_c,
           "tol": 1e-8, "max_iters": a.max_iters, "operator": "strict", "E": 1e6, "nu": 0.35, "mu": 0.4, "dt": 1e-3,
           "side_m": 0.1, "press": "bottom conformed 0.1 mm into the heightfield + 50 N on the top face",
           "nnz_stored": ps.nnz, "nnz_numeric": nnz_num, "build_s": t_build, "variants": []}
    h = _lib.handle(0)
    for cheb in (False, True):
        cfg = SolverConfig(residual_tol=1e-8, max_iters=20 if a.ncu else a.max_iters, chebyshev=cheb)
        solve_packed(ps, cfg, np.zeros(ps.n))  # warm-up (allocations, graph capture)
        best = None
        for _ in range(1 if a.ncu else 3):
            v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
            if best is None or rep.timings["loop_s"] < best[2].timings["loop_s"]:
                best = (v, lam, rep)
        rep = best[2]
        it = rep.iterations
        loop = rep.timings["loop_s"]
        setup = rep.timings["setup_s"]
        bi = b_iter(ps.n, nnz_num, ps.n_c, cheb)
        gbs = bi * it / loop / 1e9 if loop > 0 else 0.0
        out["variants"].append({
            "chebyshev": cheb, "iterations": it, "converged": rep.converged, "loop_ms": loop * 1e3,
            "setup_ms": setup * 1e3, "resident": h.last_layout()["resident"], "ctas": h.last_layout()["ctas"],
            "contact_iter_per_s": ps.n_c * it / (loop + setup), "bytes_per_iter": bi,
            "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak})
    if not a.ncu and a.cpu_iters > 0:
        from oracle import vfpi_oracle as O  # CPU baseline only
        s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64),
                     ps.col_j.astype(np.int64), ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
        t1 = time.perf_counter()
        O.solve(s, O.Config(residual_tol=0.0, max_iters=a.cpu_iters), np.zeros(ps.n))
        dt = time.perf_counter() - t1
        out["cpu_baseline"] = {"kind": "port", "cores": 1, "sample": f"oracle solve capped at {a.cpu_iters} "
                               "iterations (setup included)", "seconds": dt,
                               "contact_iter_per_s": ps.n_c * a.cpu_iters / dt}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
