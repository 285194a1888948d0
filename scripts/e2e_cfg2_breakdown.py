"""configs[2] e2e breakdown (wall clock): FemBatch creation from pinned host
arrays (upload + K row SELL + node layouts), one 200-step run, final state
download. Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(operator="strict", residual_tol=bench.TOL, max_iters=bench.MAX_ITERS, chebyshev=False)
    shard = bench.Shard(0, 1, 0)
    shard.pin()
    out = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fbs = shard.batches(shard.pinned)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ci = sum(fb.run(cfg, bench.SIM_STEPS)["contact_iterations"] for fb in fbs)
        t2 = time.perf_counter()
        n = fbs[0].S * fbs[0].n_scene
        xh = torch.empty(n, dtype=torch.float64).pin_memory()
        vh = torch.empty(n, dtype=torch.float64).pin_memory()
        fbs[0].state_into(xh.numpy(), vh.numpy())
        t3 = time.perf_counter()
        for fb in fbs:
            fb.close()
        out.append({"create_s": t1 - t0, "run_s": t2 - t1, "download_s": t3 - t2, "total_s": t3 - t0,
                    "h2d_bytes": sum(fb.h2d_bytes for fb in fbs), "fem_create_s": fbs[0].timings["create_s"],
                    "node_layout_s": fbs[0].timings["node_layout_s"]})
    print(json.dumps({"workload": "configs[2] e2e breakdown", "reps": out}), flush=True)


if __name__ == "__main__":
    main()
