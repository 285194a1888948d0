"""Per-step, per-scene V-FPI iteration counts of configs[2] (all 1024 scenes,
200 steps, device pipeline) -> gpurun_out/iter_profile.npz (load-balance
analysis of the sharded runs)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(operator="strict", residual_tol=bench.TOL, max_iters=bench.MAX_ITERS, chebyshev=False)
    shard = bench.Shard(0, 1, 0)
    fb = shard.batches()[0]
    st = fb.run(cfg, bench.SIM_STEPS, per_step=True)
    its = st["iterations_per_step"]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "iter_profile.npz"), its=its, cts=st["contacts_per_step"])
    print("steps", its.shape, "mean", its.mean(), "max", its.max())


if __name__ == "__main__":
    main()
