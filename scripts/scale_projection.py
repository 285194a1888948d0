"""Per-rank cost of `bench.py --gpus N` measured on ONE GPU (a projection, not a
multi-GPU measurement): for each N, the scene block rank N-1 would own
(`batch.shard_bounds(1024, N, N-1)`) is built and run exactly as bench.py's
rank does (FemBatch.run, 200 steps, no host sync per step; cluster kernel when
the block is too small to fill the GPU), timed with CUDA events on the
pipeline stream. With no data-path collective, an N-GPU run takes
max over ranks of this time plus the closing NCCL all-reduce / gather (not
included here). Prints one JSON line per N.

usage: python scripts/scale_projection.py [--ns 1 2 4 8] [--steps 3] [--warmup 1]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cluster", type=int, default=0, help="force CTAs per scene (tuning key 9; 0 = automatic)")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(operator="strict", residual_tol=bench.TOL, max_iters=bench.MAX_ITERS, chebyshev=False)
    h = _lib.handle(0)
    if a.cluster:
        h.L.vfpi_set_tuning(h.h, 9, a.cluster)
    stream = h.torch_stream()
    base = None
    for n in a.ns:
        shard = bench.Shard(n - 1, n, 0)
        batches = shard.batches()

        def one():
            ci = 0
            for fb in batches:
                fb.reset()
            for fb in batches:
                ci += fb.run(cfg, bench.SIM_STEPS)["contact_iterations"]
            return ci

        for _ in range(a.warmup):
            one()
        torch.cuda.synchronize()
        ms, ci = [], 0
        for _ in range(a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ci += one()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.median(ms))
        if base is None:
            base = t * n
        line = {"n_gpus_projected": n, "rank": n - 1, "scenes": [shard.lo, shard.hi], "ms_per_run_rank": t,
                "ms_per_run_all": ms, "rank_contact_iter_per_s": ci / (sum(ms) * 1e-3),
                "projected_job_contact_iter_per_s": n * ci / (sum(ms) * 1e-3),
                "projected_strong_scaling_eff": base / (n * t),
                "note": "one GPU running rank N-1's block alone; excludes the closing NCCL all-reduce/gather"}
        print(json.dumps(line), flush=True)
        for fb in batches:
            fb.close()


if __name__ == "__main__":
    main()
