"""Per-launch algorithmic bytes of the configs[2] iteration kernel (bench.py's
batch, its 200 steps), to pair an ncu capture of launch k (e.g. the
``--launch-skip 150 -c 1`` one) with the bytes that launch should move.
Prints one JSON line: per step the kernel time, SURVEY §8(d) algorithmic bytes
and the node-block layout's streamed bytes."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from bench import MAX_ITERS, NX, SIM_STEPS, TOL, bytes_per_scene_iter, scene_params
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.scenes import fem_assemble
    from paper_2201_09212_b200.solver import SolverConfig

    E, drop, yaw = scene_params()
    plan, X, kd, ad, m3 = fem_assemble(NX, E, drop, yaw)
    fb = FemBatch.assembled(plan, X, kd, ad, m3)
    cost = bytes_per_scene_iter(np.count_nonzero(ad, axis=1), plan["n"]).astype(np.float64)
    cfg = SolverConfig(residual_tol=TOL, max_iters=MAX_ITERS)
    rows = []
    for step in range(SIM_STEPS):
        st = fb.step(cfg, per_scene=True)
        its = st["iterations_per_scene"].astype(np.float64)
        alg = float(np.dot(cost, its)) + 128.0 * st["contact_iterations"]
        lay = float(its.sum()) * fb.layout_bytes_per_scene_iter + 128.0 * st["contact_iterations"]
        rows.append(dict(step=step, loop_ms=st["loop_ms"], algorithmic_bytes=alg, layout_bytes=lay,
                         iterations=int(its.sum()), contacts=int(st["contacts"])))
    print(json.dumps({"node_kernel": fb.node_kernel, "layout_bytes_per_scene_iter": fb.layout_bytes_per_scene_iter,
                      "steps": rows}))


if __name__ == "__main__":
    main()
