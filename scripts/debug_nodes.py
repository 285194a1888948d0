"""Step a FEM batch with the node-block kernel, synchronising after every step
(set VFPI_LIB to a -DVFPI_NB_DEBUG build for device-side bounds checks)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    op = sys.argv[1] if len(sys.argv) > 1 else "proximal"
    cheb = "cheb" in sys.argv
    g = np.random.default_rng(3)
    cubes = [FemCube(nx=6, E=float(g.uniform(5e4, 2e5)), drop=float(g.uniform(0.0005, 0.004)),
                     yaw=float(g.uniform(0, 2 * np.pi))) for _ in range(12)]
    fb = FemBatch(cubes, node_layout="rows" not in sys.argv)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=400, operator=op, chebyshev=cheb)
    for step in range(40):
        st = fb.step(cfg, per_scene=True)
        print("step", step, "contacts", st["contacts"], "its", st["iterations_per_scene"].tolist()[:6],
              "node", st["node_kernel"], flush=True)


if __name__ == "__main__":
    main()
