"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py <case>
cases: nodes-<op>[-cheb], rows-<op>, resident, streaming, fallback, heightfield, pile, augment."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cubes(nx=5, n=6, seed=3):
    from paper_2201_09212_b200.scenes import FemCube

    g = np.random.default_rng(seed)
    return [FemCube(nx=nx, E=float(g.uniform(5e4, 2e5)), drop=float(g.uniform(0.0005, 0.004)),
                    yaw=float(g.uniform(0, 2 * np.pi))) for _ in range(n)]


def main(case):
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    if case.startswith("nodes") or case.startswith("rows"):
        parts = case.split("-")
        op = {"strict": "strict", "prox": "proximal", "aniso": "strict-anisotropic"}[parts[1]]
        kw = dict(operator=op, chebyshev="cheb" in parts, residual_tol=1e-8, max_iters=60)
        if "alpha" in parts:
            kw["step_strategy"] = "fixed-alpha"
        fb = FemBatch(cubes(), node_layout=case.startswith("nodes"))
        for _ in range(25):
            st = fb.step(SolverConfig(**kw))
        print(case, "node_kernel", st["node_kernel"], "contacts", st["contacts"])
    elif case in ("resident", "streaming"):
        from paper_2201_09212_b200 import _lib
        from paper_2201_09212_b200.scenes import rigid_contact_system

        ps = rigid_contact_system(64, 160, seed=5)
        _lib.handle().set_kernel(case)
        v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-8, max_iters=30), np.zeros(ps.n))
        print(case, rep.iterations, _lib.handle().last_layout())
    elif case == "fallback":
        fb = FemBatch(cubes(n=3))
        st = fb.step(SolverConfig(residual_tol=1e-8, max_iters=50, step_strategy="fixed-alpha", fixed_alpha=1e3))
        st = fb.step(SolverConfig(residual_tol=1e-8, max_iters=50, step_strategy="fixed-alpha", fixed_alpha=1e3))
        print(case, st["diverged_scenes"])
    elif case == "heightfield":
        from paper_2201_09212_b200.heightfield import HeightfieldStepper
        from paper_2201_09212_b200.scenes import HeightfieldBlock

        st = HeightfieldStepper(HeightfieldBlock(nx=8))
        for _ in range(3):
            r = st.step(SolverConfig(residual_tol=1e-8, max_iters=40))
        print(case, r["n_c"], r["iterations"])
    elif case == "pile":
        from paper_2201_09212_b200.pile import CubePile, PileStepper

        st = PileStepper(CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, gap=0.0, jitter=0.00005, seed=5))
        for _ in range(3):
            r = st.step(SolverConfig(residual_tol=1e-8, max_iters=40))
        print(case, r["n_c"], r["n_face"], r["iterations"])
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1])
