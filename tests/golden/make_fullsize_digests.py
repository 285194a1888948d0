"""Full-size parity pins at BASELINE sizes, generated here with the CPU oracle
(and cross-checked against the reference package where it applies), checked
on the GPU by ``tests/test_gpu_fullsize_digests.py``:

* configs[2]: four scenes of bench.py's seeded 1024-scene batch (0, 1, 511,
  1023) stepped all 200 steps through the host pipeline
  (``oracle.fem_host.oracle_steps``; the reference pipeline
  ``reference_steps`` gives the same iteration counts and final bits):
  per-step V-FPI iteration counts and SHA-256 of the final x and v;
* configs[3]: the 64^3-node heightfield block at its pressed start state, one
  500-iteration solve, plain (SHA-256 of v and lam) and Chebyshev (norms and a
  strided sample of v and lam, compared to 1e-9);
* configs[4]: the 8x8x4 pile of 16^3-node cubes stacked in contact (k_v 1e2),
  one contact step of 500 iterations from a zero warm start (SHA-256 of v and
  lam).

Inputs are rebuilt on the GPU box by the same deterministic code (their
SHA-256 is stored too, so a host-arithmetic difference shows up as such).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_digests.py [cfg2] [cfg3] [cfg4]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
OUT = os.path.join(HERE, "fullsize_digests.json")

CFG2_SCENES = (0, 1, 511, 1023)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sample(a, k=4001):
    a = np.asarray(a, dtype=np.float64).ravel()
    idx = np.linspace(0, a.size - 1, min(k, a.size)).astype(np.int64)
    return idx.tolist(), a[idx].tolist()


def cfg2():
    from bench import MAX_ITERS, NX, SIM_STEPS, TOL, scene_params
    from oracle import fem_host
    from paper_2201_09212_b200.scenes import FemCube

    E, drop, yaw = scene_params()
    out = {}
    for k in CFG2_SCENES:
        cube = FemCube(nx=NX, E=float(E[k]), drop=float(drop[k]), yaw=float(yaw[k]))
        x_in = sha(cube.X)
        rec = []
        fem_host.oracle_steps(cube, SIM_STEPS, residual_tol=TOL, max_iters=MAX_ITERS, record=rec)
        d = {"input_X": x_in, "iterations": [r["iterations"] for r in rec], "n_c": [r["n_c"] for r in rec],
             "final_x": sha(cube.x), "final_v": sha(cube.v)}
        try:  # the reference pipeline (condsim) around the same FEM matrices
            ref = FemCube(nx=NX, E=float(E[k]), drop=float(drop[k]), yaw=float(yaw[k]))
            rrec = []
            fem_host.reference_steps(ref, SIM_STEPS, residual_tol=TOL, max_iters=MAX_ITERS, record=rrec)
            d["reference_same_iterations"] = [r["iterations"] for r in rrec] == d["iterations"]
            d["reference_same_final_bits"] = sha(ref.x) == d["final_x"] and sha(ref.v) == d["final_v"]
        except ImportError:
            d["reference_same_iterations"] = None
        out[str(k)] = d
        print("cfg2 scene", k, sum(d["iterations"]), d.get("reference_same_iterations"),
              d.get("reference_same_final_bits"), flush=True)
    return out


def _oracle_solve(ps, cfg):
    from oracle import vfpi_oracle as O

    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    return O.solve(s, cfg, np.zeros(ps.n))


def cfg3():
    from oracle import fem_host
    from oracle import vfpi_oracle as O
    from paper_2201_09212_b200.scenes import HeightfieldBlock

    blk = HeightfieldBlock(nx=64)
    ps = fem_host.heightfield_system(blk)
    out = {"input_b": sha(ps.b), "input_data": sha(ps.data), "n_c": int(ps.n_c), "n": int(ps.n)}
    t = time.perf_counter()
    v, lam, rep = _oracle_solve(ps, O.Config(residual_tol=1e-8, max_iters=500))
    out["plain"] = {"iterations": rep.iterations, "converged": rep.converged, "v": sha(v), "lam": sha(lam)}
    print("cfg3 plain", rep.iterations, time.perf_counter() - t, flush=True)
    v, lam, rep = _oracle_solve(ps, O.Config(residual_tol=1e-8, max_iters=500, chebyshev=True))
    iv, sv = sample(v)
    il, sl = sample(lam)
    out["chebyshev"] = {"iterations": rep.iterations, "converged": rep.converged,
                        "v_norm": float(np.linalg.norm(v)), "lam_norm": float(np.linalg.norm(lam)),
                        "v_idx": iv, "v_val": sv, "lam_idx": il, "lam_val": sl}
    print("cfg3 chebyshev", rep.iterations, flush=True)
    return out


def cfg4():
    from oracle import pile_host
    from oracle import vfpi_oracle as O
    from paper_2201_09212_b200.pile import CubePile

    pile = CubePile(gap=0.005, jitter=0.002, gap_z=0.0, jitter_z=0.0, k_v=100.0)
    pc = pile_host.contacts(pile)
    b_o = pile_host.rhs(pile)
    p, i, x, b = O.augment(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, b_o, pc.jv, pile.k_v)
    s = O.System(pile.n + pc.jv.shape[0], p, i, x, b, pc.col_i.astype(np.int64), pc.col_j.astype(np.int64),
                 pc.frames, pc.mu, pc.mu, pc.phi)
    out = {"input_b": sha(b), "input_data": sha(x), "n_c": int(pc.n_c), "n": int(s.n)}
    t = time.perf_counter()
    v, lam, rep = O.solve(s, O.Config(residual_tol=1e-8, max_iters=500), np.zeros(s.n))
    out["plain"] = {"iterations": rep.iterations, "converged": rep.converged, "v": sha(v), "lam": sha(lam)}
    print("cfg4", rep.iterations, time.perf_counter() - t, flush=True)
    return out


def main():
    which = sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for name in which:
        data[name] = globals()[name]()
        with open(OUT, "w") as f:
            json.dump(data, f, indent=0)


if __name__ == "__main__":
    main()
