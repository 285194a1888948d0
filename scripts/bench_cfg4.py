"""configs[4] measurement: a pile of 8x8x4 deformable 16^3-node cubes
(3,145,728 DOF per scene) stepped entirely on one GPU by PileStepper
(device contact detection + nodalization, right-hand side, augmentation,
V-FPI solve, integration), with per-step timings, the streaming kernel's
algorithmic-byte roofline and the fraction of contact steps that converge.
Prints one JSON line.

Scene parameters BASELINE leaves open (recorded in the output): side 0.1 m
(configs[0]'s cube), lateral gap 5 mm with jitter U[-2,2] mm in x and y,
layers and the bottom layer 0.5 mm apart (no z jitter: stacked cubes would
otherwise start interpenetrating), tol 1e-8, max_iters 500, k_v 1e2 (SURVEY's
1e5 comes from unit-mass rigid bodies; against 16^3-node FEM cubes, whose
node mass term (2/dt) m is about 1, k_v = 1e5 makes the non-converged
V-FPI impulses pump energy into the pile until the mesh tears; 1e3 already
does so at this resolution, 1e2 stays bounded -- scripts/pile_trace.py).

usage: python scripts/bench_cfg4.py [--steps 400] [--kv 100] [--scenes 1] [--max-iters 500]
       [--nodes 16] [--cubes 8 8 4]
Under torchrun the scenes shard across ranks (contiguous blocks, no data-path
collective; counters all-reduced and the wall time max-reduced at the end)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def b_iter(n, nnz_num, n_c):
    return 12 * nnz_num + 4 * (n + 1) + 32 * n + 128 * n_c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--scenes", type=int, default=1)
    ap.add_argument("--first-scene", type=int, default=0,
                    help="seed of the first variant (e.g. 224 with --scenes 32: the share of rank 7 of 8 of the 256)")
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--nodes", type=int, default=16)
    ap.add_argument("--cubes", type=int, nargs=3, default=[8, 8, 4])
    ap.add_argument("--kv", type=float, default=100.0)
    ap.add_argument("--chebyshev", action="store_true")
    ap.add_argument("--csv", default="", help="write scene 0's per-step metrics in the reference CSV format")
    ap.add_argument("--tune", nargs="*", default=[], help="key=value tuning knobs of the handle (vfpi_set_tuning)")
    a = ap.parse_args()
    import torch

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    dev = torch.cuda.current_device()
    from paper_2201_09212_b200 import _lib

    for kv in a.tune:
        k, v = kv.split("=")
        _lib.handle(dev).L.vfpi_set_tuning(_lib.handle(dev).h, int(k), int(v))
    from paper_2201_09212_b200.pile import CubePile, PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    peak = 6650.0
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        peak = float(json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    cfg = SolverConfig(residual_tol=1e-8, max_iters=a.max_iters, chebyshev=a.chebyshev)
    from paper_2201_09212_b200.pile import run_piles_sharded

    last = {}

    def make_pile(sc):
        return CubePile(*a.cubes, nodes=a.nodes, gap=0.005, jitter=0.002, gap_z=0.0005, jitter_z=0.0,
                        seed=a.first_scene + sc, k_v=a.kv)

    def stepper(pile):
        last["st"] = PileStepper(pile, device=dev)
        return last["st"]

    # warm-up on a throwaway two-cube pile in contact (loads the lazily-loaded
    # kernels of every stage outside the timed run)
    wp = PileStepper(CubePile(1, 1, 2, nodes=4, gap=0.0, jitter=0.0, gap_z=0.0, jitter_z=0.0, k_v=a.kv), device=dev)
    for _ in range(3):
        wp.step(cfg)
    del wp
    torch.cuda.synchronize()
    res, tot = run_piles_sharded(a.scenes, a.steps, cfg, make_pile, stepper=stepper)
    wall = tot["wall_s"]
    if rank == 0:
        allrows = [r for sc in res for r in sc["rows"]]
        rows = [{k2: (round(v, 4) if isinstance(v, float) else v) for k2, v in r.items()} for r in res[0]["rows"]]
        totals = dict(steps=tot["scene_steps"], contact_iterations=tot["contact_iterations"],
                      iterations=tot["iterations"],
                      bytes=sum((b_iter(r["n"], r["nnz"], r["n_c"]) + (8 * r["n"] if a.chebyshev else 0)) * r["vfpi_iterations"]
                                for r in allrows),
                      loop_s=sum(r["loop_ms"] for r in allrows) * 1e-3,
                      setup_s=sum(r["setup_ms"] for r in allrows) * 1e-3)
        if a.csv:
            from paper_2201_09212_b200.metrics import report_csv
            from paper_2201_09212_b200.pile import step_metrics_row

            report_csv([step_metrics_row(k, r) for k, r in enumerate(res[0]["rows"])], a.csv)
        last = last["st"]
        ctc = [r for r in rows if r["n_c"] > 0]
        loop_gbs = totals["bytes"] / totals["loop_s"] / 1e9 if totals["loop_s"] > 0 else 0.0
        out = {"workload": f"configs[4] cube pile {a.cubes[0]}x{a.cubes[1]}x{a.cubes[2]} cubes of {a.nodes}^3 nodes",
               "scenes": a.scenes, "n_gpus": world, "steps_per_scene": a.steps, "n_orig": last.pile.n,
               "nnz_A_o": int(last.pile.a_data.shape[0]), "dt": last.pile.dt, "mu": last.pile.mu, "k_v": last.pile.k_v,
               "tol": cfg.residual_tol, "max_iters": cfg.max_iters, "operator": "strict", "chebyshev": a.chebyshev,
               "seeds": f"scene k uses default_rng(k) for its jitter, k = {a.first_scene} .. {a.first_scene + a.scenes - 1}", "gap_m": 0.005, "gap_z_m": 0.0005,
               "jitter_m": 0.002,
               "wall_s": wall, "scene_steps_per_s": totals["steps"] / wall,
               "contact_iter_per_s": totals["contact_iterations"] / wall,
               "loop": {"iterations": totals["iterations"], "loop_s": totals["loop_s"], "setup_s": totals["setup_s"],
                        "achieved_gbs": loop_gbs, "peak_gbs": peak, "frac": loop_gbs / peak,
                        "bytes_rule": "12 nnz + 4 (n+1) + 32 n + 128 n_c per iteration (SURVEY 8(d))"},
               "contact_steps": len(ctc),
               "converged_contact_steps": int(sum(bool(r["converged"]) for r in ctc)),
               "converged_fraction": (float(np.mean([bool(r["converged"]) for r in ctc])) if ctc else None),
               "diverged_steps": int(sum(bool(r["diverged"]) for r in rows)),
               "mean_contacts": float(np.mean([r["n_c"] for r in ctc])) if ctc else 0.0,
               "mean_iterations_contact_steps": float(np.mean([r["iterations"] for r in ctc])) if ctc else 0.0,
               "per_step_first_scene": rows[-5:]}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
