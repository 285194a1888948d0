"""configs[2]: batched FEM scenes, sharded over ranks.

    python scripts/bench_scenes.py [--scenes 1024] [--steps 200] [--nx 10]
    torchrun --nproc-per-node N scripts/bench_scenes.py ...

Each rank owns a contiguous block of seeded FemCube scenes (E ~ U[5e4, 2e5],
drop ~ U[0.02, 0.1] m, yaw ~ U[0, 2 pi)), steps them with one
vfpi_solve_scenes launch per step (one CTA per scene), and at the end the
ranks all-reduce the counters (sum of contact-iterations, max of device solve
time) and gather the final node positions to rank 0. Host-side FEM assembly
and contact detection are outside the timed solve (SURVEY §8(f) item 1 moves
them to the device).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _cpu_scene(args):
    """One configs[2] scene stepped on the host with the oracle solver (CPU baseline worker)."""
    E, drop, yaw, nx, steps = args
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import vfpi_oracle as O  # CPU baseline only
    from paper_2201_09212_b200.scenes import FemCube

    cube = FemCube(nx=nx, E=E, drop=drop, yaw=yaw)
    prev = None
    ci = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        ps = cube.system()
        s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                     ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
        v, lam, rep = O.solve(s, O.Config(residual_tol=1e-8, max_iters=500), np.zeros(ps.n) if prev is None else prev)
        ci += ps.n_c * rep.iterations
        cube.advance(v)
        prev = v
    return ci, time.perf_counter() - t0


def cpu_baseline(E, drop, yaw, nx, steps):
    """a process pool of P = len(sched_getaffinity) workers, one scene
    per task; the sample is the first P scenes of the batch, all their steps."""
    import multiprocessing as mp

    P = len(os.sched_getaffinity(0))
    work = [(float(E[k]), float(drop[k]), float(yaw[k]), nx, steps) for k in range(min(P, len(E)))]
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(P) as pool:
        res = pool.map(_cpu_scene, work)
    wall = time.perf_counter() - t0
    ci = sum(r[0] for r in res)
    return {"value": ci / wall, "unit": "contact-iter/s", "cores": P, "kind": "port",
            "scene_steps_per_s": len(work) * steps / wall, "wall_s": wall,
            "sample": f"the first {len(work)} scenes x {steps} steps, one process per core (host FemCube assembly + "
                      "numpy/scipy oracle restating solve_vfpi), pool start-up included"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--nx", type=int, default=10)
    ap.add_argument("--seed", type=int, default=2022)
    ap.add_argument("--chebyshev", action="store_true")
    ap.add_argument("--cpu-baseline", action="store_true", help="time the host CPU path on a bounded sample")
    ap.add_argument("--solve-only-steps", type=int, default=0,
                    help="time only the last K steps (earlier steps still run)")
    ap.add_argument("--host-pipeline", action="store_true",
                    help="assemble/detect/integrate on the host (default: vfpi_fem_step on the device)")
    args = ap.parse_args()
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    from paper_2201_09212_b200.batch import shard_bounds, solve_scenes
    from paper_2201_09212_b200.scenes import FemCube
    from paper_2201_09212_b200.solver import SolverConfig

    g = np.random.default_rng(args.seed)
    E = g.uniform(5e4, 2e5, args.scenes)
    drop = g.uniform(0.02, 0.1, args.scenes)
    yaw = g.uniform(0, 2 * np.pi, args.scenes)
    lo, hi = shard_bounds(args.scenes, world, rank)
    t0 = time.perf_counter()
    cubes = [FemCube(nx=args.nx, E=float(E[k]), drop=float(drop[k]), yaw=float(yaw[k])) for k in range(lo, hi)]
    t_build = time.perf_counter() - t0
    cfg = SolverConfig(residual_tol=1e-8, max_iters=500, chebyshev=args.chebyshev)
    if not args.host_pipeline:
        return device_pipeline(args, cubes, cfg, t_build, rank, world, dist, torch)
    warms = [np.zeros(c.n) for c in cubes]
    solve_ms = 0.0
    setup_ms = 0.0
    ci = 0
    iters = 0
    t_host = 0.0
    t_wall0 = time.perf_counter()
    for step in range(args.steps):
        th = time.perf_counter()
        systems = [c.system() for c in cubes]
        t_host += time.perf_counter() - th
        res, rep = solve_scenes(systems, cfg, warms=warms, device=local)
        solve_ms += rep.setup_ms + rep.loop_ms
        setup_ms += rep.setup_ms
        for k, (c, s, r) in enumerate(zip(cubes, systems, res)):
            v, lam, sr = r
            ci += s.n_c * sr.iterations
            iters += sr.iterations
            c.advance(v)
            warms[k] = v
    wall = time.perf_counter() - t_wall0
    tot = torch.tensor([float(ci), solve_ms, wall, float(iters)], dtype=torch.float64, device="cuda")
    if dist:
        s_ = tot.clone()
        dist.all_reduce(s_, op=dist.ReduceOp.SUM)
        m_ = tot.clone()
        dist.all_reduce(m_, op=dist.ReduceOp.MAX)
        ci_all, solve_max, wall_max, it_all = s_[0].item(), m_[1].item(), m_[2].item(), s_[3].item()
        xs = [c.x for c in cubes]
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(xs, gathered, dst=0)
    else:
        ci_all, solve_max, wall_max, it_all = ci, solve_ms, wall, iters
    if rank == 0:
        line = {"metric": "contact-iterations/sec", "workload": "configs[2] batched FEM scenes",
                "scenes": args.scenes, "n_gpus": world, "steps": args.steps, "nx": args.nx,
                "value": ci_all / (solve_max * 1e-3), "unit": "contact-iter/s",
                "device_solve_s": solve_max * 1e-3, "device_setup_s_rank0": setup_ms * 1e-3, "scene_steps_per_s_solve": args.scenes * args.steps / (solve_max * 1e-3),
                "scene_steps_per_s_wall": args.scenes * args.steps / wall_max, "mean_iters": it_all / (args.scenes * args.steps),
                "contact_iterations": ci_all, "host_build_s": t_build, "host_assembly_s_rank0": t_host,
                "chebyshev": args.chebyshev, "scaling": "strong (fixed scene count split over ranks)"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def device_pipeline(args, cubes, cfg, t_build, rank, world, dist, torch):
    """Whole step loop on the device (FemBatch / vfpi_fem_step), chunks of <= 1024 scenes per rank."""
    from paper_2201_09212_b200.fembatch import FemBatch

    chunks = [FemBatch(cubes[a:a + 1024]) for a in range(0, len(cubes), 1024)]
    # warm-up on a throwaway one-cube batch (same config, pressed into the plane so
    # the contact path runs): loads the kernels lazily-loaded modules would
    # otherwise load inside the first timed step
    from paper_2201_09212_b200.scenes import FemCube

    wcube = FemCube(nx=args.nx, drop=0.0)
    wcube.x = wcube.X.copy()
    wcube.x[:, 2] -= 5e-4
    wb = FemBatch([wcube])
    for _ in range(3):
        wb.step(cfg)
    wb.close()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ci = iters = contacts = 0
    step_ms = setup_ms = loop_ms = 0.0
    t0 = time.perf_counter()
    for step in range(args.steps):
        for fb in chunks:
            st = fb.step(cfg)
            ci += st["contact_iterations"]
            iters += st["iterations"]
            contacts += st["contacts"]
            step_ms += st["step_ms"]
            setup_ms += st["setup_ms"]
            loop_ms += st["loop_ms"]
    wall = time.perf_counter() - t0
    tot = torch.tensor([float(ci), step_ms, wall, float(iters)], dtype=torch.float64, device="cuda")
    if dist:
        s_ = tot.clone()
        dist.all_reduce(s_, op=dist.ReduceOp.SUM)
        m_ = tot.clone()
        dist.all_reduce(m_, op=dist.ReduceOp.MAX)
        ci_all, step_max, wall_max, it_all = s_[0].item(), m_[1].item(), m_[2].item(), s_[3].item()
        xs = [fb.state()[0] for fb in chunks]
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(xs, gathered, dst=0)
    else:
        ci_all, step_max, wall_max, it_all = ci, step_ms, wall, iters
    if rank == 0:
        line = {"metric": "contact-iterations/sec", "workload": "configs[2] batched FEM scenes, device step pipeline",
                "scenes": args.scenes, "n_gpus": world, "steps": args.steps, "nx": args.nx,
                "value": ci_all / wall_max, "unit": "contact-iter/s",
                "scene_steps_per_s_wall": args.scenes * args.steps / wall_max,
                "device_step_ms_total": step_max, "device_setup_ms_rank0": setup_ms, "device_loop_ms_rank0": loop_ms,
                "wall_s": wall_max, "mean_iters": it_all / (args.scenes * args.steps), "contact_iterations": ci_all,
                "host_build_s": t_build, "chebyshev": args.chebyshev,
                "seed": args.seed, "operator": cfg.operator, "tol": cfg.residual_tol, "max_iters": cfg.max_iters,
                "scene_params": "E ~ U[5e4, 2e5], drop ~ U[0.02, 0.1] m, yaw ~ U[0, 2pi) from default_rng(seed)",
                "scaling": "strong (fixed scene count split over ranks)"}
        if args.cpu_baseline and world == 1:
            g = np.random.default_rng(args.seed)
            E = g.uniform(5e4, 2e5, args.scenes)
            drop = g.uniform(0.02, 0.1, args.scenes)
            yaw = g.uniform(0, 2 * np.pi, args.scenes)
            line["cpu_baseline"] = cpu_baseline(E, drop, yaw, args.nx, args.steps)
        print(json.dumps(line), flush=True)
    for fb in chunks:
        fb.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
