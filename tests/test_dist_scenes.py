"""Host-side multi-rank logic of the scene batch on CPU with
gloo, world_size 2. The per-scene solver is the oracle here (test-only); the
GPU path of the same function is covered by tests/test_gpu_scenes.py."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2201_09212_b200.batch import shard_bounds


def test_shard_bounds_cover_and_balance():
    for S in (0, 1, 7, 8, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(S, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scenes():
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from golden_cases import load

    from gpu_util import packed

    names = ["rand_strict_cheb", "rand_prox_conv0", "resting", "diverge_fixed", "rand_bb2", "scn_particle_stack_s2",
             "rand_cheb_ls3"]
    ds = [load(n) for n in names]
    return ds, [packed(d) for d in ds]


def _oracle_solver(ps, cfg, warm):
    from oracle import vfpi_oracle as O

    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    c = O.Config(**{k: getattr(cfg, k) for k in ("operator", "step_strategy", "residual_tol", "max_iters",
                                                 "chebyshev", "cheby_start", "under_relax", "omega",
                                                 "fixed_alpha", "consistency_factor")})
    try:
        with np.errstate(over="ignore", invalid="ignore"):
            v, lam, rep = O.solve(s, c, np.zeros(ps.n) if warm is None else warm)
    except O.OracleDivergence as exc:
        from paper_2201_09212_b200.errors import DivergenceError

        return DivergenceError("non-finite iterate in V-FPI", exc.residual_trace)
    return v, lam, rep


def _worker(rank, world, port, q):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2201_09212_b200.batch import solve_scenes_sharded
    from paper_2201_09212_b200.solver import SolverConfig

    ds, scenes = _scenes()
    cfg = SolverConfig(residual_tol=1e-8, max_iters=3000, chebyshev=True)
    res, totals = solve_scenes_sharded(scenes, cfg, solver=_oracle_solver)
    if rank == 0:
        seq = [_oracle_solver(s, cfg, None) for s in scenes]
        ok = len(res) == len(seq)
        ci = 0
        for a, b_, s in zip(res, seq, scenes):
            if isinstance(b_, tuple):
                ok &= isinstance(a, tuple) and a[2].iterations == b_[2].iterations
                ok &= bool(np.array_equal(a[0], b_[0]))
                ci += s.n_c * b_[2].iterations
            else:
                ok &= not isinstance(a, tuple)
        ok &= totals["contact_iterations"] == ci and totals["scenes"] == len(scenes)
        q.put(bool(ok))
    dist.destroy_process_group()


def test_sharded_scene_batch_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
