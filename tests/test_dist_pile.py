"""configs[4] scene sharding on CPU: gloo, world_size 2, with a
host stepper driven by the oracle (test-only). Rank 0 must receive the same
per-scene final states and rows as a single-rank run, and the reduced
counters must add up. The GPU stepper of the same function is PileStepper."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2201_09212_b200.pile import CubePile, run_piles_sharded


class OracleStepper:
    def __init__(self, pile):
        self.pile, self.prev = pile, None

    def step(self, cfg):
        from oracle import pile_host as H
        from oracle import vfpi_oracle as O

        p = self.pile
        pc = H.contacts(p)
        a_p, a_i, a_x, b = O.augment(p.n, p.a_indptr, p.a_indices, p.a_data, H.rhs(p), pc.jv, p.k_v)
        s = O.System(p.n + pc.jv.shape[0], a_p, a_i, a_x, b, pc.col_i, pc.col_j, pc.frames, pc.mu, pc.mu, pc.phi)
        v, lam, rep = O.solve(s, O.Config(residual_tol=cfg.residual_tol, max_iters=cfg.max_iters),
                              H.warm(p, self.prev, pc))
        H.advance(p, v)
        self.prev = v
        return dict(n_c=pc.n_c, n_ground=pc.n_ground, n_face=pc.n_face, iterations=rep.iterations,
                    converged=rep.converged)

    def state(self):
        return self.pile.x, self.pile.v


def make_pile(sc):
    return CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=3, gap=0.0, jitter=0.0001, seed=100 + sc)


def _cfg():
    from paper_2201_09212_b200.solver import SolverConfig

    return SolverConfig(residual_tol=1e-8, max_iters=60)


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res, tot = run_piles_sharded(3, 3, _cfg(), make_pile, stepper=OracleStepper)
        if rank == 0:
            np.savez(out, **{f"x{r['scene']}": r["x"] for r in res}, **{f"v{r['scene']}": r["v"] for r in res},
                     ci=tot["contact_iterations"], steps=tot["scene_steps"],
                     nc=np.array([[row["n_c"] for row in r["rows"]] for r in res]))
    finally:
        dist.destroy_process_group()


def test_pile_shards_match_single_rank(tmp_path):
    single, tot1 = run_piles_sharded(3, 3, _cfg(), make_pile, stepper=OracleStepper)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    d = np.load(out)
    assert int(d["steps"]) == tot1["scene_steps"] == 9
    assert int(d["ci"]) == tot1["contact_iterations"] and tot1["contact_iterations"] > 0
    for r in single:
        assert np.array_equal(d[f"x{r['scene']}"], r["x"]) and np.array_equal(d[f"v{r['scene']}"], r["v"])
    assert d["nc"].tolist() == [[row["n_c"] for row in r["rows"]] for r in single]
