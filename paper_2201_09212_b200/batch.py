"""Scene batches: many independent systems per call, sharded across ranks.

``solve_scenes`` solves a list of independent augmented systems (each a
reference ``AugmentedDynamics`` or a ``PackedSystem``) with ``solve_vfpi``
semantics per scene — own iteration count, convergence test and divergence
flag — in one ``vfpi_solve_scenes`` launch per chunk of <= 1024 scenes (one
CTA per scene on the device).

``solve_scenes_sharded`` is the multi-GPU form: contiguous
scene blocks per rank, no data-path collective, and one gather of the
per-scene results to rank 0 plus a sum/max reduction of the counters at the
end. The per-rank solver is injectable so the host-side sharding logic is
testable on CPU (gloo) with the oracle as the per-scene solver.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import VfpiConfig, as_f64, as_i32, ptr
from .errors import DivergenceError
from .solver import SolverConfig, SolverReport, _c_config, _raise_for
from .system import PackedSystem, make_packed, pack

MAX_SCENES_PER_LAUNCH = 1024


class _SceneResult(C.Structure):
    """vfpi_scene_result (include/vfpi.h)."""

    _fields_ = [
        ("v", _lib._f64p), ("lam", _lib._f64p), ("residual_trace", _lib._f64p), ("scc", _lib._f64p),
        ("iterations", C.POINTER(C.c_int32)), ("converged", C.POINTER(C.c_int32)),
        ("diverged", C.POINTER(C.c_int32)), ("consistency", _lib._f64p),
        ("setup_ms", C.c_double), ("loop_ms", C.c_double),
    ]


def _bind():
    L = _lib.lib()
    if not hasattr(L, "_scenes_bound"):
        fn = L.vfpi_solve_scenes
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.POINTER(_lib.VfpiSystem), C.c_int32, _lib._i32p, _lib._i32p,
                       C.POINTER(VfpiConfig), _lib._f64p, _lib._f64p, C.POINTER(_SceneResult)]
        L._scenes_bound = True
    return L


def concat_scenes(scenes: list) -> tuple[PackedSystem, np.ndarray, np.ndarray]:
    """Block-diagonal concatenation -> (system, scene_row_ptr, scene_ct_ptr)."""
    ps = [pack(s) for s in scenes]
    rows = np.zeros(len(ps) + 1, dtype=np.int64)
    cts = np.zeros(len(ps) + 1, dtype=np.int64)
    nnzs = np.zeros(len(ps) + 1, dtype=np.int64)
    for k, p in enumerate(ps):
        rows[k + 1] = rows[k] + p.n
        cts[k + 1] = cts[k] + p.n_c
        nnzs[k + 1] = nnzs[k] + p.nnz
    if rows[-1] >= 2**31 or nnzs[-1] >= 2**31:
        raise ValueError("scene batch too large for int32 indices; split it")
    indptr = np.concatenate([p.indptr[:-1].astype(np.int64) + nnzs[k] for k, p in enumerate(ps)] + [nnzs[-1:]])
    indices = np.concatenate([p.indices.astype(np.int64) + rows[k] for k, p in enumerate(ps)]) if ps else []
    col_i = np.concatenate([p.col_i.astype(np.int64) + rows[k] for k, p in enumerate(ps)])
    col_j = np.concatenate([np.where(p.col_j >= 0, p.col_j.astype(np.int64) + rows[k], -1) for k, p in enumerate(ps)])
    cat = make_packed(
        int(rows[-1]), indptr, indices, np.concatenate([p.data for p in ps]), np.concatenate([p.b for p in ps]),
        col_i, col_j, np.concatenate([p.frames for p in ps]), np.concatenate([p.mu for p in ps]),
        np.concatenate([p.mu2 for p in ps]), np.concatenate([p.phi for p in ps]))
    return cat, as_i32(rows), as_i32(cts)


@dataclass
class SceneBatchReport:
    reports: list = field(default_factory=list)
    setup_ms: float = 0.0
    loop_ms: float = 0.0
    wall_s: float = 0.0


def _solve_chunk(scenes, cfg: SolverConfig, warms, device=None):
    h = _lib.handle(device)
    L = _bind()
    cat, rptr, cptr = concat_scenes(scenes)
    S = len(scenes)
    warm = as_f64(np.concatenate([as_f64(w) for w in warms])) if warms is not None else np.zeros(cat.n)
    if warm.shape != (cat.n,):
        raise ValueError("warm starts do not match the scenes")
    tr = max(int(cfg.max_iters), 1)
    v = np.empty(cat.n)
    lam = np.empty((cat.n_c, 3))
    trace = np.empty((S, tr))
    scc = np.empty(cat.n_c)
    iters = np.empty(S, dtype=np.int32)
    conv = np.empty(S, dtype=np.int32)
    div = np.empty(S, dtype=np.int32)
    cons = np.empty(S)
    res = _SceneResult()
    res.v, res.lam, res.residual_trace, res.scc = ptr(v), ptr(lam), ptr(trace), ptr(scc)
    i32 = C.POINTER(C.c_int32)
    res.iterations, res.converged, res.diverged = ptr(iters, i32), ptr(conv, i32), ptr(div, i32)
    res.consistency = ptr(cons)
    code = L.vfpi_solve_scenes(h.h, cat.c_struct(), S, ptr(rptr, _lib._i32p), ptr(cptr, _lib._i32p),
                               _c_config(cfg), ptr(warm), None, res)
    _raise_for(code, h)
    out = []
    for k in range(S):
        r0, r1, c0, c1 = rptr[k], rptr[k + 1], cptr[k], cptr[k + 1]
        it = int(iters[k])
        if div[k]:
            out.append(DivergenceError("non-finite iterate in V-FPI", trace[k, :it].tolist()))
            continue
        rep = SolverReport(iterations=it, residual_trace=trace[k, :it].tolist(), lam=lam[c0:c1].copy(),
                           converged=bool(conv[k]), diverged=False,
                           scc_residuals=scc[c0:c1].copy() if c1 > c0 else None, consistency=float(cons[k]))
        out.append((v[r0:r1].copy(), lam[c0:c1].copy(), rep))
    return out, float(res.setup_ms), float(res.loop_ms)


def solve_scenes(scenes: list, cfg: SolverConfig, warms=None, device=None):
    """Solve independent scenes. Returns (results, SceneBatchReport); results[k]
    is ``(v, lam, SolverReport)`` or a ``DivergenceError`` for a diverged scene."""
    t0 = time.perf_counter()
    results, rep = [], SceneBatchReport()
    for a in range(0, len(scenes), MAX_SCENES_PER_LAUNCH):
        chunk = scenes[a:a + MAX_SCENES_PER_LAUNCH]
        w = None if warms is None else warms[a:a + MAX_SCENES_PER_LAUNCH]
        out, su, lo = _solve_chunk(chunk, cfg, w, device)
        results.extend(out)
        rep.setup_ms += su
        rep.loop_ms += lo
    rep.reports = [r[2] if isinstance(r, tuple) else r for r in results]
    rep.wall_s = time.perf_counter() - t0
    return results, rep


def shard_bounds(num_scenes: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced scene block of ``rank``."""
    per = num_scenes // world
    extra = num_scenes % world
    lo = rank * per + min(rank, extra)
    hi = lo + per + (1 if rank < extra else 0)
    return lo, hi


def solve_scenes_sharded(scenes: list, cfg: SolverConfig, warms=None, group=None, solver=None, device=None):
    """Multi-rank scene batch. Every rank passes the same scene list; rank r
    solves its contiguous block with ``solver`` (default: the GPU
    ``solve_scenes`` on the rank's device) and rank 0 receives every scene's
    result in order. Returns (results or None on ranks > 0, totals) where
    totals = {'contact_iterations': sum over all scenes, 'max_solve_s': max
    over ranks} reduced over the group."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(len(scenes), world, rank)
    mine = scenes[lo:hi]
    my_w = None if warms is None else warms[lo:hi]
    t0 = time.perf_counter()
    if solver is None:
        if device is None:
            device = _lib.default_device()  # the rank's own GPU (torch's current device / LOCAL_RANK)
        local, _ = solve_scenes(mine, cfg, my_w, device=device) if mine else ([], None)
    else:
        local = [solver(s, cfg, None if my_w is None else my_w[k]) for k, s in enumerate(mine)]
    dt = time.perf_counter() - t0
    ci = 0
    for s, r in zip(mine, local):
        if isinstance(r, tuple):
            ci += pack(s).n_c * r[2].iterations
    totals = {"contact_iterations": ci, "max_solve_s": dt, "scenes": len(mine)}
    if world == 1:
        return local, totals
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(ci), dt, float(len(mine))], dtype=torch.float64, device=dev)
    s_ = t.clone()
    dist.all_reduce(s_, op=dist.ReduceOp.SUM, group=group)
    m_ = t.clone()
    dist.all_reduce(m_, op=dist.ReduceOp.MAX, group=group)
    totals = {"contact_iterations": int(s_[0].item()), "max_solve_s": float(m_[1].item()),
              "scenes": int(s_[2].item())}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(local, gathered, dst=0, group=group)
    if rank != 0:
        return None, totals
    out = []
    for part in gathered:
        out.extend(part)
    return out, totals
