"""Drop-in V-FPI solver API (mirror of ``condsim/solver.py``).

Same names, argument meaning and error behaviour as the reference; every
numeric call goes through ``libvfpi.so`` (hand-written sm_100a kernels).
Scalar schedule helpers (``chebyshev_nu``, ``estimate_rho``,
``step_matrix_bb``) are host arithmetic exactly as in the reference.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import VfpiConfig, VfpiResult, as_f64, ptr
from .errors import DeviceError, DimensionMismatchError, DivergenceError, InvalidMatrixError, UnsupportedInputError
from .system import PackedSystem, pack

OPERATORS = ("strict", "proximal", "strict-anisotropic")
STEP_STRATEGIES = ("frobenius", "bb1", "bb2", "bb-alternating", "fixed-alpha")


@dataclass
class StepMatrix:
    """Diagonal surrogate step matrix (``solver.py:37-42``)."""

    w: np.ndarray
    tied_nodes: list = field(default_factory=list)


@dataclass
class SurrogateDelassus:
    gamma: np.ndarray


@dataclass
class SolverConfig:
    """``solver.py:50-62``."""

    operator: str = "strict"
    step_strategy: str = "frobenius"
    residual_tol: float = 1e-4
    max_iters: int = 500
    chebyshev: bool = False
    cheby_start: int = 10
    under_relax: float = 0.9
    omega: float = 0.0
    fixed_alpha: float | None = None
    consistency_factor: float = 10.0
    w_recycle_period: int = 1


@dataclass
class SolverReport:
    """``solver.py:65-74``; ``timings`` adds device times in ms."""

    iterations: int = 0
    residual_trace: list = field(default_factory=list)
    lam: np.ndarray | None = None
    converged: bool = False
    diverged: bool = False
    timings: dict = field(default_factory=dict)
    scc_residuals: np.ndarray | None = None
    consistency: float = float("nan")


def _c_config(cfg) -> VfpiConfig:
    if cfg.operator not in _lib.OPERATORS:
        raise ValueError(f"unknown operator {cfg.operator!r}")
    if cfg.step_strategy not in _lib.STRATEGIES:
        raise ValueError(f"unknown step strategy {cfg.step_strategy!r}")
    c = VfpiConfig()
    c.op = _lib.OPERATORS[cfg.operator]
    c.step_strategy = _lib.STRATEGIES[cfg.step_strategy]
    c.max_iters = int(cfg.max_iters)
    c.chebyshev = 1 if cfg.chebyshev else 0
    c.cheby_start = int(cfg.cheby_start)
    c.residual_tol = float(cfg.residual_tol)
    c.under_relax = float(cfg.under_relax)
    c.omega = float(cfg.omega)
    c.fixed_alpha = float("nan") if cfg.fixed_alpha is None else float(cfg.fixed_alpha)
    c.consistency_factor = float(cfg.consistency_factor)
    return c


def _raise_for(code: int, h, trace=None):
    msg = h.error()
    if code == _lib.OK:
        return
    if code == _lib.DIVERGED:
        raise DivergenceError("non-finite iterate in V-FPI", trace or [])
    if code in (_lib.INVALID_MATRIX, _lib.TIE_VIOLATION):
        raise InvalidMatrixError(msg)
    if code == _lib.DIM_MISMATCH:
        raise DimensionMismatchError(msg)
    if code == _lib.UNSUPPORTED:
        raise UnsupportedInputError(msg)
    if code == _lib.BAD_ARGUMENT:
        raise ValueError(msg)
    raise DeviceError(f"libvfpi error {code}: {msg}")


def _check_tie_host(w: np.ndarray, cols: np.ndarray):
    t = w[cols[:, None] + np.arange(3)]
    if not (np.all(t[:, 0] == t[:, 1]) and np.all(t[:, 0] == t[:, 2])):
        raise InvalidMatrixError("step matrix violates the per-node tie groups")


def solve_packed(ps: PackedSystem, cfg: SolverConfig, warm, w_cached: np.ndarray | None = None, device=None):
    """V-FPI solve of a packed system. Returns (v, lam, SolverReport)."""
    h = _lib.handle(device)
    warm = as_f64(warm)
    if warm.shape != (ps.n,):
        raise DimensionMismatchError(f"spmv: x has shape {warm.shape}, expected ({ps.n},)")
    wc = None
    if w_cached is not None and cfg.step_strategy != "fixed-alpha":
        wc = as_f64(w_cached)
        if wc.shape != (ps.n,):
            raise DimensionMismatchError("w_cached has the wrong length")
    n, n_c = ps.n, ps.n_c
    v = np.empty(n)
    lam = np.empty((n_c, 3))
    trace = np.empty(max(int(cfg.max_iters), 1))
    scc = np.empty(n_c)
    res = VfpiResult()
    res.v, res.lam, res.residual_trace, res.scc = ptr(v), ptr(lam), ptr(trace), ptr(scc)
    res.w = None
    t0 = time.perf_counter()
    sysc = ps.c_struct()
    code = h.L.vfpi_solve(h.h, sysc, _c_config(cfg), ptr(warm), ptr(wc), res)
    wall = time.perf_counter() - t0
    it = int(res.iterations)
    if code == _lib.DIVERGED:
        raise DivergenceError("non-finite iterate in V-FPI", trace[:it].tolist())
    _raise_for(code, h)
    rep = SolverReport(
        iterations=it, residual_trace=trace[:it].tolist(), lam=lam, converged=bool(res.converged),
        diverged=False, scc_residuals=scc if n_c else None, consistency=float(res.consistency),
        timings={"setup_s": res.setup_ms * 1e-3, "loop_s": res.loop_ms * 1e-3, "wall_s": wall},
    )
    return v, lam, rep


def solve_vfpi(aug, cfg: SolverConfig, warm: np.ndarray, w_cached: StepMatrix | None = None,
               project_override=None):
    """Drop-in for ``condsim.solver.solve_vfpi`` (``solver.py:345-461``)."""
    if project_override is not None:
        raise NotImplementedError("project_override callables have no device implementation")
    ps = pack(aug)
    wc = None
    if w_cached is not None and cfg.step_strategy != "fixed-alpha":
        wc = np.asarray(w_cached.w, dtype=float)
        if ps.n_c:  # reference raises from surrogate_gamma before iterating
            _check_tie_host(wc, ps.col_i.astype(np.int64))
            has_j = ps.col_j >= 0
            if has_j.any():
                _check_tie_host(wc, ps.col_j[has_j].astype(np.int64))
    return solve_packed(ps, cfg, warm, wc)


# ---- per-subsystem entry points (reference names) --------------------------

def step_matrix_frobenius(a, aug=None, pair_tie: bool = False) -> StepMatrix:
    """``solver.py:216-229`` on the device."""
    h = _lib.handle()
    if aug is not None:
        ps = pack(aug)
    else:
        from .system import make_packed

        ps = make_packed(a.dim, a.indptr, a.indices, a.data, np.zeros(a.dim), [], [], [], [])
    w = np.empty(ps.n)
    code = h.L.vfpi_step_matrix_frobenius(h.h, ps.c_struct(), 1 if pair_tie else 0, ptr(w))
    _raise_for(code, h)
    tied = []
    if ps.n_c:
        tied = sorted(set(ps.col_i.tolist()) | set(int(c) for c in ps.col_j if c >= 0))
    return StepMatrix(w, tied)


def surrogate_gamma(w: StepMatrix, aug, omega: float = 0.0) -> SurrogateDelassus:
    """``solver.py:244-253`` on the device."""
    h = _lib.handle()
    ps = pack(aug)
    g = np.empty(ps.n_c)
    code = h.L.vfpi_surrogate_gamma(h.h, ps.c_struct(), ptr(as_f64(w.w)), float(omega), ptr(g))
    _raise_for(code, h)
    return SurrogateDelassus(g)


def contact_solve_oneshot(gamma: SurrogateDelassus, eta, phi, mu, operator: str = "strict", mu2=None,
                          omega_included: bool = True, omega: float = 0.0) -> np.ndarray:
    """``solver.py:262-281`` on the device."""
    h = _lib.handle()
    g = as_f64(gamma.gamma if omega_included else np.asarray(gamma.gamma) + omega)
    eta = as_f64(eta).reshape(-1, 3)
    n_c = eta.shape[0]
    mu = as_f64(np.broadcast_to(mu, (n_c,)))
    mu2v = mu if mu2 is None else as_f64(np.broadcast_to(mu2, (n_c,)))
    phi = as_f64(np.broadcast_to(phi, (n_c,)))
    if operator not in _lib.OPERATORS:
        raise ValueError(f"unknown operator {operator!r}")
    lam = np.empty((n_c, 3))
    code = h.L.vfpi_contact_solve_oneshot(h.h, n_c, ptr(g), ptr(eta), ptr(phi), ptr(mu), ptr(mu2v),
                                          _lib.OPERATORS[operator], ptr(lam))
    _raise_for(code, h)
    return lam


def _project_one(lam_star, mu, mu2, operator):
    lam_star = as_f64(lam_star).reshape(1, 3)
    # identity surrogate: gamma = 1, eta = -lam*, phi = 0 gives lam* exactly
    out = contact_solve_oneshot(SurrogateDelassus(np.ones(1)), -lam_star, np.zeros(1), np.array([float(mu)]),
                                operator, None if mu2 is None else np.array([float(mu2)]))
    return out.reshape(3)


def project_strict(lam_star, mu: float) -> np.ndarray:
    """``solver.py:77-85``."""
    return _project_one(lam_star, mu, None, "strict")


def project_proximal(lam_star, mu: float) -> np.ndarray:
    """``solver.py:88-100``."""
    return _project_one(lam_star, mu, None, "proximal")


def project_strict_anisotropic(lam_star, mu1: float, mu2: float) -> np.ndarray:
    """``solver.py:129-141``."""
    return _project_one(lam_star, mu1, mu2, "strict-anisotropic")


def scc_residual(v_contact, lam, phi, mu) -> np.ndarray:
    """``solver.py:304-334`` on the device."""
    h = _lib.handle()
    vc = as_f64(np.atleast_2d(v_contact)).reshape(-1, 3)
    lm = as_f64(np.atleast_2d(lam)).reshape(-1, 3)
    n_c = vc.shape[0]
    phi = as_f64(np.broadcast_to(np.atleast_1d(phi), (n_c,)))
    mu = as_f64(np.broadcast_to(np.atleast_1d(mu), (n_c,)))
    out = np.empty(n_c)
    code = h.L.vfpi_scc_residual(h.h, n_c, ptr(vc), ptr(lm), ptr(phi), ptr(mu), ptr(out))
    _raise_for(code, h)
    return out


def inverse_contact(aug, v_hat, omega: float, operator: str = "proximal") -> np.ndarray:
    """``solver.py:468-475`` on the device."""
    h = _lib.handle()
    ps = pack(aug)
    lam = np.empty((ps.n_c, 3))
    code = h.L.vfpi_inverse_contact(h.h, ps.c_struct(), ptr(as_f64(v_hat)), float(omega),
                                    _lib.OPERATORS[operator], ptr(lam))
    _raise_for(code, h)
    return lam


def chebyshev_nu(l: int, l_s: int, rho: float, nu_prev: float) -> float:
    """``solver.py:284-290`` (the device kernel evaluates the same schedule)."""
    if l < l_s:
        return 1.0
    if l == l_s:
        return 2.0 / (2.0 - rho * rho)
    return 4.0 / (4.0 - rho * rho * nu_prev)


def chebyshev_update(v_ss, v_prevprev, nu: float):
    """``solver.py:293-294``."""
    return nu * (np.asarray(v_ss) - v_prevprev) + v_prevprev


def estimate_rho(norm_l: float, norm_lm1: float, prev_rho: float = 0.0) -> float:
    """``solver.py:297-301``."""
    if norm_lm1 <= 0.0:
        return prev_rho
    return min(norm_l / norm_lm1, 1.0)


def step_matrix_bb(s, z, variant: str, prev_alpha: float) -> float:
    """``solver.py:232-241`` (scalar form; the kernel fuses it per iteration)."""
    sz = float(np.dot(s, z))
    if sz <= 0.0:
        return prev_alpha
    if variant == "bb1":
        return float(np.dot(s, s)) / sz
    if variant == "bb2":
        return sz / float(np.dot(z, z))
    raise ValueError(f"unknown BB variant {variant!r}")


__all__ = [
    "OPERATORS", "STEP_STRATEGIES", "SolverConfig", "SolverReport", "StepMatrix", "SurrogateDelassus",
    "solve_vfpi", "solve_packed", "step_matrix_frobenius", "surrogate_gamma", "contact_solve_oneshot",
    "project_strict", "project_proximal", "project_strict_anisotropic", "scc_residual", "inverse_contact",
    "chebyshev_nu", "chebyshev_update", "estimate_rho", "step_matrix_bb",
]
