"""configs[3] stepped on the device: a ``scenes.HeightfieldBlock`` (64^3 nodes,
786,432 DOF) pressed onto z = 0.005 sin(40x) sin(40y).

Per step, all on the device (the reference's harness loop, harness.py:538-617,
for this scene): b = (2/dt) M v - K (x - X) + M g + f_ext
(``vfpi_fem_rhs_sell_device`` with K packed once as SELL-32, then
``vfpi_add_device``), node-vs-heightfield contacts
(``vfpi_heightfield_contacts_device``), the V-FPI solve warm-started from the
previous step (``vfpi_solve_device``; single-system streaming kernel), the
contact-free CG step if it diverges (``vfpi_cg_device``, harness.py:586-593)
and midpoint integration (``vfpi_advance_device``). A and K stay resident.
The host restatement (the checker) is ``oracle/fem_host.py``
(``heightfield_rhs`` / ``heightfield_contacts`` / ``fem_advance``).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .solver import _c_config, _raise_for


class HeightfieldStepper:
    def __init__(self, blk, device: int | None = None):
        import torch

        self.h = _lib.handle(device)
        self.blk, self.device = blk, self.h.device
        self.dev = torch.device("cuda", self.device)
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.dev)  # noqa: E731
        A = blk.A
        self.a = (up(A.indptr, np.int32), up(A.indices, np.int32), up(A.data, np.float64))
        k = (up(blk.K.indptr, np.int64), up(blk.K.indices, np.int32), up(blk.K.data, np.float64))  # K^T = K bitwise
        n = blk.n
        nsl = (n + 31) // 32
        self.k_off = torch.empty(nsl + 1, dtype=torch.int64, device=self.dev)
        elems = C.c_int64(0)
        L, hh = self.h.L, self.h.h
        _raise_for(L.vfpi_sell_layout_device(hh, n, k[0].data_ptr(), self.k_off.data_ptr(), C.byref(elems)), self.h)
        self.k_val = torch.empty(max(elems.value, 1), dtype=torch.float64, device=self.dev)
        self.k_col = torch.empty(max(elems.value, 1), dtype=torch.int32, device=self.dev)
        _raise_for(L.vfpi_sell_pack_device(hh, n, k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(),
                                           self.k_off.data_ptr(), self.k_val.data_ptr(), self.k_col.data_ptr()),
                   self.h)
        del k
        self.m, self.g = up(blk.m, np.float64), up(blk.gravity, np.float64)
        self.f_ext = up(blk.f_ext, np.float64)
        self.X = up(blk.X.ravel(), np.float64)
        self.x = up(blk.x.ravel(), np.float64)
        self.v = up(blk.v.ravel(), np.float64)
        self.b = torch.empty(n, dtype=torch.float64, device=self.dev)
        self.vh = torch.empty(n, dtype=torch.float64, device=self.dev)
        self.warm = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.prm = _lib.VfpiHeightfieldParams(blk.amp, blk.freq, blk.amp * blk.freq, blk.margin, blk.mu,
                                              -(blk.beta / blk.dt))
        self.steps = 0
        self.last = None

    def state(self):
        return self.x.cpu().numpy().reshape(-1, 3), self.v.cpu().numpy().reshape(-1, 3)

    def _p(self, t):
        return C.c_void_p(t.data_ptr())

    def contacts_device(self):
        """Device detection of the current state, copied to the host (checks)."""
        import torch

        oc = _lib.VfpiHeightfieldContacts()
        h = self.h
        _raise_for(h.L.vfpi_heightfield_contacts_device(h.h, C.byref(self.prm), self.blk.n // 3, self._p(self.x),
                                                        C.byref(oc), None), h)
        n_c = int(oc.n_c)
        out = {}
        for name, cnt, dt in (("col_i", n_c, np.int32), ("col_j", n_c, np.int32), ("frames", 9 * n_c, np.float64),
                              ("mu", n_c, np.float64), ("phi", n_c, np.float64)):
            out[name] = _lib.device_to_numpy(getattr(oc, name), cnt, dt, self.device)
        torch.cuda.synchronize(self.device)
        return out

    def step(self, cfg) -> dict:
        import torch

        blk, h, P = self.blk, self.h, self._p
        L = h.L
        st = h.stream_ptr()  # everything on the handle's stream, in order
        sp_ = C.c_void_p(st)
        t0 = time.perf_counter()
        n = blk.n
        _raise_for(L.vfpi_fem_rhs_sell_device(h.h, n, P(self.k_off), P(self.k_val), P(self.k_col), P(self.x),
                                              P(self.X), P(self.v), P(self.m), P(self.g), blk.dt, P(self.b), sp_), h)
        _raise_for(L.vfpi_add_device(h.h, n, P(self.f_ext), P(self.b), sp_), h)
        oc = _lib.VfpiHeightfieldContacts()
        _raise_for(L.vfpi_heightfield_contacts_device(h.h, C.byref(self.prm), n // 3, P(self.x), C.byref(oc), sp_),
                   h)
        t_detect = time.perf_counter() - t0
        n_c = int(oc.n_c)
        s = _lib.VfpiSystem()
        s.n, s.n_c, s.nnz = n, n_c, int(blk.A.nnz)
        s.indptr, s.indices = (C.cast(P(t), _lib._i32p) for t in self.a[:2])
        s.data = C.cast(P(self.a[2]), _lib._f64p)
        s.b = C.cast(P(self.b), _lib._f64p)
        s.col_i, s.col_j, s.frames, s.mu, s.phi = oc.col_i, oc.col_j, oc.frames, oc.mu, oc.phi
        s.mu2 = oc.mu
        lam = torch.empty(max(3 * n_c, 1), dtype=torch.float64, device=self.dev)
        trace = torch.empty(max(cfg.max_iters, 1), dtype=torch.float64, device=self.dev)
        res = _lib.VfpiResult()
        res.v, res.lam, res.residual_trace = (C.cast(P(t), _lib._f64p) for t in (self.vh, lam, trace))
        res.scc, res.w = None, None
        code = L.vfpi_solve_device(h.h, C.byref(s), _c_config(cfg), C.cast(P(self.warm), _lib._f64p), None,
                                   C.byref(res), sp_)
        _raise_for(code, h)
        code = L.vfpi_wait(h.h, C.byref(res))
        if code not in (_lib.OK, _lib.DIVERGED):
            _raise_for(code, h)
        diverged = code == _lib.DIVERGED
        if diverged:  # harness.py:586-593: contact-free CG step, lam = 0
            cg_it = C.c_int32(0)
            _raise_for(L.vfpi_cg_device(h.h, n, P(self.a[0]), P(self.a[1]), P(self.a[2]), P(self.b), P(self.vh),
                                        1e-10, 10 * n, C.byref(cg_it), sp_), h)
            lam.zero_()
        depth_max = None
        if n_c:
            # deepest contact (phi = -(beta/dt) depth) before integrating
            phi_t = torch.empty(n_c, dtype=torch.float64, device=self.dev)
            _lib.lib().vfpi_memcpy_d2d(phi_t.data_ptr(), oc.phi, 8 * n_c)
            depth_max = phi_t.min()
        _raise_for(L.vfpi_advance_device(h.h, n, blk.dt, P(self.vh), P(self.x), P(self.v), sp_), h)
        torch.cuda.ExternalStream(st, device=self.dev).synchronize()
        self.warm.copy_(self.vh)
        it = int(res.iterations)
        ke = float(0.5 * torch.dot(self.m * self.v, self.v))
        resid = float(trace[it - 1]) if it > 0 and not diverged else 0.0
        max_pen = 0.0 if depth_max is None else float(depth_max) * (-(blk.dt / blk.beta))
        self.steps += 1
        self.last = dict(v_hat=self.vh, lam=lam[: 3 * n_c])
        return dict(n_c=n_c, n=n, vfpi_iterations=it, iterations=0 if diverged else it,
                    converged=bool(res.converged) and not diverged, diverged=diverged,
                    setup_ms=float(res.setup_ms), loop_ms=float(res.loop_ms), detect_s=t_detect,
                    residual=resid, max_pen_m=max_pen, ke_J=ke, wall_s=time.perf_counter() - t0)

    def metrics_row(self, step: int, r: dict):
        """``harness.MetricsRow`` (``harness.py:598-611``) of a step result."""
        from .pile import step_metrics_row

        return step_metrics_row(step, r)
