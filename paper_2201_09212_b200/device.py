"""Device-resident solves: inputs already in HBM (torch tensors as plain
device memory), enqueued on a caller's CUDA stream via ``vfpi_solve_device``.

PyTorch is plumbing here (allocation, streams, events); the solve itself is
``libvfpi.so``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import VfpiResult, VfpiSystem
from .solver import SolverConfig, _c_config, _raise_for
from .system import PackedSystem


def _dptr(t: torch.Tensor, typ):
    return C.cast(C.c_void_p(t.data_ptr()), typ)


class DeviceSystem:
    """A PackedSystem copied once into device memory on ``device``."""

    def __init__(self, ps: PackedSystem, device: int = 0):
        self.ps = ps
        self.device = device
        dev = torch.device("cuda", device)

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self.t = {k: up(getattr(ps, k)) for k in ("indptr", "indices", "data", "b", "col_i", "col_j", "frames",
                                                   "mu", "mu2", "phi")}
        n, n_c = ps.n, ps.n_c
        self.v = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        self.lam = torch.empty(max(3 * n_c, 1), dtype=torch.float64, device=dev)
        self.scc = torch.empty(max(n_c, 1), dtype=torch.float64, device=dev)
        self.trace = torch.empty(1, dtype=torch.float64, device=dev)
        self.sysc = VfpiSystem()
        s, t = self.sysc, self.t
        s.n, s.n_c, s.nnz = n, n_c, ps.nnz
        i32, f64 = _lib._i32p, _lib._f64p
        s.indptr, s.indices = _dptr(t["indptr"], i32), _dptr(t["indices"], i32)
        s.data, s.b = _dptr(t["data"], f64), _dptr(t["b"], f64)
        s.col_i, s.col_j = _dptr(t["col_i"], i32), _dptr(t["col_j"], i32)
        s.frames, s.mu = _dptr(t["frames"], f64), _dptr(t["mu"], f64)
        s.mu2, s.phi = _dptr(t["mu2"], f64), _dptr(t["phi"], f64)

    def enqueue(self, cfg: SolverConfig, warm: torch.Tensor, stream: torch.cuda.Stream | None = None) -> VfpiResult:
        """Enqueue one solve on ``stream`` (default: torch's current stream); no host sync
        except the one inside layout setup. Call ``finish`` to get the scalars."""
        h = _lib.handle(self.device)
        if self.trace.numel() < max(cfg.max_iters, 1):
            self.trace = torch.empty(max(cfg.max_iters, 1), dtype=torch.float64, device=self.v.device)
        res = VfpiResult()
        f64 = _lib._f64p
        res.v, res.lam, res.residual_trace = _dptr(self.v, f64), _dptr(self.lam, f64), _dptr(self.trace, f64)
        res.scc, res.w = _dptr(self.scc, f64), None
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        # torch's default stream is the legacy NULL stream; the C-ABI reads NULL
        # as "the handle's own stream", so pass cudaStreamLegacy explicitly
        sp = st.cuda_stream if st.cuda_stream else 1
        code = h.L.vfpi_solve_device(h.h, self.sysc, _c_config(cfg), _dptr(warm, f64), None, res, C.c_void_p(sp))
        _raise_for(code, h)
        self._res = res
        return res

    def finish(self) -> VfpiResult:
        h = _lib.handle(self.device)
        res = self._res
        code = h.L.vfpi_wait(h.h, res)
        if code not in (_lib.OK, _lib.DIVERGED):
            _raise_for(code, h)
        return res
