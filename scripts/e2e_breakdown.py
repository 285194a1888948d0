"""configs[1] e2e breakdown: pinned H2D bandwidth, vfpi_solve (host buffers) wall vs its setup/loop, device path."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200._lib import VfpiResult, ptr  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, _c_config  # noqa: E402
from paper_2201_09212_b200.system import PackedSystem  # noqa: E402

ps = rigid_contact_system()
keys = ("indptr", "indices", "data", "b", "col_i", "col_j", "frames", "mu", "mu2", "phi")
pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(ps, k))).pin_memory() for k in keys}
nbytes = sum(t.numel() * t.element_size() for t in pin.values())
dev = {k: torch.empty_like(t, device="cuda") for k, t in pin.items()}
for _ in range(3):
    for k in keys:
        dev[k].copy_(pin[k], non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    for k in keys:
        dev[k].copy_(pin[k], non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"H2D {nbytes/1e6:.1f} MB pinned: {dt*1e3:.3f} ms = {nbytes/dt/1e9:.1f} GB/s")
pps = PackedSystem(ps.n, *[pin[k].numpy() for k in keys])
cfg = _c_config(SolverConfig(residual_tol=1e-8, max_iters=1000))
h = _lib.handle(0)
warm = torch.zeros(ps.n, dtype=torch.float64).pin_memory().numpy()
ov = torch.empty(ps.n, dtype=torch.float64).pin_memory().numpy()
ol = torch.empty(3 * ps.n_c, dtype=torch.float64).pin_memory().numpy()
ot = torch.empty(1000, dtype=torch.float64).pin_memory().numpy()
os_ = torch.empty(ps.n_c, dtype=torch.float64).pin_memory().numpy()
for rep in range(6):
    res = VfpiResult()
    res.v, res.lam, res.residual_trace, res.scc, res.w = ptr(ov), ptr(ol), ptr(ot), ptr(os_), None
    t0 = time.perf_counter()
    code = h.L.vfpi_solve(h.h, pps.c_struct(), cfg, ptr(warm), None, res)
    wall = time.perf_counter() - t0
    print(f"vfpi_solve wall {wall*1e3:.3f} ms  setup {res.setup_ms:.3f}  loop {res.loop_ms:.3f}  code {code}")
