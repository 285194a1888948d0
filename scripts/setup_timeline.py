"""Kernel timeline of one configs[1] solve via the CUDA activity trace
(torch.profiler / CUPTI): per-kernel durations and the idle gaps between them."""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

ps = rigid_contact_system(4096, 16384, 2201)
cfg = SolverConfig(residual_tol=1e-8, max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 50)
torch.zeros(1, device="cuda")
for _ in range(2):
    solve_packed(ps, cfg, np.zeros(ps.n))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
print("setup_ms", rep.timings["setup_s"] * 1e3, "loop_ms", rep.timings["loop_s"] * 1e3)
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = 0.0
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    gap = st - prev_end
    busy += en - st
    print(f"{(st - t0):9.1f} us  dur {en - st:8.1f}  gap {gap:7.1f}  {e.name[:80]}")
    prev_end = max(prev_end, en)
print("span", prev_end - t0, "busy", busy)
