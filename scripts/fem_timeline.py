"""Kernel timeline of one FEM batch step (device pipeline) via the CUDA
activity trace (tuning aid). usage: python scripts/fem_timeline.py [scenes]"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2201_09212_b200.fembatch import FemBatch  # noqa: E402
from paper_2201_09212_b200.scenes import FemCube  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = np.random.default_rng(1)
cubes = [FemCube(nx=10, E=float(g.uniform(5e4, 2e5)), drop=0.0005, yaw=float(g.uniform(0, 6.28))) for _ in range(S)]
fb = FemBatch(cubes)
cfg = SolverConfig(residual_tol=1e-8, max_iters=500)
torch.zeros(1, device="cuda")
for _ in range(12):
    st = fb.step(cfg)
print("contacts", st["contacts"], "step_ms", st["step_ms"], "setup_ms", st["setup_ms"], "loop_ms", st["loop_ms"])
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    st = fb.step(cfg)
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = t0
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} us dur {e.time_range.end - e.time_range.start:8.1f} "
          f"gap {e.time_range.start - prev:7.1f}  {e.name[:70]}")
    prev = max(prev, e.time_range.end)
