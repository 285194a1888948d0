"""Per-step trace of a pile run (physics sanity): contacts, iterations, speeds, penetration."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2201_09212_b200.pile import CubePile, PileStepper
from paper_2201_09212_b200.solver import SolverConfig
import os
args = [int(a) for a in sys.argv[1:]] or [2, 2, 2, 8, 120]
kv = float(os.environ.get("KV", "1e5"))
print("k_v", kv)
pile = CubePile(args[0], args[1], args[2], nodes=args[3], gap=0.005, jitter=0.002, gap_z=0.0005, jitter_z=0.0, seed=0, k_v=kv)
st = PileStepper(pile)
cfg = SolverConfig(residual_tol=1e-8, max_iters=500)
for k in range(args[4]):
    r = st.step(cfg)
    if k % 10 == 0:
        x = st.x.view(-1, 3); v = st.v.view(-1, 3)
        print(k, "n_c", r["n_c"], "g", r["n_ground"], "f", r["n_face"], "its", r["iterations"], "conv", r["converged"],
              "zmin %.2e" % float(x[:, 2].min()), "vmax %.3e" % float(v.abs().max()), "loop %.2f setup %.2f" % (r["loop_ms"], r["setup_ms"]), flush=True)
