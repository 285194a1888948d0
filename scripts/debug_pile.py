"""Debug: device vs host pile contacts after a few steps."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2201_09212_b200.pile import CubePile, PileStepper
from paper_2201_09212_b200.solver import SolverConfig
mk = lambda: CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, gap=0.0, jitter=0.00005, seed=5, dt=5e-4)
dev = PileStepper(mk(), detect="host")
for step in range(4):
    pile = dev.pile
    pile.x = dev.x.cpu().numpy().reshape(-1, 3); pile.v = dev.v.cpu().numpy().reshape(-1, 3)
    hc = pile.contacts()
    dc = dev.device_contacts()
    print("step", step, "n_c", hc.n_c, dc.n_c, "face", hc.n_face, dc.n_face)
    if hc.n_c == dc.n_c:
        for name in ("col_i", "col_j", "frames", "phi", "mu"):
            a, b = getattr(hc, name), getattr(dc, name)
            print("  ", name, np.array_equal(a, b), float(np.abs(np.asarray(a, float) - np.asarray(b, float)).max()) if a.size else 0)
        print("   jv", np.array_equal(hc.jv.indptr, dc.jv.indptr), np.array_equal(hc.jv.indices, dc.jv.indices),
              np.array_equal(hc.jv.data, dc.jv.data), float(np.abs(hc.jv.data - dc.jv.data).max()) if hc.jv.nnz == dc.jv.nnz else "nnz differ")
        bad = np.nonzero(np.any(hc.frames != dc.frames, axis=(1, 2)))[0]
        if bad.size:
            k = bad[0]; print("   first bad frame", k, hc.frames[k], dc.frames[k], sep="\n")
    dev.step(SolverConfig(residual_tol=1e-8, max_iters=200))
