"""Per-CTA phase timing of the resident iteration kernel on configs[1] (tuning aid)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_09212_b200 import _lib  # noqa: E402
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402
from paper_2201_09212_b200.solver import SolverConfig, solve_packed  # noqa: E402

nb, nc = 4096, 16384
ps = rigid_contact_system(nb, nc, 2201)
if "--nocontacts" in sys.argv:
    from paper_2201_09212_b200.system import make_packed
    ps = make_packed(ps.n, ps.indptr, ps.indices, ps.data, ps.b, [], [], [], [])
h = _lib.handle(0)
for a in sys.argv[1:]:  # key=value tuning knobs, e.g. 1=1 5=0 (anchor order, contact cost)
    if "=" in a:
        k_, v_ = a.split("=")
        h.L.vfpi_set_tuning(h.h, int(k_), int(v_))
cfg = SolverConfig(residual_tol=0.0, max_iters=1000)
solve_packed(ps, cfg, np.zeros(ps.n))
v, lam, rep = solve_packed(ps, cfg, np.zeros(ps.n))
print("layout", h.last_layout(), "loop_ms", rep.timings["loop_s"] * 1e3, "setup_ms", rep.timings["setup_s"] * 1e3)
h.L.vfpi_set_profile(h.h, 500)
solve_packed(ps, cfg, np.zeros(ps.n))
G = h.last_layout()["ctas"]
buf = (C.c_longlong * (64 * G))()
h.L.vfpi_get_profile(h.h, buf, 64 * G)
a = np.frombuffer(buf, dtype=np.int64).reshape(G, 4, 16)
def show(nm, d):
    print(f"{nm:22s} cycles mean {d.mean():9.0f}  max {d.max():9.0f}  min {d.min():9.0f}")
show("products", a[:, :, 2] - a[:, :, 0])
show("pass B contact rows", a[:, :, 3] - a[:, :, 2])
show("contact warps", np.where(a[:, :, 6] > 0, a[:, :, 6] - a[:, :, 3], 0))
show("free-row warps", np.where(a[:, :, 1] > 0, a[:, :, 1] - a[:, :, 3], 0))
show("role phase (sync)", a[:, :, 4] - a[:, :, 3])
show("reduce+barrier", a[:, :, 5] - a[:, :, 4])
tot = a[:, :, 5] - a[:, :, 0]
print(f"{'iteration':16s} cycles mean {tot.mean():9.0f}  max {tot.max():9.0f}")
work = a[:, :, 4] - a[:, :, 0]
print("work (pre-barrier) per CTA: mean", work.mean(), "max", work.max(), "argmax cta", int(work.mean(1).argmax()))
for b_ in (0, 20, 40, 55, 60, 61, 62, 63, 64, 80, 100, 147):
    r = a[b_].mean(0)
    print(f"cta {b_:3d}: stage {r[2]-r[0]:6.0f} passB {r[3]-r[2]:6.0f} role {r[4]-r[3]:6.0f} "
          f"cw {r[6]-r[3] if r[6] > 0 else 0:6.0f} fw {r[1]-r[3] if r[1] > 0 else 0:6.0f} red+bar {r[5]-r[4]:6.0f}"
          + (f" | sweep {r[8]-r[3]:6.0f} oneshot {r[10]-r[8]:6.0f}"
             if r[8] > 0 else ""))
arr = a[:, :, 7]
print("arrival skew (globaltimer ns) per iteration:", (arr.max(0) - arr.min(0)).tolist())
h.L.vfpi_set_profile(h.h, 0)
