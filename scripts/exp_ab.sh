cat > /tmp/ab.py <<'PY'
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2201_09212_b200.scenes import rigid_contact_system
from paper_2201_09212_b200.solver import SolverConfig, solve_packed
ps = rigid_contact_system()
cfg = SolverConfig(residual_tol=1e-8, max_iters=1000)
best = min(solve_packed(ps, cfg, np.zeros(ps.n))[2].timings["loop_s"] for _ in range(6))
print("loop %.3f ms" % (best * 1e3))
PY
for i in 1 2; do
for lib in exp/libvfpi_ru8.so exp/libvfpi_ru6.so exp/libvfpi_ru10.so exp/libvfpi_ru12.so; do
  echo "== $lib"; VFPI_LIB=$lib timeout 200 python /tmp/ab.py 2>&1 | tail -1
done; done
