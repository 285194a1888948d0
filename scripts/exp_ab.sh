# A/B of the resident kernel: exp/libvfpi_pair.so vs the default build; parity of the variant
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
for lib in exp/libvfpi_oldres.so exp/libvfpi_pair.so; do
  echo "== $lib"; VFPI_LIB=$lib timeout 200 python /tmp/ab.py 2>&1 | tail -1
done; done
VFPI_LIB=exp/libvfpi_pair.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_bench_contract.py 2>&1 | tail -3
