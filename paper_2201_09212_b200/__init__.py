"""B200-native V-FPI contact solver (arXiv 2201.09212, COND).

Drop-in for ``condsim.solver.solve_vfpi``: assembled system in, velocities and
contact impulses out, computed by hand-written sm_100a CUDA kernels in
``libvfpi.so`` (C ABI: ``include/vfpi.h``). No CPU fallback.
"""

from .errors import CondsimError, DimensionMismatchError, DivergenceError, InvalidMatrixError  # noqa: F401
from .solver import (  # noqa: F401
    SolverConfig,
    SolverReport,
    StepMatrix,
    SurrogateDelassus,
    solve_packed,
    solve_vfpi,
)
from .system import AugmentedDynamics, Contact, NodalContactSet, PackedSystem, SparseSymmetric, pack  # noqa: F401

__version__ = "0.1.0"
