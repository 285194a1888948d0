"""Exception taxonomy of the reference (``condsim/errors.py:1-48``).

When the reference package is importable its classes are reused, so code
written against ``condsim`` catches the drop-in's errors unchanged.
"""

try:  # pragma: no cover - depends on the environment
    from condsim.errors import (  # type: ignore
        CondsimError,
        DimensionMismatchError,
        DivergenceError,
        InvalidMatrixError,
    )
except Exception:  # the reference is not installed: same names, same bases

    class CondsimError(Exception):
        """Base class for all solver errors."""

    class DimensionMismatchError(CondsimError, ValueError):
        """Vector or matrix dimensions do not agree."""

    class InvalidMatrixError(CondsimError):
        """Matrix violates a structural requirement (zero row, broken tie group)."""

    class DivergenceError(CondsimError):
        """Fixed-point iteration produced a non-finite iterate; carries the trace."""

        def __init__(self, message, residual_trace=None):
            super().__init__(message)
            self.residual_trace = list(residual_trace) if residual_trace is not None else []


class DeviceError(RuntimeError):
    """CUDA failure inside libvfpi.so (no CPU fallback exists)."""


class UnsupportedInputError(CondsimError):
    """Input the GPU solver rejects (e.g. two contacts on one node column)."""
