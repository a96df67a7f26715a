"""Exception types — mirror of the reference's ``minima.errors`` (errors.py:4-33).

The C-ABI reports failures as ``tnl_status`` codes; ``_native.check`` maps
them onto these classes so callers of the reference API catch the same types.
"""


class MinimaError(Exception):
    """Base class for all package-specific errors (errors.py:4)."""


class ShapeError(MinimaError):
    """Incompatible tensor shapes or mode sizes (errors.py:8)."""


class NumericsError(MinimaError):
    """Non-finite values where finite floats are required (errors.py:12)."""


class RankError(MinimaError):
    """Requested ranks are out of the feasible range (errors.py:16)."""


class DegenerateReferenceError(MinimaError):
    """Relative error against a zero-norm reference is undefined (errors.py:20)."""


class InfeasibleBudgetError(MinimaError):
    """A parameter budget below the smallest admissible configuration (errors.py:24-33)."""

    def __init__(self, message, best_achievable=None):
        super().__init__(message)
        self.best_achievable = best_achievable


class DeviceError(MinimaError):
    """CUDA failure, missing GPU, or missing native library (no CPU fallback exists)."""


class UnsupportedError(MinimaError):
    """Valid layer, but no kernel exists for the request."""
