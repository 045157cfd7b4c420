"""Exception types of the reference API (same names, same base classes)."""


class DenseError(RuntimeError):
    """Mirror of ``adrom.dense.DenseError`` (dense.py:35-36): non-finite
    input, rank deficiency, singular Jacobian, SVD non-convergence."""


class RomStepError(RuntimeError):
    """Mirror of ``adrom.projection.RomStepError`` (projection.py:37-38)."""
