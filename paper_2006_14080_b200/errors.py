"""Exception types, named and typed as the reference's (so callers that catch
csrecon's exceptions keep working)."""


class ShapeMismatchError(ValueError):
    """Operand shapes or dtypes are incompatible (tensor.py:17-18)."""


class MemoryBudgetError(RuntimeError):
    """Device memory exhausted (operators.py:26-27)."""


class CgDivergenceError(RuntimeError):
    """CG residual turned non-finite (solver.py:30-31)."""


class SpmdError(RuntimeError):
    """Collective failure across workers (sharding.py:18-19)."""


class NativeError(RuntimeError):
    """The CUDA library is missing or a CUDA/NCCL call failed."""
