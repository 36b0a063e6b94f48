"""B200-native ADMM compressed-sensing MRI reconstruction (arXiv 2006.14080
hot path), drop-in for the csrecon reference API.

The public names mirror csrecon/__init__.py:14-21 for the hot path
(encoding operator, transform, vector algebra, ADMM/CG solver, sharding).
All arithmetic runs in libcsrecon_b200.so (hand-written sm_100a CUDA behind
a C ABI, include/csrecon_b200.h); PyTorch only provides device memory and
streams.  There is no CPU fallback.
"""

from .acquisition import (ImageGrid, KSpaceDataset, SensitivityMaps, Trajectory,
                          simulate_kspace)
from .errors import (CgDivergenceError, MemoryBudgetError, NativeError,
                     ShapeMismatchError, SpmdError)
from .operators import (DEFAULT_MEMORY_BUDGET, ChunkedDftOperator, DftFactors,
                        DftOperator, build_factors, sample_chunking)
from .sharding import (CommStats, ShardPlan, allreduce_sum, coil_shard_plan,
                       default_chunk_size, make_shard_plan, ordered_chunk_sum,
                       sample_shard_plan)
from .solver import (AdmmState, CgOutcome, ReconParams, RunReport,
                     admm_reconstruct, admm_step, adjoint_reconstruct, build_rhs,
                     cg_solve, normal_operator, objective, relative_change_sq,
                     should_continue)
from .tensor import axpy, hermitian_dot, norm2_squared
from .transform import soft_threshold, theta, theta_adjoint

__version__ = "0.1.0"


def active_backend():
    """The only backend: sm_100a CUDA (cf. kernels.active_backend,
    kernels.py:50-53)."""
    return "cuda-sm100a"


__all__ = [
    "ImageGrid", "KSpaceDataset", "SensitivityMaps", "Trajectory", "simulate_kspace",
    "CgDivergenceError", "MemoryBudgetError", "NativeError", "ShapeMismatchError",
    "SpmdError", "DEFAULT_MEMORY_BUDGET", "ChunkedDftOperator", "DftFactors",
    "DftOperator", "build_factors", "sample_chunking", "CommStats", "ShardPlan",
    "allreduce_sum", "coil_shard_plan", "default_chunk_size", "make_shard_plan",
    "ordered_chunk_sum", "sample_shard_plan", "AdmmState", "CgOutcome",
    "ReconParams", "RunReport", "admm_reconstruct", "admm_step",
    "adjoint_reconstruct", "build_rhs", "cg_solve", "normal_operator",
    "objective", "relative_change_sq", "should_continue", "axpy",
    "hermitian_dot", "norm2_squared", "soft_threshold", "theta",
    "theta_adjoint", "active_backend",
]
