"""ctypes binding of libcsrecon_b200.so (include/csrecon_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2006_14080_b200.build``).  There is no CPU fallback: if the
library or a CUDA device is missing, every operator raises.
"""

import ctypes
import os
import threading

from .errors import (CgDivergenceError, MemoryBudgetError, NativeError,
                     ShapeMismatchError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcsrecon_b200.so")
# profiling variants (tools/build_variants.py) live next to the product
# library; CSR_VARIANT=<name> loads paper_2006_14080_b200/variants/<name>.so
if os.environ.get("CSR_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants",
                            os.environ["CSR_VARIANT"] + ".so")

CSR_OK, CSR_ERR_SHAPE, CSR_ERR_OOM, CSR_ERR_CUDA, CSR_ERR_NCCL, \
    CSR_ERR_NONFINITE, CSR_ERR_ARG = range(7)


class PlanDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("n_frames", ctypes.c_int32), ("n_coils", ctypes.c_int32),
                ("n_samples", ctypes.c_int64),
                ("coords", ctypes.POINTER(ctypes.c_double)),
                ("sens", ctypes.c_void_p), ("device", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("chunk_samples", ctypes.c_int64),
                ("total_samples", ctypes.c_int64)]

CSR_PLAN_FRAME_SHARD = 1
CSR_PLAN_ORDERED_SAMPLES = 2


class FactorDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("n_coils", ctypes.c_int32), ("n_samples", ctypes.c_int64),
                ("phase0", ctypes.c_void_p), ("phase1", ctypes.c_void_p),
                ("phase1_layout", ctypes.c_int32), ("sens", ctypes.c_void_p),
                ("device", ctypes.c_int32)]

CSR_P1_ROWS, CSR_P1_T, CSR_P1_CONJ = 0, 1, 2


class PlanInfo(ctypes.Structure):
    _fields_ = [("factor_bytes", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("gemm_path", ctypes.c_int32), ("split_k", ctypes.c_int32)]


class AdmmParams(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("lam_t", ctypes.c_double),
                ("beta", ctypes.c_double), ("admm_rtol", ctypes.c_double),
                ("cg_atol", ctypes.c_double), ("admm_max_iters", ctypes.c_int32),
                ("cg_max_iters", ctypes.c_int32)]


class IterLog(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_int32), ("cg_iterations", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("cg_final_residual_sq", ctypes.c_double)]


class RunStats(ctypes.Structure):
    _fields_ = [("n_iterations", ctypes.c_int32), ("allreduce_calls", ctypes.c_int32),
                ("setup_ms", ctypes.c_double), ("solve_ms", ctypes.c_double),
                ("graph_used", ctypes.c_int32), ("kernels_per_iter", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64, _F, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double

SIGNATURES = {
    "csr_plan_create": [ctypes.POINTER(PlanDesc), ctypes.POINTER(_P)],
    "csr_plan_create_from_factors": [ctypes.POINTER(FactorDesc), ctypes.POINTER(_P)],
    "csr_plan_destroy": [_P],
    "csr_nudft_forward_sep": [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I64, _P],
    "csr_nudft_adjoint_sep": [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I64, _P],
    "csr_plan_get_info": [_P, ctypes.POINTER(PlanInfo)],
    "csr_plan_get_factors": [_P, _I32, _P, _P, _P],
    "csr_forward": [_P, _P, _P, _P],
    "csr_adjoint": [_P, _P, _P, _P],
    "csr_adjoint_chunks": [_P, _P, _P, _P],
    "csr_adjoint_chunks_bound": [_P, _P, _P, _F, _P],
    "csr_sample_chunking": [_I32, _I32, _I32, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I32)],
    "csr_normal": [_P, _P, _P, _D, _P],
    "csr_theta": [_I32, _I32, _I32, _P, _P, _P],
    "csr_theta_adjoint": [_I32, _I32, _I32, _P, _P, _P],
    "csr_soft_threshold": [_P, _I64, _F, _P, _P],
    "csr_hermitian_dot": [_P, _P, _I64, _P, _P],
    "csr_abs_sum": [_P, _I64, _P, _P],
    "csr_axpy": [_D, _D, _P, _P, _I64, _P, _P],
    "csr_admm_run": [_P, ctypes.POINTER(AdmmParams), _P, _P, ctypes.POINTER(IterLog),
                     ctypes.POINTER(RunStats), _P, _P],
    "csr_plan_set_timing": [_P, _P, _I64, _P],
    "csr_plan_kernel_times": [_P, _P, _P, _P, _P],
    "csr_plan_probe": [_P, _I32, _P, _P],
    "csr_simulate_kspace": [_I32, _I32, _I32, _I32, _I64, _P, _P, _P, _P, _P],
    "csr_adjoint_reconstruct": [_P, _P, _P, _P],
    "csr_comm_unique_id": [_P],
    "csr_comm_create": [_P, _I32, _I32, _I32, ctypes.POINTER(_P)],
    "csr_comm_destroy": [_P],
    "csr_plan_set_comm": [_P, _P],
    "csr_comm_allreduce": [_P, _P, _I64, _P],
    "csr_last_error": [],
    "csr_kernel_launches": [],
}
RESTYPES = {"csr_last_error": ctypes.c_char_p, "csr_kernel_launches": ctypes.c_int64}

_lib = None
_lock = threading.Lock()


def load(path=LIB_PATH):
    """Load (once) and return the native library; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeError(
                f"{path} is missing: the CUDA extension has not been built "
                "(run __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def last_error():
    return load().csr_last_error().decode(errors="replace")


def check(rc):
    """Map a CSR_* status to the reference's exception types."""
    if rc == CSR_OK:
        return
    msg = last_error()
    if rc == CSR_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if rc == CSR_ERR_NONFINITE:
        raise CgDivergenceError(msg)
    if rc == CSR_ERR_OOM:
        raise MemoryBudgetError(msg)
    if rc == CSR_ERR_ARG:
        raise ValueError(msg)
    raise NativeError(f"csrecon_b200 error {rc}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))
