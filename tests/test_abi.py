"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point include/*.h declares (no compute calls here)."""

import ctypes
import glob
import os
import re
import subprocess

import pytest

from conftest import REPO
from paper_2006_14080_b200 import _native


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(csr_\w+)\s*\(",
                                text, flags=re.M))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("csr_plan_create", "csr_forward", "csr_adjoint", "csr_admm_run",
                 "csr_theta", "csr_theta_adjoint", "csr_soft_threshold",
                 "csr_hermitian_dot", "csr_axpy", "csr_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) <= set(_native.SIGNATURES)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_calls_fail_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _native.load()
    desc = _native.PlanDesc(nx=4, ny=4, n_frames=1, n_coils=1, n_samples=4,
                            coords=None, sens=None, device=0, flags=0)
    plan = ctypes.c_void_p()
    rc = lib.csr_plan_create(ctypes.byref(desc), ctypes.byref(plan))
    assert rc != 0
    coords = (ctypes.c_double * 8)()
    desc.coords = ctypes.cast(coords, ctypes.POINTER(ctypes.c_double))
    desc.sens = 1
    rc = lib.csr_plan_create(ctypes.byref(desc), ctypes.byref(plan))
    assert rc == _native.CSR_ERR_CUDA
    assert "no CUDA device" in _native.last_error()
