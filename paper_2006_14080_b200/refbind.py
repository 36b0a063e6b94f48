"""Bind the B200 kernels into the reference's own kernel table.

The reference dispatches every hot kernel through ``csrecon.kernels._IMPL``
(kernels.py:212-231, dispatchers kernels.py:249-274).  ``install(kernels)``
adds a ``"cuda"`` entry whose functions have the reference's signatures and
numpy-in / numpy-out semantics, and makes it the active table, so the
reference's unmodified operators and solver (DftOperator, admm_reconstruct,
adjoint_reconstruct, ...) run their NUDFTs, finite differences and soft
thresholds on the B200:

    import csrecon.kernels
    import paper_2006_14080_b200.refbind as rb
    rb.install(csrecon.kernels)

The separable NUDFT entries keep one device plan per operator (keyed by the
identity of the operator's ``phase0`` and coil-map arrays, which a
``DftOperator`` holds for its lifetime, operators.py:128-139) built from the
reference's own factor arrays (``csr_plan_create_from_factors``), so repeated
applications cost one H2D copy, the tensor-core contraction and one D2H
copy.  Arithmetic is complex64 (the reference's ``precision="single"``);
complex128 operands raise, as does the materialized mode, whose explicit
(M, N) matrix the B200 path never forms: build
operators with ``mode="separable"``.
"""

import ctypes
import threading
from collections import OrderedDict

import numpy as np

from . import _dev, _native
from .errors import ShapeMismatchError
from .transform import soft_threshold, theta, theta_adjoint

#: operators whose plans stay cached (least recently used beyond this are released)
MAX_PLANS = 512


class _PlanCache:
    """Plans by operator identity; thread-safe (the reference's workers are
    threads, sharding.py:274-314, each with its own operators)."""

    def __init__(self, device=None):
        self.device = device
        self.plans = OrderedDict()
        self.lock = threading.Lock()

    def get(self, phase0, phase1, layout, sens):
        key = (id(phase0), phase0.__array_interface__["data"][0], phase0.shape,
               id(sens), sens.__array_interface__["data"][0], sens.shape)
        with self.lock:
            hit = self.plans.get(key)
            if hit is not None:
                self.plans.move_to_end(key)
                return hit[0]
        entry = self._build(phase0, phase1, layout, sens)
        with self.lock:
            # the arrays stay referenced so their ids cannot be reused while cached
            self.plans[key] = (entry, phase0, sens)
            while len(self.plans) > MAX_PLANS:
                self.plans.popitem(last=False)
        return entry

    def _build(self, phase0, phase1, layout, sens):
        dev = _dev.device_of(None) if self.device is None else _dev.torch.device(self.device)
        m, nx = phase0.shape
        n_coils, sx, sy = sens.shape
        ny = phase1.shape[0] if layout == _native.CSR_P1_T else phase1.shape[1]
        if (sx, sy) != (nx, ny):
            raise ShapeMismatchError(f"sensitivity grid {(sx, sy)} != factor grid {(nx, ny)}")
        t0 = _c64_dev(phase0, dev)
        t1 = _c64_dev(phase1, dev)
        ts = _c64_dev(sens, dev)
        _dev.torch.cuda.current_stream(dev).synchronize()
        fd = _native.FactorDesc(nx=nx, ny=ny, n_coils=n_coils, n_samples=m,
                                phase0=t0.data_ptr(), phase1=t1.data_ptr(),
                                phase1_layout=layout, sens=ts.data_ptr(), device=dev.index)
        plan = ctypes.c_void_p()
        _native.call("csr_plan_create_from_factors", ctypes.byref(fd), ctypes.byref(plan))
        return _Plan(plan, dev, nx, ny, n_coils, m)


class _Plan:
    def __init__(self, plan, dev, nx, ny, n_coils, m):
        self.plan, self.dev = plan, dev
        self.nx, self.ny, self.n_coils, self.m = nx, ny, n_coils, m

    def __del__(self):
        if self.plan is not None and self.plan.value:
            try:
                _native.load().csr_plan_destroy(self.plan)
            except Exception:
                pass
            self.plan = None


def _c64_dev(arr, dev):
    a = np.asarray(arr)
    if a.dtype != np.complex64:
        raise ShapeMismatchError(
            f"dtype {a.dtype}: the B200 kernels compute in complex64 (precision='single')")
    return _dev.torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def kernel_table(device=None):
    """The reference's seven kernel entries (kernels.py:212-231) on the B200."""
    cache = _PlanCache(device)

    def forward_sep(phase0, phase1_t, sens, image):
        p = cache.get(phase0, phase1_t, _native.CSR_P1_T, sens)
        x = _c64_dev(image, p.dev)
        if tuple(x.shape) != (p.nx, p.ny):
            raise ShapeMismatchError(f"image shape {tuple(x.shape)}, expected {(p.nx, p.ny)}")
        out = _dev.empty_c64((p.m, p.n_coils), p.dev)
        _native.call("csr_forward", p.plan, x.data_ptr(), out.data_ptr(), _dev.stream_ptr(p.dev))
        return out.cpu().numpy()

    def adjoint_sep(phase0, phase1_conj, sens, data):
        p = cache.get(phase0, phase1_conj, _native.CSR_P1_CONJ, sens)
        y = _c64_dev(data, p.dev)
        if tuple(y.shape) != (p.m, p.n_coils):
            raise ShapeMismatchError(f"data shape {tuple(y.shape)}, expected {(p.m, p.n_coils)}")
        out = _dev.empty_c64((p.nx, p.ny), p.dev)
        _native.call("csr_adjoint", p.plan, y.data_ptr(), out.data_ptr(), _dev.stream_ptr(p.dev))
        return out.cpu().numpy()

    def materialized(*_):
        raise NotImplementedError(
            "the B200 kernels never form the explicit (M, nx*ny) encoding matrix "
            "(materialized mode); build operators with mode='separable'")

    def soft(z, threshold):
        return soft_threshold(np.asarray(z), float(threshold))

    return {"forward_mat": materialized, "adjoint_mat": materialized,
            "forward_sep": forward_sep, "adjoint_sep": adjoint_sep,
            "theta": theta, "theta_adj": theta_adjoint, "soft": soft,
            "_cache": cache}


def install(kernels, device=None, name="cuda"):
    """Register the B200 table as ``kernels._IMPL[name]`` and make it the
    active backend of the reference's dispatchers (kernels.py:246-274).
    Returns the previous (active table, backend name) for ``uninstall``."""
    prev = (kernels._ACTIVE, kernels._BACKEND)
    table = kernel_table(device)
    kernels._IMPL[name] = table
    kernels._ACTIVE = table
    kernels._BACKEND = name
    return prev


def uninstall(kernels, prev, name="cuda"):
    kernels._ACTIVE, kernels._BACKEND = prev
    kernels._IMPL.pop(name, None)
