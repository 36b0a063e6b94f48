"""Complex vector primitives on the device (mirror of csrecon/tensor.py).

hermitian_dot accumulates in f64 with a deterministic two-stage reduction
(K8); axpy casts alpha to complex64 first, as tensor.py:58-64 does.
"""

import numpy as np

from . import _dev, _native
from .errors import ShapeMismatchError

COMPLEX_DTYPES = {"single": np.complex64}
REAL_DTYPES = {"single": np.float32}
PRECISIONS = ("single",)


def validate_precision(precision):
    """Only "single" (complex64) exists on this path; "double" is rejected
    rather than silently run on the CPU (no CPU fallback)."""
    if precision == "double":
        raise ValueError("precision 'double' is not supported by the B200 path "
                         "(complex64 kernels only; use the reference for f64)")
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}, got {precision!r}")
    return precision


def _pair(a, b):
    if tuple(a.shape) != tuple(b.shape):
        raise ShapeMismatchError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    dev = _dev.device_of(a if _dev.is_tensor(a) else b)
    ta = _dev.as_c64(a, a.shape, "a", dev)
    tb = _dev.as_c64(b, b.shape, "b", dev)
    return dev, ta, tb


def hermitian_dot(a, b):
    """<a, b> = sum(conj(a) * b) (tensor.py:44-50); returns a Python complex."""
    dev, ta, tb = _pair(a, b)
    out = _dev.torch.empty(2, dtype=_dev.torch.float64, device=dev)
    _native.call("csr_hermitian_dot", ta.data_ptr(), tb.data_ptr(), ta.numel(),
                 out.data_ptr(), _dev.stream_ptr(dev))
    re, im = out.tolist()
    return complex(re, im)


def norm2_squared(a):
    """Re<a, a> (tensor.py:53-55)."""
    return hermitian_dot(a, a).real


def axpy(alpha, x, y):
    """y + alpha * x with alpha cast to complex64 (tensor.py:58-64)."""
    dev, tx, ty = _pair(x, y)
    a = complex(np.complex64(alpha))
    out = _dev.empty_c64(tx.shape, dev)
    _native.call("csr_axpy", a.real, a.imag, tx.data_ptr(), ty.data_ptr(),
                 tx.numel(), out.data_ptr(), _dev.stream_ptr(dev))
    return _dev.out_like(out, y)
