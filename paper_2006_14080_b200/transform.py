"""Circular finite differences and the soft threshold on the device (mirror
of csrecon/transform.py).

theta maps (nx, ny) -> (2, nx, ny) exactly as the reference; a 3-D
(T, nx, ny) input gets the 2-D+t transform (3, T, nx, ny) whose third
component is the circular temporal difference (extension).
"""

import numpy as np

from . import _dev, _native
from .errors import ShapeMismatchError


def theta(image):
    """transform.py:14-18 (+ temporal component for 3-D input)."""
    if image.ndim not in (2, 3):
        raise ShapeMismatchError(f"image must be 2-D (or 3-D T,nx,ny), got shape "
                                 f"{tuple(image.shape)}")
    T, nx, ny = (1,) + tuple(image.shape) if image.ndim == 2 else tuple(image.shape)
    dev = _dev.device_of(image)
    x = _dev.as_c64(image, image.shape, "image", dev)
    D = 2 if image.ndim == 2 else 3
    out = _dev.empty_c64((D,) + tuple(image.shape), dev)
    _native.call("csr_theta", T, nx, ny, x.data_ptr(), out.data_ptr(),
                 _dev.stream_ptr(dev))
    return _dev.out_like(out, image)


def theta_adjoint(diffs):
    """transform.py:21-26 (+ temporal component for (3, T, nx, ny))."""
    ok2 = diffs.ndim == 3 and diffs.shape[0] == 2
    ok3 = diffs.ndim == 4 and diffs.shape[0] == 3
    if not (ok2 or ok3):
        raise ShapeMismatchError(
            f"diff stack must have shape (2, nx, ny) or (3, T, nx, ny), got "
            f"{tuple(diffs.shape)}")
    if ok2:
        T, nx, ny = 1, diffs.shape[1], diffs.shape[2]
    else:
        T, nx, ny = diffs.shape[1], diffs.shape[2], diffs.shape[3]
    dev = _dev.device_of(diffs)
    x = _dev.as_c64(diffs, diffs.shape, "diffs", dev)
    out = _dev.empty_c64(tuple(diffs.shape[1:]), dev)
    _native.call("csr_theta_adjoint", T, nx, ny, x.data_ptr(), out.data_ptr(),
                 _dev.stream_ptr(dev))
    return _dev.out_like(out, diffs)


def soft_threshold(z, threshold):
    """S_t(z) = z*(1 - t/|z|) where |z| > t else 0, t cast to float32
    (transform.py:29-42)."""
    if threshold < 0:
        raise ValueError(f"threshold must be >= 0, got {threshold}")
    dev = _dev.device_of(z)
    x = _dev.as_c64(z, z.shape, "z", dev)
    out = _dev.empty_c64(tuple(z.shape), dev)
    _native.call("csr_soft_threshold", x.data_ptr(), x.numel(),
                 float(np.float32(threshold)), out.data_ptr(), _dev.stream_ptr(dev))
    return _dev.out_like(out, z)
