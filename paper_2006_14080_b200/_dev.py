"""Device plumbing: numpy <-> torch CUDA complex64 buffers and streams.

PyTorch is only the allocator/stream provider here; all arithmetic runs in
libcsrecon_b200.so.
"""

import numpy as np

from .errors import NativeError, ShapeMismatchError

try:  # torch is plumbing only; the package must import on CPU-only hosts
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise NativeError("a CUDA device is required: csrecon_b200 has no CPU fallback")


def is_tensor(x):
    return torch is not None and isinstance(x, torch.Tensor)


def device_of(x=None):
    require_cuda()
    if is_tensor(x) and x.is_cuda:
        return x.device
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


def as_c64(x, shape, what, device):
    """Return a contiguous complex64 CUDA tensor holding x, checking the shape
    and dtype strictly as DftOperator._check does (operators.py:178-183)."""
    if is_tensor(x):
        if tuple(x.shape) != tuple(shape):
            raise ShapeMismatchError(f"{what} shape {tuple(x.shape)}, expected {tuple(shape)}")
        if x.dtype != torch.complex64:
            raise ShapeMismatchError(f"{what} dtype {x.dtype}, operator runs in complex64")
        return x.to(device).contiguous()
    arr = np.asarray(x)
    if arr.shape != tuple(shape):
        raise ShapeMismatchError(f"{what} shape {arr.shape}, expected {tuple(shape)}")
    if arr.dtype != np.complex64:
        raise ShapeMismatchError(f"{what} dtype {arr.dtype}, operator runs in complex64")
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(device, non_blocking=False)


def empty_c64(shape, device):
    return torch.empty(tuple(shape), dtype=torch.complex64, device=device)


def out_like(result, template):
    """numpy in -> numpy out; tensor in -> tensor out."""
    if is_tensor(template):
        return result
    return result.cpu().numpy()
