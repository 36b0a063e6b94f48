"""Multi-coil NUDFT encoding operator on the B200 (mirror of
csrecon/operators.py).

``DftOperator.build`` uploads the coordinates and coil maps and generates
the separable phase factors on the device (f64 angle, one rounding to
complex64 — operators.py:50-82).  forward/adjoint run the tensor-core
separable contraction (K3/K4, ``csrc/nudft_tc.cuh``).  The explicit
(M, nx*ny) matrix of the reference's "materialized" mode is never formed
(SURVEY.md §2.2 K1/K11): ``mode`` is accepted and recorded only.
"""

from dataclasses import dataclass

import ctypes
import numpy as np

from . import _dev, _native
from .acquisition import ImageGrid, sample_coords
from .errors import ShapeMismatchError
from .tensor import validate_precision

DEFAULT_MEMORY_BUDGET = 2 * 1024 ** 3
MODES = ("auto", "materialized", "separable")


@dataclass
class DftFactors:
    """phase0 (M, nx) and phase1 (M, ny) (operators.py:30-47)."""
    phase0: np.ndarray
    phase1: np.ndarray

    @property
    def n_samples(self):
        return self.phase0.shape[0]

    @property
    def grid_shape(self):
        return (self.phase0.shape[1], self.phase1.shape[1])


def _maps_of(sens):
    return getattr(sens, "maps", sens)


class DftOperator:
    """forward(image) -> (n_samples, n_coils); adjoint(data) -> image.

    image is (nx, ny) for n_frames == 1, else (n_frames, nx, ny); frame t
    uses rows [t*M, (t+1)*M) of the coordinates and data.
    """

    def __init__(self, plan, grid, n_coils, n_frames, m_per_frame, device, mode):
        self._plan = plan
        self.grid = grid
        self.nx, self.ny = grid.nx, grid.ny
        self._n_coils = n_coils
        self.n_frames = n_frames
        self.m_per_frame = m_per_frame
        self.device = device
        self.mode = mode
        self.comm = None

    @classmethod
    def build(cls, trajectory, grid, sens, mode="auto", precision="single",
              memory_budget=DEFAULT_MEMORY_BUDGET, n_frames=1, device=None,
              frame_shard=False, chunk_grid=None):
        """operators.py:141-164 (factor-cached, never materialized).

        frame_shard: the frames are one rank's block of a 2-D+t problem split
        over ranks (temporal differences at the block edges use halo frames).
        chunk_grid: (chunk_samples, total_samples) of an order-stable sample
        split (``sample_chunking``); the coordinates are then a run of whole
        chunks of that grid, and every k-space value and chunk partial comes
        out bit-identical to a plan of the whole problem."""
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
        validate_precision(precision)
        maps = _maps_of(sens)
        if tuple(maps.shape[1:]) != tuple(grid.shape):
            raise ShapeMismatchError(
                f"sensitivity grid {tuple(maps.shape[1:])} != image grid {grid.shape}")
        coords = sample_coords(trajectory)
        if coords.shape[0] == 0:
            raise ValueError("trajectory has no samples")
        if n_frames < 1 or coords.shape[0] % n_frames:
            raise ValueError("coords rows must split evenly into n_frames frames")
        dev = _dev.device_of(maps) if device is None else _dev.torch.device(device)
        if _dev.is_tensor(maps):
            tmaps = maps.to(dev, _dev.torch.complex64).contiguous()
        else:
            tmaps = _dev.torch.from_numpy(
                np.ascontiguousarray(np.asarray(maps).astype(np.complex64))).to(dev)
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        m = coords.shape[0] // n_frames
        flags = _native.CSR_PLAN_FRAME_SHARD if frame_shard else 0
        chunk, total = (0, 0) if chunk_grid is None else (int(chunk_grid[0]), int(chunk_grid[1]))
        if chunk_grid is not None:
            flags |= _native.CSR_PLAN_ORDERED_SAMPLES
        desc = _native.PlanDesc(
            nx=grid.nx, ny=grid.ny, n_frames=n_frames, n_coils=tmaps.shape[0],
            n_samples=m,
            coords=coords.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            sens=tmaps.data_ptr(), device=dev.index, flags=flags,
            chunk_samples=chunk, total_samples=total)
        _dev.torch.cuda.current_stream(dev).synchronize()
        plan = ctypes.c_void_p()
        _native.call("csr_plan_create", ctypes.byref(desc), ctypes.byref(plan))
        resolved = "separable" if mode == "auto" else mode
        return cls(plan, ImageGrid(grid.nx, grid.ny), tmaps.shape[0], n_frames, m,
                   dev, resolved)

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                _native.load().csr_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    # -- properties mirroring operators.py:166-176 -------------------------
    @property
    def n_samples(self):
        return self.m_per_frame * self.n_frames

    @property
    def n_coils(self):
        return self._n_coils

    @property
    def dtype(self):
        return np.dtype(np.complex64)

    @property
    def image_shape(self):
        if self.n_frames == 1:
            return (self.nx, self.ny)
        return (self.n_frames, self.nx, self.ny)

    @property
    def plan(self):
        return self._plan

    def info(self):
        info = _native.PlanInfo()
        _native.call("csr_plan_get_info", self._plan, ctypes.byref(info))
        return {"factor_bytes": info.factor_bytes,
                "workspace_bytes": info.workspace_bytes,
                "gemm_path": "tcgen05" if info.gemm_path else "simt",
                "split_k": info.split_k}

    def factors(self, frame=0):
        """The device-generated factors of one frame as DftFactors (numpy)."""
        p0 = _dev.empty_c64((self.m_per_frame, self.nx), self.device)
        p1 = _dev.empty_c64((self.m_per_frame, self.ny), self.device)
        _native.call("csr_plan_get_factors", self._plan, frame, p0.data_ptr(),
                     p1.data_ptr(), _dev.stream_ptr(self.device))
        return DftFactors(p0.cpu().numpy(), p1.cpu().numpy())

    # -- operator application (operators.py:185-203) -------------------------
    def forward(self, image):
        """Encode an image into per-coil k-space samples."""
        x = _dev.as_c64(image, self.image_shape, "image", self.device)
        out = _dev.empty_c64((self.n_samples, self.n_coils), self.device)
        _native.call("csr_forward", self._plan, x.data_ptr(), out.data_ptr(),
                     _dev.stream_ptr(self.device))
        return _dev.out_like(out, image)

    def adjoint(self, data):
        """Conjugate transpose, no normalisation."""
        y = _dev.as_c64(data, (self.n_samples, self.n_coils), "data", self.device)
        out = _dev.empty_c64(self.image_shape, self.device)
        _native.call("csr_adjoint", self._plan, y.data_ptr(), out.data_ptr(),
                     _dev.stream_ptr(self.device))
        return _dev.out_like(out, data)

    def adjoint_chunks(self, data, data_bound=None):
        """Per-chunk adjoint partials (n_chunks, nx, ny), unsummed
        (ChunkedDftOperator.adjoint, operators.py:254-265).

        data_bound: a bound on max(|Re|, |Im|) of the data of ALL workers
        (e.g. an allreduce-max of the workers' maxima).  With it, every
        worker's fp16 operand scale is the same power of two and each chunk
        partial is bit-identical whichever worker computes it; without it,
        the scale follows this worker's own data."""
        if self.n_frames != 1:
            raise ValueError("chunk partials are defined for static (single-frame) plans")
        y = _dev.as_c64(data, (self.n_samples, self.n_coils), "data", self.device)
        out = _dev.empty_c64((self.info()["split_k"], self.nx, self.ny), self.device)
        if data_bound is None:
            _native.call("csr_adjoint_chunks", self._plan, y.data_ptr(), out.data_ptr(),
                         _dev.stream_ptr(self.device))
        else:
            _native.call("csr_adjoint_chunks_bound", self._plan, y.data_ptr(), out.data_ptr(),
                         float(data_bound), _dev.stream_ptr(self.device))
        return _dev.out_like(out, data)

    def normal(self, x, beta=0.0):
        """F^H F x + (beta/2) Theta^H Theta x on this operator's shard."""
        t = _dev.as_c64(x, self.image_shape, "image", self.device)
        out = _dev.empty_c64(self.image_shape, self.device)
        _native.call("csr_normal", self._plan, t.data_ptr(), out.data_ptr(),
                     float(beta), _dev.stream_ptr(self.device))
        return _dev.out_like(out, x)


def sample_chunking(grid, n_coils, n_samples):
    """(chunk_samples, n_chunks) of the global sample-chunk grid of a static
    problem: the k ranges of the adjoint's per-chunk partials, a multiple of
    128 samples (csr_sample_chunking).  Plays the role of the reference's
    default_chunk_size (sharding.py:66-73) for order-stable plans."""
    chunk, n = ctypes.c_int64(), ctypes.c_int32()
    _native.call("csr_sample_chunking", grid.nx, grid.ny, int(n_coils), int(n_samples),
                 ctypes.byref(chunk), ctypes.byref(n))
    return chunk.value, n.value


class ChunkedDftOperator:
    """One worker's shard as a run of fixed global sample chunks
    (operators.py:206-272).  The reference builds one DftOperator per chunk;
    here one device plan covers the worker's contiguous chunk run and
    computes each chunk's forward rows and adjoint partial exactly as a plan
    of the whole problem would (``DftOperator.build(chunk_grid=...)``).
    forward concatenates the chunks' rows; adjoint returns the per-chunk
    partial images stacked (n_chunks, nx, ny), unsummed, for an
    order-stable reduction keyed by chunk id (``ordered_chunk_sum``)."""

    def __init__(self, op, chunk_ids):
        self.op = op
        self.chunk_ids = tuple(chunk_ids)
        self.mode = op.mode
        if len(self.chunk_ids) != op.info()["split_k"]:
            raise ValueError(f"{len(self.chunk_ids)} chunk ids for a plan of "
                             f"{op.info()['split_k']} chunks")

    @classmethod
    def build(cls, coords, grid, sens, chunk_ranges, chunk_ids, mode="auto",
              precision="single", memory_budget=DEFAULT_MEMORY_BUDGET, chunk_size=None,
              n_total=None, device=None):
        """Chunks are absolute sample ranges of coords (consecutive).  The
        chunk grid defaults to ``sample_chunking`` of the whole coords."""
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
        coords = sample_coords(coords)
        n_total = coords.shape[0] if n_total is None else n_total
        maps = _maps_of(sens)
        if chunk_size is None:
            chunk_size, _ = sample_chunking(grid, maps.shape[0], n_total)
        ranges = [tuple(r) for r in chunk_ranges]
        if not ranges:
            raise ValueError("chunked operator needs at least one chunk")
        for (a, b), (c, _) in zip(ranges, ranges[1:]):
            if b != c:
                raise ValueError("chunk ranges must be consecutive")
        for i, (a, b) in zip(chunk_ids, ranges):
            if a != i * chunk_size or b != min((i + 1) * chunk_size, n_total):
                raise ValueError(f"chunk {i} range {(a, b)} is not on the grid of "
                                 f"{chunk_size}-sample chunks")
        start, stop = ranges[0][0], ranges[-1][1]
        op = DftOperator.build(coords[start:stop], grid, sens, mode=mode, precision=precision,
                               memory_budget=memory_budget, device=device,
                               chunk_grid=(chunk_size, n_total))
        return cls(op, chunk_ids)

    @property
    def n_samples(self):
        return self.op.n_samples

    @property
    def n_coils(self):
        return self.op.n_coils

    @property
    def dtype(self):
        return self.op.dtype

    def forward(self, image):
        return self.op.forward(image)

    def adjoint(self, data, data_bound=None):
        """Chunk partials; pass the same data_bound on every worker for
        partials that are bitwise independent of the worker split."""
        return self.op.adjoint_chunks(data, data_bound)


def build_factors(trajectory, grid, precision="single", device=None):
    """Device-generated phase factors (operators.py:72-82)."""
    validate_precision(precision)
    coords = sample_coords(trajectory)
    if coords.shape[0] == 0:
        raise ValueError("trajectory has no samples")
    ones = np.ones((1, grid.nx, grid.ny), np.complex64)
    op = DftOperator.build(coords, grid, ones, mode="separable", device=device)
    return op.factors(0)
