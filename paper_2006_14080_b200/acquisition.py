"""Input containers, field-compatible with csrecon.acquisition
(acquisition.py:15-122) so reference objects and these are interchangeable
(the solver only reads ``.data``, ``.trajectory.coords``, ``.maps``).

``KSpaceDataset.n_frames`` (default 1) marks a 2-D+time acquisition whose
rows are T equal consecutive frames (extension; the reference is static).
"""

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ImageGrid:
    """nx-by-ny grid, pixel n = x*ny + y at r = (x - nx//2, y - ny//2)
    (acquisition.py:15-43)."""

    nx: int
    ny: int

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError(f"grid dims must be >= 1, got {self.nx}x{self.ny}")

    @property
    def n_pixels(self):
        return self.nx * self.ny

    @property
    def shape(self):
        return (self.nx, self.ny)

    def coords(self):
        rx = np.arange(self.nx, dtype=np.float64) - self.nx // 2
        ry = np.arange(self.ny, dtype=np.float64) - self.ny // 2
        return rx, ry


@dataclass
class Trajectory:
    """Sample locations in cycles/pixel, every component in [-0.5, 0.5)
    (acquisition.py:46-73)."""

    coords: np.ndarray
    n_readouts: int
    n_samples_per_readout: int

    def __post_init__(self):
        c = np.asarray(self.coords, dtype=np.float64)
        if c.ndim != 2 or c.shape[1] != 2:
            raise ValueError(f"coords must have shape (n_k, 2), got {c.shape}")
        if c.shape[0] != self.n_readouts * self.n_samples_per_readout:
            raise ValueError(
                f"coords rows {c.shape[0]} != n_readouts * n_samples_per_readout "
                f"= {self.n_readouts * self.n_samples_per_readout}")
        if c.size and (c.min() < -0.5 or c.max() >= 0.5):
            raise ValueError("trajectory coordinates must lie in [-0.5, 0.5)")
        self.coords = c

    @property
    def n_samples(self):
        return self.coords.shape[0]


@dataclass
class SensitivityMaps:
    """(n_coils, nx, ny) complex coil maps (acquisition.py:76-96)."""

    maps: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.maps)
        if m.ndim != 3:
            raise ValueError(f"maps must have shape (n_coils, nx, ny), got {m.shape}")
        if not np.iscomplexobj(m):
            m = m.astype(np.complex128)
        self.maps = m

    @property
    def n_coils(self):
        return self.maps.shape[0]

    @property
    def grid(self):
        return ImageGrid(self.maps.shape[1], self.maps.shape[2])


@dataclass
class KSpaceDataset:
    """(n_k, n_coils) samples with their trajectory (acquisition.py:99-122)."""

    data: np.ndarray
    trajectory: Trajectory
    n_frames: int = 1

    def __post_init__(self):
        d = np.asarray(self.data)
        if d.ndim != 2:
            raise ValueError(f"data must have shape (n_k, n_coils), got {d.shape}")
        if d.shape[0] != self.trajectory.n_samples:
            raise ValueError(f"data rows {d.shape[0]} != trajectory samples "
                             f"{self.trajectory.n_samples}")
        if self.n_frames < 1 or d.shape[0] % self.n_frames:
            raise ValueError("rows must split evenly into n_frames frames")
        self.data = d

    @property
    def n_coils(self):
        return self.data.shape[1]

    @property
    def n_samples(self):
        return self.data.shape[0]


def sample_coords(trajectory):
    """Coordinate rows of a Trajectory or a plain (n, 2) array
    (operators.py:62-69)."""
    coords = getattr(trajectory, "coords", None)
    if coords is None:
        coords = np.asarray(trajectory, dtype=np.float64)
        if coords.ndim != 2 or coords.shape[1] != 2:
            raise ValueError(f"coords must have shape (n, 2), got {coords.shape}")
    return np.asarray(coords, dtype=np.float64)


def simulate_kspace(image, sens, trajectory, n_frames=1, device=None):
    """Direct multi-coil encoding in double precision on the GPU
    (acquisition.py:233-257): d[k, c] = sum_n s_c[n] image[n] exp(-2 pi i
    k_k . r_n), pixels on the centred integer grid, no normalisation.  For
    2-D+t pass image (T, nx, ny) and a trajectory of T*M rows (frame-major).
    Returns a KSpaceDataset with complex128 samples."""
    from . import _dev, _native
    maps = np.asarray(getattr(sens, "maps", sens))
    img = np.asarray(image)
    frames = img.reshape((-1,) + img.shape[-2:]) if img.ndim == 3 else img[None]
    if frames.shape[1:] != maps.shape[1:]:
        raise ValueError(f"image shape {img.shape} != sensitivity grid {maps.shape[1:]}")
    T = frames.shape[0]
    if img.ndim == 3 and T != n_frames:
        n_frames = T
    coords = sample_coords(trajectory)
    if coords.shape[0] % T:
        raise ValueError("trajectory rows must split evenly into the image frames")
    M = coords.shape[0] // T
    dev = device if device is not None else _dev.device_of()
    torch = _dev.torch
    c = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
    s = torch.from_numpy(np.ascontiguousarray(maps.astype(np.complex128))).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(frames.astype(np.complex128))).to(dev)
    out = torch.empty((T * M, maps.shape[0]), dtype=torch.complex128, device=dev)
    _native.call("csr_simulate_kspace", maps.shape[1], maps.shape[2], T, maps.shape[0], M,
                 c.data_ptr(), s.data_ptr(), x.data_ptr(), out.data_ptr(),
                 _dev.stream_ptr(dev))
    data = out.cpu().numpy()
    traj = trajectory if isinstance(trajectory, Trajectory) else \
        Trajectory(coords, coords.shape[0], 1)
    return KSpaceDataset(data, traj, n_frames=T)
