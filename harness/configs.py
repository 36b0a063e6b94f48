"""Seeded synthetic inputs for the five BASELINE.json configurations.

Input synthesis is outside the hot path; this module is
the harness shared by tests, ``bench.py`` and ``__graft_entry__``.  The
generators follow SURVEY.md §8(d) (there is no public dataset: the paper's
scanner phantom is not available, so seeded synthetic inputs with the
BASELINE shapes stand in for it):

* trajectory: golden-angle radial, theta_j = (j*pi*(sqrt5-1)/2) mod pi with j
  the global spoke index (continuing across frames), readout radius
  (t - R/2)/R cycles/pixel, rows readout-major (acquisition.py:46-53);
* phantom: 10 random ellipses on the reference's [-1,1]^2 pixel-centre map
  (acquisition.py:192-193), centres U[-0.6,0.6], semi-axes U[0.05,0.4],
  angle U[0,pi], intensity U[0.1,1], additive; dynamic configs modulate
  intensity and radii by (1 + A sin(2 pi f/P + phi)), P~U[8,32], A~U[0,0.3];
* coils: Gaussian (sigma 0.5) centred on radius 0.8, times exp(i * a smooth
  random quadratic phase), normalised to unit sum of squares;
* noise: complex Gaussian at 1 % of the data RMS, i.e. the reference's
  ``add_noise(ds, snr_db=40)`` formula (acquisition.py:260-270);
* k-space: the f64 encoding model d[k,c] = sum_n s_c[n] rho[n] e^{-2 pi i k.r_n}
  (acquisition.py:233-257), evaluated separably (identical up to rounding).

One ``np.random.default_rng(seed)`` per config, drawn in the fixed order
phantom -> coils -> noise.
"""

from dataclasses import dataclass

import numpy as np

GOLDEN = np.pi * (np.sqrt(5.0) - 1.0) / 2.0

#: BASELINE.json configs (index = position in ``configs``).  CG is fixed at 5
#: and the tolerances at 1e-150 so every run does the same work.
CONFIGS = {
    0: dict(nx=64, ny=64, n_frames=1, n_coils=4, spokes=32, readout=128,
            admm_iters=20, lam=1e-3, lam_t=None, beta=1e-2),
    1: dict(nx=128, ny=128, n_frames=1, n_coils=8, spokes=64, readout=256,
            admm_iters=50, lam=1e-3, lam_t=None, beta=1e-2),
    2: dict(nx=256, ny=256, n_frames=1, n_coils=16, spokes=128, readout=512,
            admm_iters=50, lam=1e-3, lam_t=None, beta=1e-2),
    3: dict(nx=192, ny=192, n_frames=32, n_coils=8, spokes=13, readout=384,
            admm_iters=50, lam=1e-3, lam_t=5e-3, beta=1e-2),
    4: dict(nx=256, ny=256, n_frames=64, n_coils=16, spokes=21, readout=512,
            admm_iters=100, lam=1e-3, lam_t=5e-3, beta=1e-2),
}
CG_ITERS = 5
TOL = 1e-150
SEED_BASE = 20060000


@dataclass
class Problem:
    cfg: int
    nx: int
    ny: int
    n_frames: int
    n_coils: int
    coords: np.ndarray     # (T*M, 2) f64 cycles/pixel
    sens: np.ndarray       # (C, nx, ny) c128
    data: np.ndarray       # (T*M, C) c128
    truth: np.ndarray      # (nx, ny) or (T, nx, ny) c128
    params: dict           # ReconParams kwargs (+ lam_t)

    @property
    def m_per_frame(self):
        return self.coords.shape[0] // self.n_frames


def golden_angle_coords(n_spokes, readout, first_spoke=0):
    j = np.arange(first_spoke, first_spoke + n_spokes, dtype=np.float64)
    phi = np.mod(j * GOLDEN, np.pi)
    r = (np.arange(readout, dtype=np.float64) - readout / 2.0) / readout
    kx = np.cos(phi)[:, None] * r[None, :]
    ky = np.sin(phi)[:, None] * r[None, :]
    return np.stack([kx.ravel(), ky.ravel()], axis=1)


def _pixel_map(nx, ny):
    u = (2 * np.arange(nx, dtype=np.float64) - (nx - 1)) / nx
    v = (2 * np.arange(ny, dtype=np.float64) - (ny - 1)) / ny
    return u[:, None], v[None, :]


def draw_ellipses(rng, n=10):
    e = []
    for _ in range(n):
        x0, y0 = rng.uniform(-0.6, 0.6, size=2)
        a, b = rng.uniform(0.05, 0.4, size=2)
        ang = rng.uniform(0.0, np.pi)
        inten = rng.uniform(0.1, 1.0)
        period = rng.uniform(8.0, 32.0)
        amp = rng.uniform(0.0, 0.3)
        phase = rng.uniform(0.0, 2 * np.pi)
        e.append((x0, y0, a, b, ang, inten, period, amp, phase))
    return e


def render_phantom(ellipses, nx, ny, frame=None):
    uu, vv = _pixel_map(nx, ny)
    img = np.zeros((nx, ny), dtype=np.float64)
    for x0, y0, a, b, ang, inten, period, amp, phase in ellipses:
        m = 1.0 if frame is None else 1.0 + amp * np.sin(2 * np.pi * frame / period + phase)
        ct, st = np.cos(ang), np.sin(ang)
        xr = (uu - x0) * ct + (vv - y0) * st
        yr = -(uu - x0) * st + (vv - y0) * ct
        img += inten * m * ((xr / (a * m)) ** 2 + (yr / (b * m)) ** 2 <= 1.0)
    return img


def gaussian_coils(rng, nx, ny, n_coils, sigma=0.5, radius=0.8):
    uu, vv = _pixel_map(nx, ny)
    maps = np.empty((n_coils, nx, ny), dtype=np.complex128)
    for c in range(n_coils):
        ang = 2 * np.pi * c / n_coils
        cx, cy = radius * np.cos(ang), radius * np.sin(ang)
        mag = np.exp(-((uu - cx) ** 2 + (vv - cy) ** 2) / (2 * sigma ** 2))
        p0 = rng.uniform(0.0, 2 * np.pi)
        p = rng.normal(0.0, 0.5, size=5)
        phase = (p0 + p[0] * uu + p[1] * vv + p[2] * uu * uu
                 + p[3] * uu * vv + p[4] * vv * vv)
        maps[c] = mag * np.exp(1j * phase)
    sos = np.sqrt(np.sum(np.abs(maps) ** 2, axis=0))
    return maps / sos[None]


def encode_f64(image, sens, coords, chunk=4096):
    """f64 multi-coil encoding of one frame, separable evaluation of
    acquisition.py:233-257 (phase angle in f64 as operators.py:50-59)."""
    n_coils, nx, ny = sens.shape
    rx = np.arange(nx, dtype=np.float64) - nx // 2
    ry = np.arange(ny, dtype=np.float64) - ny // 2
    x = (sens * image[None]).reshape(n_coils * nx, ny)
    out = np.empty((coords.shape[0], n_coils), dtype=np.complex128)
    for s in range(0, coords.shape[0], chunk):
        e = min(s + chunk, coords.shape[0])
        p0 = np.exp(-2j * np.pi * np.outer(coords[s:e, 0], rx))
        p1 = np.exp(-2j * np.pi * np.outer(coords[s:e, 1], ry))
        g = (x @ p1.T).reshape(n_coils, nx, e - s)
        out[s:e] = np.einsum("kx,cxk->kc", p0, g)
    return out


def make_problem(cfg, seed=None, encoder=None):
    """Build config ``cfg`` (0-4) with its fixed seed (or ``seed``).
    ``encoder(img, sens, coords)`` replaces the CPU f64 separable encode (the
    GPU f64 simulate_kspace for the large configs; identical to 1e-12)."""
    c = CONFIGS[cfg]
    rng = np.random.default_rng(SEED_BASE + cfg if seed is None else seed)
    nx, ny, T, C = c["nx"], c["ny"], c["n_frames"], c["n_coils"]
    ellipses = draw_ellipses(rng)
    sens = gaussian_coils(rng, nx, ny, C)
    coords, data, truth = [], [], []
    for f in range(T):
        img = render_phantom(ellipses, nx, ny, None if T == 1 else f)
        kc = golden_angle_coords(c["spokes"], c["readout"], f * c["spokes"])
        coords.append(kc)
        data.append((encoder or encode_f64)(img.astype(np.complex128), sens, kc))
        truth.append(img)
    coords = np.concatenate(coords, 0)
    data = np.concatenate(data, 0)
    rms = np.sqrt(np.mean(np.abs(data) ** 2))
    sigma = rms / 10.0 ** (40.0 / 20.0)
    noise = rng.standard_normal(data.shape) + 1j * rng.standard_normal(data.shape)
    data = data + (sigma / np.sqrt(2)) * noise
    truth = np.asarray(truth, dtype=np.complex128)
    if T == 1:
        truth = truth[0]
    params = dict(lam=c["lam"], beta=c["beta"], admm_rtol=TOL,
                  admm_max_iters=c["admm_iters"], cg_atol=TOL,
                  cg_max_iters=CG_ITERS)
    if c["lam_t"] is not None:
        params["lam_t"] = c["lam_t"]
    return Problem(cfg, nx, ny, T, C, coords, sens, data, truth, params)


def data_probe(data):
    """Size-independent fingerprint of a k-space array: v^T d for a fixed
    seeded complex v (one value per coil).  The committed fixtures of the
    large configs store it instead of the data (the GPU f64 encoder used at
    test time reproduces the CPU encode to ~1e-12)."""
    rng = np.random.default_rng(123)
    v = rng.standard_normal(data.shape[0]) + 1j * rng.standard_normal(data.shape[0])
    return v @ data


def array_sha(arr):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def nudft_flops_per_cg(cfg):
    """Algorithmic NUDFT flops per CG iteration, 16*C*M_f*N*T."""
    c = CONFIGS[cfg]
    m = c["spokes"] * c["readout"]
    return 16.0 * c["n_coils"] * m * c["nx"] * c["ny"] * c["n_frames"]
