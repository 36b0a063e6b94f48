"""numpy restatement of the csrecon hot path (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py``: this module is the checker for the CUDA path and
the CPU arm of ``bench.py``; the product package never imports it.

Every function names the reference file:line it restates (paths relative to
``/root/reference/pkg/src/csrecon``).  The arithmetic follows the reference's
numpy backend (``kernels.py:61-108``) and solver (``solver.py:87-204``) so
that, in ``precision="double"``, results agree with the reference to
rounding (pinned by ``tests/test_oracle_golden.py`` against fixtures the
reference itself produced).

2-D+time (n_frames > 1) is an extension the reference does not have
(SURVEY.md App. A): per-frame operators built exactly like the static one,
a third circular finite-difference component along time that follows the
spatial convention of ``kernels.py:93-94,196-197``, and a separate threshold
lam_t/beta for that component.  That part is "parity unpinned".
"""

from dataclasses import dataclass, field

import numpy as np

COMPLEX_DTYPES = {"single": np.complex64, "double": np.complex128}
REAL_DTYPES = {"single": np.float32, "double": np.float64}


class OracleDivergence(RuntimeError):
    """Mirror of CgDivergenceError (solver.py:30-31)."""


# ---------------------------------------------------------------------------
# geometry and encoding factors
# ---------------------------------------------------------------------------

def grid_coords(nx, ny):
    """Centred integer pixel coordinates (acquisition.py:39-43)."""
    return (np.arange(nx, dtype=np.float64) - nx // 2,
            np.arange(ny, dtype=np.float64) - ny // 2)


def unit_phase(kr, cdtype):
    """exp(-2j*pi*kr) with the angle in f64, phasor rounded once
    (operators.py:50-59)."""
    ang = (-2 * np.pi) * np.asarray(kr, dtype=np.float64)
    out = np.empty(ang.shape, dtype=np.complex128)
    out.real = np.cos(ang)
    out.imag = np.sin(ang)
    return out.astype(cdtype, copy=False)


def build_factors(coords, nx, ny, precision="double"):
    """P0[k,x] = e^{-2pi i kx_k rx_x}, P1[k,y] likewise (operators.py:72-82)."""
    coords = np.asarray(coords, dtype=np.float64)
    if coords.ndim != 2 or coords.shape[1] != 2:
        raise ValueError(f"coords must have shape (n, 2), got {coords.shape}")
    if coords.shape[0] == 0:
        raise ValueError("trajectory has no samples")
    cdt = COMPLEX_DTYPES[precision]
    rx, ry = grid_coords(nx, ny)
    return (unit_phase(np.outer(coords[:, 0], rx), cdt),
            unit_phase(np.outer(coords[:, 1], ry), cdt))


def forward_sep(p0, p1, sens, image):
    """Separable forward, per coil (kernels.py:71-78):
    out[k,c] = sum_x P0[k,x] * ((s_c*img) @ P1^T)[x,k]."""
    n_coils = sens.shape[0]
    out = np.empty((p0.shape[0], n_coils), dtype=p0.dtype)
    p1_t = np.ascontiguousarray(p1.T)
    for c in range(n_coils):
        g = (sens[c] * image) @ p1_t                     # (nx, M)
        out[:, c] = np.einsum("kx,xk->k", p0, g)
    return out


def adjoint_sep(p0, p1, sens, data):
    """Separable adjoint, no 1/N (kernels.py:81-88):
    out = sum_c conj(s_c) * ((conj(P0) * d_c)^T @ conj(P1))."""
    n_coils, nx, ny = sens.shape
    out = np.zeros((nx, ny), dtype=p0.dtype)
    p0c = np.conj(p0)
    p1c = np.conj(p1)
    for c in range(n_coils):
        wt = (p0c * data[:, c:c + 1]).T                  # (nx, M)
        out += np.conj(sens[c]) * (wt @ p1c)
    return out


def forward_direct(image, sens, coords, chunk=4096):
    """f64 direct-summation forward model (acquisition.py:233-257)."""
    image = np.asarray(image)
    n_coils, nx, ny = sens.shape
    rx, ry = grid_coords(nx, ny)
    r_x = np.repeat(rx, ny)
    r_y = np.tile(ry, nx)
    coil_images = (sens.astype(np.complex128)
                   * image.astype(np.complex128)).reshape(n_coils, -1)
    coords = np.asarray(coords, dtype=np.float64)
    out = np.empty((coords.shape[0], n_coils), dtype=np.complex128)
    for s in range(0, coords.shape[0], chunk):
        e = min(s + chunk, coords.shape[0])
        phase = coords[s:e, 0:1] * r_x[None, :] + coords[s:e, 1:2] * r_y[None, :]
        out[s:e] = np.exp(-2j * np.pi * phase) @ coil_images.T
    return out


class Operator:
    """Multi-coil NUDFT over n_frames frames of m samples each (frames share
    the coil maps).  n_frames == 1 is the reference's DftOperator
    (operators.py:109-203) in separable mode; frame f uses the rows
    [f*m, (f+1)*m) of coords and of the data (readout-major, as the
    reference's Trajectory, acquisition.py:46-53)."""

    def __init__(self, coords, sens, n_frames=1, precision="double"):
        cdt = COMPLEX_DTYPES[precision]
        coords = np.asarray(coords, dtype=np.float64)
        self.sens = np.ascontiguousarray(np.asarray(sens).astype(cdt))
        self.n_coils, self.nx, self.ny = self.sens.shape
        self.n_frames = int(n_frames)
        if coords.shape[0] % self.n_frames:
            raise ValueError("coords rows must split evenly into frames")
        self.m = coords.shape[0] // self.n_frames
        self.factors = [build_factors(coords[f * self.m:(f + 1) * self.m],
                                      self.nx, self.ny, precision)
                        for f in range(self.n_frames)]
        self.dtype = cdt

    @property
    def image_shape(self):
        if self.n_frames == 1:
            return (self.nx, self.ny)
        return (self.n_frames, self.nx, self.ny)

    def forward(self, image):
        img = image.reshape(self.n_frames, self.nx, self.ny)
        return np.concatenate([forward_sep(p0, p1, self.sens, img[f])
                               for f, (p0, p1) in enumerate(self.factors)], 0)

    def adjoint(self, data):
        out = np.stack([adjoint_sep(p0, p1, self.sens,
                                    data[f * self.m:(f + 1) * self.m])
                        for f, (p0, p1) in enumerate(self.factors)])
        return out.reshape(self.image_shape)


# ---------------------------------------------------------------------------
# sparsifying transform (kernels.py:91-108, transform.py:14-42)
# ---------------------------------------------------------------------------

def theta(image):
    """Circular backward differences.  (nx,ny) -> (2,nx,ny)
    (kernels.py:91-95); (T,nx,ny) -> (3,T,nx,ny) with the temporal
    component D_t = rho_f - rho_{f-1} (extension, same convention)."""
    if image.ndim == 2:
        out = np.empty((2,) + image.shape, dtype=image.dtype)
        out[0] = image - np.roll(image, 1, axis=0)
        out[1] = image - np.roll(image, 1, axis=1)
        return out
    out = np.empty((3,) + image.shape, dtype=image.dtype)
    out[0] = image - np.roll(image, 1, axis=1)
    out[1] = image - np.roll(image, 1, axis=2)
    out[2] = image - np.roll(image, 1, axis=0)
    return out


def theta_adjoint(diffs):
    """Exact adjoint of theta (kernels.py:98-101 and its temporal twin)."""
    if diffs.shape[0] == 2:
        d0, d1 = diffs[0], diffs[1]
        return (d0 - np.roll(d0, -1, axis=0)) + (d1 - np.roll(d1, -1, axis=1))
    d0, d1, d2 = diffs[0], diffs[1], diffs[2]
    return ((d0 - np.roll(d0, -1, axis=1)) + (d1 - np.roll(d1, -1, axis=2))
            + (d2 - np.roll(d2, -1, axis=0)))


def soft_threshold(z, threshold):
    """z*(1 - t/|z|) where |z| > t else 0, t cast to the real dtype
    (transform.py:29-42, kernels.py:104-108)."""
    if threshold < 0:
        raise ValueError(f"threshold must be >= 0, got {threshold}")
    t = np.float32(threshold) if z.dtype == np.complex64 else np.float64(threshold)
    mag = np.abs(z)
    safe = np.where(mag > 0, mag, 1)
    return np.where(mag > t, z - z * (t / safe), 0).astype(z.dtype)


def shrink_stack(v, t_s, t_t):
    """Soft threshold of a theta stack: spatial components with t_s, the
    temporal one (dynamic only) with t_t."""
    if v.shape[0] == 2:
        return soft_threshold(v, t_s)
    out = np.empty_like(v)
    out[:2] = soft_threshold(v[:2], t_s)
    out[2] = soft_threshold(v[2], t_t)
    return out


# ---------------------------------------------------------------------------
# vector algebra (tensor.py:44-64)
# ---------------------------------------------------------------------------

def hermitian_dot(a, b):
    return np.vdot(a, b)


def norm2_squared(a):
    return hermitian_dot(a, a).real


def axpy(alpha, x, y):
    return y + x.dtype.type(alpha) * x


# ---------------------------------------------------------------------------
# solver (solver.py:34-204)
# ---------------------------------------------------------------------------

@dataclass
class Params:
    """ReconParams (solver.py:34-61) plus lam_t for the temporal term."""
    lam: float = 1e-7
    beta: float = 1.0
    admm_rtol: float = 1e-4
    admm_max_iters: int = 5
    cg_atol: float = 1e-6
    cg_max_iters: int = 20
    lam_t: float = None


@dataclass
class CgResult:
    solution: np.ndarray
    iterations: int
    final_residual_sq: float
    residual_history: list = field(default_factory=list)


def cg_solve(apply_a, b, atol, max_iters):
    """Zero-start CG (solver.py:87-125)."""
    x = np.zeros_like(b)
    r = b.copy()
    d = r.copy()
    tau = float(norm2_squared(r))
    if not np.isfinite(tau):
        raise OracleDivergence("initial residual is non-finite")
    history = [tau]
    it = 0
    while it < max_iters and tau > atol * atol:
        ad = apply_a(d)
        alpha = tau / hermitian_dot(d, ad)
        x = axpy(alpha, d, x)
        r = axpy(-alpha, ad, r)
        tau_next = float(norm2_squared(r))
        if not np.isfinite(tau_next):
            raise OracleDivergence(f"residual became non-finite at CG step {it + 1}")
        d = axpy(tau_next / tau, d, r)
        tau = tau_next
        history.append(tau)
        it += 1
    return CgResult(x, it, tau, history)


def normal_operator(x, op, beta, allreduce=None):
    """A x = allreduce(F^H F x) + (beta/2) Theta^H Theta x (solver.py:128-139)."""
    partial = op.adjoint(op.forward(x))
    total = partial if allreduce is None else allreduce(partial)
    if beta == 0:
        return total
    return total + (beta / 2) * theta_adjoint(theta(x))


def relative_change_sq(new, old):
    """solver.py:149-155."""
    num = float(norm2_squared(new - old))
    den = float(norm2_squared(old))
    if den > 0:
        return num / den
    return 0.0 if num == 0 else float("inf")


def objective(rho, data, op, lam, lam_t=None):
    """||F rho - d||^2 + lam*|Theta_s rho|_1 (+ lam_t*|Theta_t rho|_1)
    (solver.py:197-204)."""
    resid = op.forward(rho) - data
    th = np.abs(theta(rho))
    reg = lam * float(np.sum(th[:2]))
    if th.shape[0] == 3:
        reg += (lam if lam_t is None else lam_t) * float(np.sum(th[2]))
    return float(norm2_squared(resid)) + reg


def admm(data, coords, sens, params, precision="double", n_frames=1,
         allreduce=None, op=None, snapshots=False):
    """admm_reconstruct's math (solver.py:274-360, admm_step :163-194).

    Returns (image, records[, snapshots]).  allreduce, when given, is the
    cross-worker sum hook applied to F^H d (twice, as solver.py:308-309) and
    to every F^H F x (solver.py:136); op may be a prebuilt Operator (a shard).
    """
    cdt = COMPLEX_DTYPES[precision]
    data = np.asarray(data).astype(cdt)
    if op is None:
        op = Operator(coords, sens, n_frames, precision)
    hook = allreduce if allreduce is not None else (lambda a: a)
    partial = op.adjoint(data)
    rho = hook(partial)
    fhd = hook(partial)
    d_comp = 2 if op.n_frames == 1 else 3
    zeros = np.zeros((d_comp,) + op.image_shape, dtype=cdt)
    mu, eta = zeros, zeros.copy()
    t_s = params.lam / params.beta
    t_t = (params.lam_t if params.lam_t is not None else params.lam) / params.beta
    records, snaps = [], [rho.copy()]
    it, alpha_admm = 0, 1.0
    while it < params.admm_max_iters and alpha_admm > params.admm_rtol ** 2:
        mu_next = shrink_stack(theta(rho) + eta, t_s, t_t)
        rhs = fhd + (params.beta / 2) * theta_adjoint(mu_next - eta)
        cg = cg_solve(lambda v: normal_operator(v, op, params.beta, allreduce),
                      rhs, params.cg_atol, params.cg_max_iters)
        rho_next = cg.solution
        eta = eta + (theta(rho_next) - mu_next)
        alpha_admm = relative_change_sq(rho_next, rho)
        rho, mu = rho_next, mu_next
        it += 1
        records.append({"iteration": it, "alpha": alpha_admm,
                        "cg_iterations": cg.iterations,
                        "cg_final_residual_sq": cg.final_residual_sq})
        snaps.append(rho.copy())
    if snapshots:
        return rho, records, snaps
    return rho, records


def adjoint_image(data, coords, sens, precision="double", n_frames=1):
    """adjoint_reconstruct's math (solver.py:363-406): F^H d."""
    op = Operator(coords, sens, n_frames, precision)
    return op.adjoint(np.asarray(data).astype(COMPLEX_DTYPES[precision]))
