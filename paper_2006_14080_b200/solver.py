"""ADMM + CG reconstruction on the B200 (mirror of csrecon/solver.py).

``admm_reconstruct`` runs the whole solve on the device through
``csr_admm_run``: the ADMM iteration (admm_step, solver.py:163-194) with its
zero-start CG (cg_solve, solver.py:87-125) is one fixed kernel sequence with
device-resident scalars, captured once as a CUDA graph and replayed; the
loop guards (tau > atol^2, alpha > rtol^2) predicate the kernels on the
device, so semantics (early stops, iteration records, divergence errors)
match the reference without host round trips.

``cg_solve``, ``normal_operator``, ``build_rhs``, ``admm_step`` and
``objective`` are the reference's composable building blocks, evaluated
with the same device kernels (used by tests and by callers that compose
their own loops).
"""

import ctypes
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _native
from .acquisition import ImageGrid
from .errors import CgDivergenceError, ShapeMismatchError
from .operators import DEFAULT_MEMORY_BUDGET, DftOperator
from .sharding import (CommStats, NcclComm, coil_shard_plan, dist_world, make_shard_plan,
                       sample_shard_plan)
from .tensor import axpy, hermitian_dot, norm2_squared, validate_precision
from .transform import soft_threshold, theta, theta_adjoint

__all__ = ["ReconParams", "AdmmState", "CgOutcome", "CgDivergenceError",
           "cg_solve", "normal_operator", "build_rhs", "relative_change_sq",
           "should_continue", "admm_step", "objective", "RunReport",
           "admm_reconstruct", "adjoint_reconstruct"]


@dataclass
class ReconParams:
    """Solver knobs (solver.py:34-61); lam_t weights the temporal
    differences of 2-D+t problems (defaults to lam)."""

    lam: float = 1e-7
    beta: float = 1.0
    admm_rtol: float = 1e-4
    admm_max_iters: int = 5
    cg_atol: float = 1e-6
    cg_max_iters: int = 20
    lam_t: float = None

    def __post_init__(self):
        if self.lam <= 0 or self.beta <= 0:
            raise ValueError("lam and beta must be > 0")
        if self.admm_rtol <= 0 or self.cg_atol <= 0:
            raise ValueError("admm_rtol and cg_atol must be > 0")
        if self.admm_max_iters < 1 or self.cg_max_iters < 1:
            raise ValueError("iteration caps must be >= 1")
        if self.lam_t is not None and self.lam_t <= 0:
            raise ValueError("lam_t must be > 0")

    def to_dict(self):
        d = {"lam": self.lam, "beta": self.beta, "admm_rtol": self.admm_rtol,
             "admm_max_iters": self.admm_max_iters, "cg_atol": self.cg_atol,
             "cg_max_iters": self.cg_max_iters}
        if self.lam_t is not None:
            d["lam_t"] = self.lam_t
        return d

    def native(self):
        return _native.AdmmParams(
            lam=self.lam, lam_t=self.lam_t if self.lam_t is not None else 0.0,
            beta=self.beta, admm_rtol=self.admm_rtol, cg_atol=self.cg_atol,
            admm_max_iters=self.admm_max_iters, cg_max_iters=self.cg_max_iters)


@dataclass
class AdmmState:
    """Image, transform variable, scaled dual (solver.py:64-72)."""
    rho: object
    mu: object
    eta: object
    iteration: int = 0
    alpha: float = 1.0


@dataclass
class CgOutcome:
    solution: object
    iterations: int
    final_residual_sq: float
    residual_history: list = field(default_factory=list)


def _no_comm(arr):
    return arr


def _to_dev(v, dev):
    return _dev.as_c64(v, tuple(v.shape), "vector", dev)


def cg_solve(apply_a, b, x0=None, atol=1e-6, max_iters=20):
    """Conjugate gradients on A x = b (solver.py:87-125), device vectors.

    apply_a is called with vectors of b's kind (numpy in -> numpy,
    CUDA tensor in -> tensor)."""
    if max_iters < 0:
        raise ValueError("max_iters must be >= 0")
    dev = _dev.device_of(b)
    tb = _to_dev(b, dev)

    def A(v):
        return _to_dev(apply_a(_dev.out_like(v, b)), dev)

    if x0 is None:
        x = _dev.torch.zeros_like(tb)
        r = tb.clone()
    else:
        x = _to_dev(x0, dev).clone()
        r = axpy(-1.0, A(x), tb)
    d = r.clone()
    tau = float(norm2_squared(r))
    if not np.isfinite(tau):
        raise CgDivergenceError("initial residual is non-finite")
    history = [tau]
    threshold = atol * atol
    iterations = 0
    while iterations < max_iters and tau > threshold:
        ad = A(d)
        alpha = tau / hermitian_dot(d, ad)
        x = axpy(alpha, d, x)
        r = axpy(-alpha, ad, r)
        tau_next = float(norm2_squared(r))
        if not np.isfinite(tau_next):
            raise CgDivergenceError(
                f"residual became non-finite at CG step {iterations + 1}")
        d = axpy(tau_next / tau, d, r)
        tau = tau_next
        history.append(tau)
        iterations += 1
    return CgOutcome(_dev.out_like(x, b), iterations, tau, history)


def normal_operator(x, op, beta, allreduce=_no_comm):
    """A x = allreduce(F^H F x) + (beta/2) Theta^H Theta x (solver.py:128-139)."""
    partial = op.adjoint(op.forward(x))
    total = allreduce(partial)
    if beta == 0:
        return total
    return axpy(beta / 2, theta_adjoint(theta(x)), total)


def build_rhs(fhd, mu, eta, beta):
    """b = F^H d + (beta/2) Theta^H (mu - eta) (solver.py:142-146)."""
    if tuple(mu.shape) != tuple(eta.shape):
        raise ShapeMismatchError(f"mu shape {tuple(mu.shape)} != eta shape "
                                 f"{tuple(eta.shape)}")
    return axpy(beta / 2, theta_adjoint(axpy(-1.0, eta, mu)), fhd)


def relative_change_sq(new, old):
    """solver.py:149-155."""
    num = float(norm2_squared(axpy(-1.0, old, new)))
    den = float(norm2_squared(old))
    if den > 0:
        return num / den
    return 0.0 if num == 0 else float("inf")


def should_continue(iteration, alpha, params):
    """solver.py:158-160."""
    return iteration < params.admm_max_iters and alpha > params.admm_rtol ** 2


def _shrink(v, params):
    t_s = params.lam / params.beta
    if v.shape[0] == 2:
        return soft_threshold(v, t_s)
    t_t = (params.lam_t if params.lam_t is not None else params.lam) / params.beta
    dev = _dev.device_of(v)
    tv = _to_dev(v, dev)
    out = _dev.torch.empty_like(tv)
    out[:2] = soft_threshold(tv[:2].contiguous(), t_s)
    out[2] = soft_threshold(tv[2].contiguous(), t_t)
    return _dev.out_like(out, v)


def admm_step(state, fhd, params, op, allreduce=_no_comm):
    """One outer iteration (solver.py:163-194), composed from device ops."""
    mu_next = _shrink(axpy(1.0, state.eta, theta(state.rho)), params)
    rhs = build_rhs(fhd, mu_next, state.eta, params.beta)
    cg = cg_solve(lambda v: normal_operator(v, op, params.beta, allreduce), rhs,
                  None, params.cg_atol, params.cg_max_iters)
    rho_next = cg.solution
    eta_next = axpy(1.0, state.eta, axpy(-1.0, mu_next, theta(rho_next)))
    nxt = AdmmState(rho=rho_next, mu=mu_next, eta=eta_next,
                    iteration=state.iteration + 1,
                    alpha=relative_change_sq(rho_next, state.rho))
    return nxt, cg


def _abs_sum(z, dev):
    tz = _to_dev(z, dev)
    out = _dev.torch.empty(1, dtype=_dev.torch.float64, device=dev)
    _native.call("csr_abs_sum", tz.data_ptr(), tz.numel(), out.data_ptr(),
                 _dev.stream_ptr(dev))
    return float(out.item())


def objective(rho, data, op, lam, lam_t=None):
    """||F rho - d||^2 + lam*sum|Theta_s rho| (+ lam_t*sum|Theta_t rho|)
    (solver.py:197-204)."""
    if tuple(data.shape) != (op.n_samples, op.n_coils):
        raise ShapeMismatchError(f"data shape {tuple(data.shape)} does not match "
                                 f"operator ({op.n_samples}, {op.n_coils})")
    dev = op.device
    resid = axpy(-1.0, _to_dev(data, dev), _to_dev(op.forward(_to_dev(rho, dev)), dev))
    th = _to_dev(theta(_to_dev(rho, dev)), dev)
    reg = lam * _abs_sum(th[:2].contiguous(), dev)
    if th.shape[0] == 3:
        reg += (lam if lam_t is None else lam_t) * _abs_sum(th[2].contiguous(), dev)
    return float(norm2_squared(resid)) + reg


@dataclass
class RunReport:
    """Everything observable about one run (solver.py:207-240)."""

    method: str
    precision: str
    n_workers: int
    op_mode: str
    grid: tuple
    n_kspace_samples: int
    n_coils: int
    params: dict
    iterations: list
    objective_initial: float = None
    comm: dict = field(default_factory=dict)
    timing: dict = field(default_factory=dict)
    backend: str = ""

    def to_dict(self):
        return {"method": self.method, "precision": self.precision,
                "n_workers": self.n_workers, "op_mode": self.op_mode,
                "grid": list(self.grid), "n_kspace_samples": self.n_kspace_samples,
                "n_coils": self.n_coils, "params": self.params,
                "iterations": self.iterations, "objective_initial": self.objective_initial,
                "comm": self.comm, "timing": self.timing, "backend": self.backend}


def _check_inputs(dataset, sens):
    maps = getattr(sens, "maps", sens)
    if dataset.data.shape[1] != maps.shape[0]:
        raise ShapeMismatchError(
            f"dataset has {dataset.data.shape[1]} coils, maps have {maps.shape[0]}")


def _frames(dataset):
    return int(getattr(dataset, "n_frames", 1))


@dataclass(frozen=True)
class ShardSpec:
    """Which part of the problem one rank owns: ``coil``
    sharding splits the coils (F^H F is a sum over coils, one image
    allreduce per CG iteration), ``frame`` sharding splits the frames of a
    2-D+t problem (F^H F is block diagonal; temporal differences exchange
    one halo frame with each ring neighbour, CG scalars are allreduced),
    ``sample`` sharding is the reference's order-stable split of a static
    problem into runs of whole sample chunks (chunk partials all-gathered
    and folded in chunk order: bitwise the same image for every world size,
    sharding.py:173-208), ``split`` the reference's plain sample split
    (order_stable=False: one image allreduce per CG iteration, like coils)."""
    mode: str
    frames: tuple
    coils: tuple
    samples: tuple = None      # sample mode: this rank's [start, stop)
    chunk_grid: tuple = None   # sample mode: (chunk_samples, total_samples)
    chunk_ids: tuple = None    # sample mode: this rank's global chunk ids


#: coils per rank below which coil sharding wastes tensor work (the
#: operator pads a plan's coils to >= 4, tc_plan_build)
MIN_COILS_PER_RANK = 4


def plan_shard(n_frames, n_coils, rank, world, shard="auto", grid=None, n_samples=None):
    """auto: frames for 2-D+t (world <= frames); coils for static problems
    with >= 4 coils per rank; otherwise the plain sample split."""
    if shard not in ("auto", "coil", "frame", "sample", "split"):
        raise ValueError(f"shard must be auto, coil, frame, sample or split, got {shard!r}")
    if shard == "auto":
        if n_frames > 1 and world > 1 and n_frames >= world:
            shard = "frame"
        elif (world > 1 and n_frames == 1 and n_coils < MIN_COILS_PER_RANK * world
              and n_samples is not None and n_samples >= world):
            shard = "split"
        else:
            shard = "coil"
    if shard == "split":
        if n_frames != 1:
            raise ValueError("the sample split is defined for static problems")
        if n_samples is None:
            raise ValueError("sample sharding needs the sample count")
        return ShardSpec("split", (0, 1), (0, n_coils),
                         make_shard_plan(n_samples, world).bounds[rank])
    if shard == "frame":
        return ShardSpec("frame", make_shard_plan(n_frames, world).bounds[rank],
                         (0, n_coils))
    if shard == "sample":
        if n_frames != 1:
            raise ValueError("order-stable sample sharding is defined for static problems")
        if grid is None or n_samples is None:
            raise ValueError("sample sharding needs the image grid and the sample count")
        plan = sample_shard_plan(grid, n_coils, n_samples, world)
        ids, _ = plan.worker_chunks(rank)
        return ShardSpec("sample", (0, 1), (0, n_coils), plan.bounds[rank],
                         (plan.chunk_size, n_samples), ids)
    return ShardSpec("coil", (0, n_frames), coil_shard_plan(n_coils, world).bounds[rank])


def shard_inputs(coords, data, maps, n_frames, spec):
    """This rank's (coords, data, maps) rows/columns for a ShardSpec."""
    if spec.mode in ("sample", "split"):
        s0, s1 = spec.samples
        return coords[s0:s1], np.asarray(data)[s0:s1], np.asarray(maps)
    m = coords.shape[0] // n_frames
    (f0, f1), (c0, c1) = spec.frames, spec.coils
    return (coords[f0 * m:f1 * m], np.asarray(data)[f0 * m:f1 * m, c0:c1],
            np.asarray(maps)[c0:c1])


COLLECTIVES = ("auto", "nccl")


def resolve_shard(shard, order_stable, n_frames, world):
    """The reference's default ``order_stable=True`` makes the reduced image
    bitwise independent of n_workers (solver.py:281-297).  For a static
    problem on several ranks, shard="auto" therefore picks the order-stable
    sample split; an explicit coil / plain-sample split is reduced by an
    NCCL sum whose bits depend on the rank count, which is reported."""
    if shard == "auto" and order_stable and n_frames == 1 and world > 1:
        return "sample"
    if order_stable and world > 1 and shard in ("coil", "split"):
        warnings.warn(f"shard={shard!r} reduces partial images with an NCCL sum: the image "
                      "is not bitwise independent of n_workers (order_stable=True asks for "
                      "that; use shard='sample' or pass order_stable=False)", stacklevel=3)
    return shard


class _Shard:
    """This rank's operator, data and communicator (one GPU per rank).

    collective="nccl" attaches an NCCL communicator even at one rank, so the
    shard mode's collective path (allreduce, halo exchange, scalar sums,
    all-gather) runs on a single GPU; "auto" attaches one when world > 1."""

    def __init__(self, dataset, sens, n_workers, op_mode, device, shard="auto",
                 collective="auto"):
        if collective not in COLLECTIVES:
            raise ValueError(f"collective must be one of {COLLECTIVES}, got {collective!r}")
        maps = np.asarray(getattr(sens, "maps", sens))
        rank, world = dist_world()
        if n_workers != world:
            raise ValueError(f"n_workers={n_workers} but torch.distributed world size is "
                             f"{world}: launch one process per GPU (torchrun)")
        T = _frames(dataset)
        self.rank, self.world, self.n_frames = rank, world, T
        grid = ImageGrid(maps.shape[1], maps.shape[2])
        coords = np.asarray(dataset.trajectory.coords, dtype=np.float64)
        self.spec = plan_shard(T, maps.shape[0], rank, world, shard, grid, coords.shape[0])
        lc, ld, lm = shard_inputs(coords, dataset.data, maps, T, self.spec)
        f0, f1 = self.spec.frames
        self.op = DftOperator.build(lc, grid, lm, mode=op_mode, n_frames=f1 - f0,
                                    device=device, frame_shard=self.spec.mode == "frame",
                                    chunk_grid=self.spec.chunk_grid)
        self.data = _dev.torch.from_numpy(
            np.ascontiguousarray(ld.astype(np.complex64))).to(self.op.device)
        self.comm = None
        if world > 1 or collective == "nccl":
            self.comm = NcclComm(rank, world, self.op.device.index)
            _native.call("csr_plan_set_comm", self.op.plan, self.comm.handle)

    def image_shape(self):
        if self.n_frames == 1:
            return (self.op.nx, self.op.ny)
        return (self.n_frames, self.op.nx, self.op.ny)

    def gather(self, local):
        """Full image on every rank (frame sharding); identity otherwise."""
        if self.spec.mode != "frame" or self.world == 1:
            return local.reshape(self.image_shape())
        import torch.distributed as dist
        parts = [None] * self.world
        dist.all_gather_object(parts, local)
        return np.concatenate(parts, axis=0).reshape(self.image_shape())


def admm_reconstruct(dataset, sens, params=None, n_workers=1, precision="single",
                     op_mode="auto", memory_budget=DEFAULT_MEMORY_BUDGET,
                     compute_objectives=True, order_stable=True,
                     barrier_timeout=600.0, device=None, return_device=False,
                     shard="auto", collective="auto"):
    """Sharded ADMM reconstruction (solver.py:274-360). Returns (image, RunReport).

    n_workers must equal the torch.distributed world size (one process per
    GPU).  shard="auto" splits coils across ranks (static; the F^H F partials
    are summed by one NCCL allreduce per CG iteration) or frames (2-D+t).
    With few coils per rank (< 4: the operator pads coils to 4) the static
    default is the plain sample split ("split", one image allreduce).
    shard="sample" is the reference's order-stable sample split: every rank
    owns a run of whole global sample chunks, the chunk partials are
    all-gathered and folded in chunk order, and the image is bitwise the same
    for every n_workers (order_stable, solver.py:281-297); it is what
    shard="auto" means for a static problem on several ranks while
    order_stable=True (the reference's default).  Objectives are evaluated
    after the solve from per-iteration device snapshots and are not timed.
    collective="nccl" runs the shard mode's NCCL collectives even on one
    rank (see _Shard).

    precision: "single" (complex64) is the only arithmetic here; the
    reference's default "double" raises.
    """
    params = ReconParams() if params is None else params
    validate_precision(precision)
    _check_inputs(dataset, sens)
    t0 = time.perf_counter()
    shard = resolve_shard(shard, order_stable, _frames(dataset), dist_world()[1])
    sh = _Shard(dataset, sens, n_workers, op_mode, device, shard, collective)
    op, dev = sh.op, sh.op.device
    n_it = params.admm_max_iters
    rho = _dev.empty_c64(op.image_shape, dev)
    snaps = _dev.empty_c64((n_it + 1,) + op.image_shape, dev) if compute_objectives else None
    log = (_native.IterLog * n_it)()
    stats = _native.RunStats()
    t_build = time.perf_counter() - t0
    rc = _native.load().csr_admm_run(
        op.plan, ctypes.byref(params.native()), sh.data.data_ptr(), rho.data_ptr(),
        log, ctypes.byref(stats), _dev.stream_ptr(dev),
        snaps.data_ptr() if snaps is not None else None)
    _native.check(rc)
    records = [{"iteration": log[i].iteration, "alpha": log[i].alpha,
                "cg_iterations": log[i].cg_iterations,
                "cg_final_residual_sq": log[i].cg_final_residual_sq}
               for i in range(stats.n_iterations)]
    cs = CommStats()
    if sh.comm is not None and sh.spec.mode in ("coil", "sample", "split"):
        cs.record("setup", op.nx * op.ny * op.n_frames, calls=2)
        cs.record("solve", op.nx * op.ny * op.n_frames,
                  calls=stats.allreduce_calls - 2)
    report = RunReport(
        method="admm", precision=precision, n_workers=n_workers, op_mode=op.mode,
        grid=(op.nx, op.ny), n_kspace_samples=dataset.data.shape[0],
        n_coils=dataset.data.shape[1], params=params.to_dict(), iterations=records,
        comm=cs.snapshot(),
        timing={"setup_seconds": t_build + stats.setup_ms / 1e3,
                "solve_seconds": stats.solve_ms / 1e3,
                "total_seconds": time.perf_counter() - t0,
                "graph": bool(stats.graph_used),
                "kernels_per_iteration": stats.kernels_per_iter},
        backend="csrecon_b200/" + op.info()["gemm_path"])
    report.timing["shard"] = sh.spec.mode
    if compute_objectives and sh.spec.mode == "frame" and sh.world > 1:
        compute_objectives = False  # the local snapshots hold only this rank's frames
    if compute_objectives:
        full = op if sh.world == 1 else DftOperator.build(
            dataset.trajectory, ImageGrid(op.nx, op.ny), np.asarray(getattr(sens, "maps", sens)),
            n_frames=op.n_frames, device=dev)
        data_full = _dev.torch.from_numpy(np.ascontiguousarray(
            np.asarray(dataset.data).astype(np.complex64))).to(dev)
        lam_t = params.lam_t
        vals = [objective(snaps[i], data_full, full, params.lam, lam_t)
                for i in range(stats.n_iterations + 1)]
        report.objective_initial = vals[0]
        for rec, val in zip(records, vals[1:]):
            rec["objective"] = val
    if return_device and (sh.spec.mode in ("coil", "sample", "split") or sh.world == 1):
        return rho.reshape(sh.image_shape()), report
    return sh.gather(rho.cpu().numpy()), report


def adjoint_reconstruct(dataset, sens, n_workers=1, precision="single",
                        op_mode="auto", memory_budget=DEFAULT_MEMORY_BUDGET,
                        order_stable=True, barrier_timeout=600.0, device=None,
                        return_device=False, shard="auto", collective="auto"):
    """Unregularised adjoint image F^H d (solver.py:363-406)."""
    validate_precision(precision)
    _check_inputs(dataset, sens)
    t0 = time.perf_counter()
    shard = resolve_shard(shard, order_stable, _frames(dataset), dist_world()[1])
    sh = _Shard(dataset, sens, n_workers, op_mode, device, shard, collective)
    op, dev = sh.op, sh.op.device
    img = _dev.empty_c64(op.image_shape, dev)
    _native.call("csr_adjoint_reconstruct", op.plan, sh.data.data_ptr(), img.data_ptr(),
                 _dev.stream_ptr(dev))
    _dev.torch.cuda.current_stream(dev).synchronize()
    cs = CommStats()
    if sh.comm is not None and sh.spec.mode in ("coil", "sample", "split"):
        cs.record("setup", op.nx * op.ny * op.n_frames)
    report = RunReport(
        method="adjoint", precision=precision, n_workers=n_workers, op_mode=op.mode,
        grid=(op.nx, op.ny), n_kspace_samples=dataset.data.shape[0],
        n_coils=dataset.data.shape[1], params={}, iterations=[], comm=cs.snapshot(),
        timing={"setup_seconds": time.perf_counter() - t0,
                "total_seconds": time.perf_counter() - t0},
        backend="csrecon_b200/" + op.info()["gemm_path"])
    if return_device and (sh.spec.mode in ("coil", "sample", "split") or sh.world == 1):
        return img.reshape(sh.image_shape()), report
    return sh.gather(img.cpu().numpy()), report
