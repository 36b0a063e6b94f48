"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (needs /root/reference; it never runs on the GPU
box, whose tests only read the committed .npz files):

    python tests/golden/make_golden.py [--big]

The reference is copied to /tmp/refpkg first (it JIT-caches numba code and
must never run in place) and imported from there.  Every
fixture records reference outputs for seeded inputs; ``--big`` adds the
config-1 ADMM run (~1 min on 8 cores) and the truncated (3-iteration)
config 2-4 runs (config 4: ~10 min on 8 cores).
"""

import argparse
import hashlib
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg"
REF_COPY = "/tmp/refpkg"


def import_reference():
    if not os.path.isdir(REF_COPY):
        shutil.copytree(REF_SRC, REF_COPY)
        os.system(f"chmod -R u+w {REF_COPY}")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, os.path.join(REF_COPY, "src"))
    import csrecon  # noqa: F401
    return csrecon


def rc(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def gen_factors(cs):
    from csrecon.acquisition import ImageGrid
    from csrecon.operators import build_factors
    rng = np.random.default_rng(42)
    coords = rng.uniform(-0.5, 0.4999, size=(20, 2))
    grid = ImageGrid(8, 6)
    f64 = build_factors(coords, grid, "double")
    f32 = build_factors(coords, grid, "single")
    save("factors.npz", coords=coords, nx=8, ny=6, p0_f64=f64.phase0,
         p1_f64=f64.phase1, p0_f32=f32.phase0, p1_f32=f32.phase1)


# (nx, ny, coils, samples): edge shapes from test_acceptance.py:79-103
OPERATOR_CASES = [(1, 1, 1, 1), (6, 4, 2, 25), (5, 4, 2, 24), (16, 12, 3, 200),
                  (13, 7, 1, 64), (3, 16, 2, 9), (32, 32, 4, 513),
                  (64, 48, 3, 1000)]


def gen_operators(cs):
    from csrecon.acquisition import ImageGrid, SensitivityMaps
    from csrecon.operators import DftOperator
    rng = np.random.default_rng(2024)
    out = {}
    for i, (nx, ny, nc, m) in enumerate(OPERATOR_CASES):
        coords = rng.uniform(-0.5, 0.4999, size=(m, 2))
        sens = rc(rng, (nc, nx, ny))
        image = rc(rng, (nx, ny))
        y = rc(rng, (m, nc))
        grid = ImageGrid(nx, ny)
        smaps = SensitivityMaps(sens)
        p = f"c{i}_"
        out.update({p + "coords": coords, p + "sens": sens, p + "image": image,
                    p + "y": y})
        for prec, cdt in (("double", np.complex128), ("single", np.complex64)):
            op = DftOperator.build(coords, grid, smaps, mode="separable",
                                   precision=prec)
            out[p + f"fwd_{prec}"] = op.forward(image.astype(cdt))
            out[p + f"adj_{prec}"] = op.adjoint(y.astype(cdt))
        opm = DftOperator.build(coords, grid, smaps, mode="materialized")
        out[p + "fwd_mat"] = opm.forward(image)
        out[p + "adj_mat"] = opm.adjoint(y)
    save("operators.npz", n_cases=len(OPERATOR_CASES),
         shapes=np.array(OPERATOR_CASES), **out)


def gen_transform(cs):
    from csrecon.transform import soft_threshold, theta, theta_adjoint
    rng = np.random.default_rng(31)
    img = rc(rng, (6, 9))
    stack = rc(rng, (2, 6, 9))
    z = rc(rng, (257,))
    out = dict(img=img, stack=stack, z=z, t=0.6)
    for prec, cdt in (("double", np.complex128), ("single", np.complex64)):
        out[f"theta_{prec}"] = theta(img.astype(cdt))
        out[f"theta_adj_{prec}"] = theta_adjoint(stack.astype(cdt))
        out[f"soft_{prec}"] = soft_threshold(z.astype(cdt), 0.6)
    save("transform.npz", **out)


def gen_admm_small(cs):
    from csrecon.acquisition import (birdcage_sensitivities, radial_trajectory,
                                     shepp_logan, simulate_kspace)
    from csrecon.acquisition import ImageGrid
    from csrecon.solver import ReconParams, admm_reconstruct, adjoint_reconstruct
    grid = ImageGrid(16, 12)
    sens = birdcage_sensitivities(grid, 3)
    ds = simulate_kspace(shepp_logan(grid), sens, radial_trajectory(10, 24))
    out = dict(coords=ds.trajectory.coords, sens=sens.maps, data=ds.data)
    runs = {
        "fixed": ReconParams(lam=1e-3, beta=1e-2, admm_rtol=1e-150,
                             admm_max_iters=8, cg_atol=1e-150, cg_max_iters=5),
        "default": ReconParams(),
    }
    for name, params in runs.items():
        for prec in ("double", "single"):
            img, rep = admm_reconstruct(ds, sens, params, precision=prec)
            out[f"{name}_{prec}_image"] = img
            out[f"{name}_{prec}_alpha"] = np.array([r["alpha"] for r in rep.iterations])
            out[f"{name}_{prec}_cg"] = np.array([r["cg_iterations"] for r in rep.iterations])
            out[f"{name}_{prec}_tau"] = np.array(
                [r["cg_final_residual_sq"] for r in rep.iterations])
            out[f"{name}_{prec}_obj"] = np.array(
                [rep.objective_initial] + [r["objective"] for r in rep.iterations])
            out[f"{name}_{prec}_comm_calls"] = rep.comm["allreduce_calls"]
        out[f"{name}_params"] = np.array([params.lam, params.beta, params.admm_rtol,
                                          params.admm_max_iters, params.cg_atol,
                                          params.cg_max_iters])
    adj, _ = adjoint_reconstruct(ds, sens)
    out["adjoint_double"] = adj
    save("admm_small.npz", **out)


def gen_admm_config(cs, cfg):
    sys.path.insert(0, REPO)
    from harness.configs import make_problem
    from csrecon.acquisition import KSpaceDataset, SensitivityMaps, Trajectory
    from csrecon.solver import ReconParams, admm_reconstruct
    prob = make_problem(cfg)
    traj = Trajectory(prob.coords, prob.coords.shape[0] // 1, 1)
    ds = KSpaceDataset(prob.data, traj)
    sens = SensitivityMaps(prob.sens)
    params = ReconParams(**prob.params)
    img, rep = admm_reconstruct(ds, sens, params, n_workers=os.cpu_count(),
                                precision="double", compute_objectives=False)
    save(f"admm_c{cfg}.npz", image=img,
         alpha=np.array([r["alpha"] for r in rep.iterations]),
         tau=np.array([r["cg_final_residual_sq"] for r in rep.iterations]),
         sha_data=sha(prob.data), sha_sens=sha(prob.sens), sha_coords=sha(prob.coords),
         solve_seconds=rep.timing["solve_seconds"], workers=os.cpu_count())


#: truncated ADMM fixtures of the large BASELINE configs:
#: 3 ADMM iterations at CG = 5; frames stored for the 2-D+t configs
TRUNC_ITERS = 3


def trunc_frames(n_frames):
    return sorted({0, n_frames // 2, n_frames - 1})


def data_probe(data):
    """Size-independent fingerprint of a k-space array: v^T d for a fixed
    seeded complex v (C values).  The GPU f64 encoder reproduces the CPU one
    to ~1e-12, so the tests compare probes instead of shipping the data."""
    v = rc(np.random.default_rng(123), data.shape[0])
    return v @ data


def gen_admm_trunc(cs, cfg):
    """Config 2: the reference's own admm_reconstruct (f64).  Configs 3-4
    (2-D+t, no reference path): the f64 restatement in oracle/.  Inputs from
    harness.configs.make_problem (CPU f64 encode)."""
    import time
    sys.path.insert(0, REPO)
    from harness.configs import make_problem
    prob = make_problem(cfg)
    params = dict(prob.params, admm_max_iters=TRUNC_ITERS)
    t0 = time.perf_counter()
    if prob.n_frames == 1:
        from csrecon.acquisition import KSpaceDataset, SensitivityMaps, Trajectory
        from csrecon.solver import ReconParams, admm_reconstruct
        traj = Trajectory(prob.coords, prob.coords.shape[0], 1)
        img, rep = admm_reconstruct(KSpaceDataset(prob.data, traj),
                                    SensitivityMaps(prob.sens), ReconParams(**params),
                                    n_workers=os.cpu_count(), precision="double",
                                    compute_objectives=False)
        recs, source = rep.iterations, "reference csrecon.admm_reconstruct, f64"
        frames = [0]
        img = img[None]
    else:
        from oracle import csrecon_oracle as O
        img, recs = O.admm(prob.data, prob.coords, prob.sens, O.Params(**params),
                           "double", prob.n_frames)
        source = "oracle/csrecon_oracle.admm (2-D+t restatement), f64"
        frames = trunc_frames(prob.n_frames)
        img = img[frames]
    save(f"admm_trunc_c{cfg}.npz", image=img, frames=np.array(frames),
         alpha=np.array([r["alpha"] for r in recs]),
         tau=np.array([r["cg_final_residual_sq"] for r in recs]),
         iters=TRUNC_ITERS, source=source, data_probe=data_probe(prob.data),
         sha_sens=sha(prob.sens), sha_coords=sha(prob.coords), sha_truth=sha(prob.truth),
         seconds=time.perf_counter() - t0, workers=os.cpu_count())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    cs = import_reference()
    jobs = {"factors": gen_factors, "operators": gen_operators,
            "transform": gen_transform, "admm_small": gen_admm_small,
            "c0": lambda c: gen_admm_config(c, 0)}
    if args.big:
        jobs["c1"] = lambda c: gen_admm_config(c, 1)
        for cfg in (2, 3, 4):
            jobs[f"t{cfg}"] = lambda c, cfg=cfg: gen_admm_trunc(c, cfg)
    for name, fn in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        fn(cs)


if __name__ == "__main__":
    main()
