"""Host-side logic that needs no GPU: parameter validation, shard plans,
comm accounting, precision policy, input containers, and that the product
path refuses to run without the CUDA device (no CPU fallback)."""

import numpy as np
import pytest

import paper_2006_14080_b200 as P
from paper_2006_14080_b200.errors import NativeError


def test_recon_params_validation():
    # solver.py:45-51, test_solver.py:148-160
    with pytest.raises(ValueError):
        P.ReconParams(lam=0.0)
    with pytest.raises(ValueError):
        P.ReconParams(beta=-1.0)
    with pytest.raises(ValueError):
        P.ReconParams(admm_rtol=0.0)
    with pytest.raises(ValueError):
        P.ReconParams(admm_max_iters=0)
    with pytest.raises(ValueError):
        P.ReconParams(lam_t=-1.0)
    d = P.ReconParams().to_dict()
    assert d["lam"] == 1e-7 and d["cg_max_iters"] == 20 and "lam_t" not in d
    assert P.ReconParams(lam_t=5e-3).to_dict()["lam_t"] == 5e-3


def test_should_continue_guard_semantics():
    params = P.ReconParams(admm_rtol=1e-4, admm_max_iters=5)
    assert P.should_continue(0, 1.0, params)
    assert not P.should_continue(5, 1.0, params)
    assert not P.should_continue(1, params.admm_rtol ** 2, params)
    assert P.should_continue(1, params.admm_rtol ** 2 * 1.0001, params)


def test_shard_plans():
    # sharding.py:76-113 semantics
    plan = P.make_shard_plan(10, 3)
    assert plan.bounds == ((0, 4), (4, 7), (7, 10))
    plan = P.make_shard_plan(1000, 4, chunk_size=P.default_chunk_size(1000))
    assert plan.chunk_size == 62 and plan.bounds[-1][1] == 1000
    ids, ranges = plan.worker_chunks(1)
    assert ranges[0][0] == plan.bounds[1][0]
    with pytest.raises(ValueError):
        P.make_shard_plan(2, 3)
    cp = P.coil_shard_plan(16, 8)
    assert all(b - a == 2 for a, b in cp.bounds)
    with pytest.raises(ValueError):
        P.coil_shard_plan(4, 8)


def test_sample_chunk_grid_and_ordered_sum():
    # the global chunk grid of the order-stable split (csr_sample_chunking is
    # host arithmetic: no GPU needed) and ordered_chunk_sum's semantics
    # (sharding.py:173-208, test_sharding.py)
    from paper_2006_14080_b200.solver import plan_shard
    for nx, ny, nc, m in [(128, 128, 8, 16384), (256, 256, 16, 65536), (64, 64, 4, 4096),
                          (96, 80, 3, 10000), (16, 12, 3, 240)]:
        grid = P.ImageGrid(nx, ny)
        chunk, n = P.sample_chunking(grid, nc, m)
        assert chunk % 128 == 0 and (n - 1) * chunk < m <= n * chunk
        for world in range(1, min(n, 8) + 1):
            plan = P.sample_shard_plan(grid, nc, m, world)
            assert plan.chunk_size == chunk and plan.bounds[-1][1] == m
            assert all(a % chunk == 0 for a, _ in plan.bounds)
            spec = plan_shard(1, nc, world - 1, world, "sample", grid, m)
            assert spec.samples == plan.bounds[world - 1]
            assert spec.chunk_grid == (chunk, m)
            assert spec.chunk_ids == plan.worker_chunks(world - 1)[0]
    with pytest.raises(ValueError):
        plan_shard(4, 3, 0, 1, "sample", P.ImageGrid(8, 8), 100)
    rng = np.random.default_rng(5)
    parts = rng.standard_normal((7, 5, 4)).astype(np.float32)
    ref = parts[0].copy()
    for p in parts[1:]:
        ref += p
    for split in ([(0, 7)], [(0, 3), (3, 7)], [(0, 1), (1, 2), (2, 7)]):
        contribs = [(list(range(a, b)), parts[a:b]) for a, b in split]
        assert np.array_equal(P.ordered_chunk_sum(contribs[::-1]), ref)
    with pytest.raises(ValueError):
        P.ordered_chunk_sum([([0, 0], parts[:2])])
    with pytest.raises(ValueError):
        P.ordered_chunk_sum([([0], parts[:2])])
    with pytest.raises(ValueError):
        P.ordered_chunk_sum([])
    assert np.array_equal(P.allreduce_sum([parts[0], parts[1]]), parts[0] + parts[1])


def test_comm_stats_accounting():
    cs = P.CommStats()
    cs.record("setup", 100, calls=2)
    cs.record("solve", 100, calls=25)
    snap = cs.snapshot()
    assert snap["allreduce_calls"] == 27
    assert snap["per_phase"]["setup"] == {"calls": 2, "elements": 200}


def test_double_precision_is_rejected_not_run_on_cpu():
    with pytest.raises(ValueError, match="double"):
        P.DftOperator.build(np.zeros((4, 2)), P.ImageGrid(2, 2),
                            np.ones((1, 2, 2), np.complex64), precision="double")


def test_containers_validate_like_the_reference():
    with pytest.raises(ValueError):
        P.Trajectory(np.full((2, 2), 0.5), 1, 2)
    traj = P.Trajectory(np.zeros((4, 2)), 2, 2)
    with pytest.raises(ValueError):
        P.KSpaceDataset(np.zeros((3, 1), complex), traj)
    with pytest.raises(ValueError):
        P.KSpaceDataset(np.zeros((4, 1), complex), traj, n_frames=3)
    assert P.SensitivityMaps(np.ones((2, 3, 4))).grid.shape == (3, 4)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(NativeError):
        P.DftOperator.build(np.zeros((4, 2)), P.ImageGrid(2, 2),
                            np.ones((1, 2, 2), np.complex64))
    with pytest.raises(NativeError):
        P.theta(np.zeros((3, 3), np.complex64))


def test_harness_configs_match_baseline_shapes():
    from harness.configs import CONFIGS, nudft_flops_per_cg
    assert CONFIGS[1]["nx"] == 128 and CONFIGS[1]["n_coils"] == 8
    assert CONFIGS[4]["n_frames"] == 64 and CONFIGS[4]["admm_iters"] == 100
    # BASELINE.md §5 GFLOP per CG iteration
    assert abs(nudft_flops_per_cg(0) / 1e9 - 1.074) < 1e-3
    assert abs(nudft_flops_per_cg(2) / 1e9 - 1099.5) < 0.1
    assert abs(nudft_flops_per_cg(4) / 1e9 - 11545) < 1


def test_order_stable_shard_resolution():
    # solver.py:281-297: order_stable=True (the reference's default) makes
    # the image bitwise independent of n_workers; on several ranks a static
    # problem's shard="auto" therefore becomes the order-stable sample split
    from paper_2006_14080_b200.solver import resolve_shard
    assert resolve_shard("auto", True, 1, 4) == "sample"
    assert resolve_shard("auto", False, 1, 4) == "auto"
    assert resolve_shard("auto", True, 1, 1) == "auto"
    assert resolve_shard("auto", True, 8, 4) == "auto"      # 2-D+t: frames
    with pytest.warns(UserWarning, match="not bitwise independent"):
        assert resolve_shard("coil", True, 1, 2) == "coil"


def test_collective_argument_is_validated():
    from paper_2006_14080_b200.solver import _Shard
    with pytest.raises(ValueError, match="collective"):
        _Shard(None, np.zeros((1, 2, 2)), 1, "auto", None, collective="mpi")


def test_refbind_installs_into_a_kernel_table():
    # the reference's plug-in point (kernels.py:212-274): the "cuda" table
    # replaces the active one and can be removed again; building the table
    # touches no device
    import types
    import paper_2006_14080_b200.refbind as rb
    numpy_table = {"forward_sep": None}
    k = types.SimpleNamespace(_IMPL={"numpy": numpy_table}, _ACTIVE=numpy_table,
                              _BACKEND="numpy")
    prev = rb.install(k)
    assert k._BACKEND == "cuda" and k._ACTIVE is k._IMPL["cuda"]
    assert set(k._ACTIVE) >= {"forward_mat", "adjoint_mat", "forward_sep", "adjoint_sep",
                              "theta", "theta_adj", "soft"}
    with pytest.raises(NotImplementedError, match="separable"):
        k._ACTIVE["forward_mat"](None, None, None)
    rb.uninstall(k, prev)
    assert k._BACKEND == "numpy" and k._ACTIVE is numpy_table and "cuda" not in k._IMPL
