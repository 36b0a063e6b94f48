"""The NCCL code paths of every shard mode, run for real on one GPU.

A plan with a communicator attached takes its shard mode's collective path
for any rank count (include/csrecon_b200.h): ``collective="nccl"`` gives a
one-rank NCCL communicator, so the image allreduce (coil / plain sample
split, sharding.py:211-250, solver.py:136), the chunk all-gather and the
k-space max-allreduce (order-stable sample split, sharding.py:173-208), and
the frame split's halo all-gather and fp64 scalar allreduces all execute
through NCCL inside the captured iteration graph.  (The halo is an
all-gather of every rank's [first | last] frames rather than a ring of
send/recv: NCCL send/recv to self inside a captured graph never completes,
tools/nccl_self_probe.cu, measured on the B200 with NCCL 2.28.9, so only a
collective lets the one-rank run take the same path as P ranks.)  Each run
is compared with the plain single-GPU run of the same problem.
"""

import numpy as np
import pytest

import paper_2006_14080_b200 as P
from conftest import golden, random_complex, rel_err
from oracle import csrecon_oracle as O

pytestmark = pytest.mark.gpu


def _dataset(coords, data, n_frames=1):
    return P.KSpaceDataset(data, P.Trajectory(coords, coords.shape[0], 1), n_frames=n_frames)


def _static_problem():
    from harness.configs import make_problem
    prob = make_problem(1)
    params = P.ReconParams(**dict(prob.params, admm_max_iters=6))
    return _dataset(prob.coords, prob.data), prob.sens, params


@pytest.mark.parametrize("shard", ["coil", "split"])
def test_allreduce_path_matches_single_gpu(cuda, shard):
    ds, sens, params = _static_problem()
    ref, rep0 = P.admm_reconstruct(ds, sens, params, compute_objectives=False, shard=shard)
    img, rep = P.admm_reconstruct(ds, sens, params, compute_objectives=False, shard=shard,
                                  collective="nccl")
    err = rel_err(img, ref)
    print(f"{shard}: NCCL path vs single GPU rel-L2 {err:.2e}, "
          f"{rep.timing['kernels_per_iteration']} vs {rep0.timing['kernels_per_iteration']} "
          f"kernels per iteration; allreduce calls {rep.comm['allreduce_calls']}")
    assert err <= 1e-6
    # two setup collectives + one per CG iteration (solver.py:136, 307-309)
    assert rep.comm["allreduce_calls"] == 2 + 5 * params.admm_max_iters
    assert rep0.comm.get("allreduce_calls", 0) == 0


def test_ordered_sample_path_is_bitwise(cuda):
    # order-stable split: chunk partials all-gathered and folded in chunk
    # order, the k-space operand scale max-allreduced -> the same bits as
    # the single-GPU order-stable plan
    ds, sens, params = _static_problem()
    ref, _ = P.admm_reconstruct(ds, sens, params, compute_objectives=False, shard="sample")
    img, rep = P.admm_reconstruct(ds, sens, params, compute_objectives=False, shard="sample",
                                  collective="nccl")
    assert np.array_equal(img, ref)
    ad0, _ = P.adjoint_reconstruct(ds, sens, shard="sample")
    ad1, _ = P.adjoint_reconstruct(ds, sens, shard="sample", collective="nccl")
    assert rel_err(ad1, ad0) <= 1e-6


def test_frame_path_halo_and_scalar_allreduce(cuda):
    # 2-D+t frame split: halo frames through the NCCL all-gather of the
    # ranks' boundary pairs, CG / ADMM scalars as fp64 NCCL sums before the
    # device-side finalize; against the plain run and the f64 restatement
    rng = np.random.default_rng(9)
    T, nx, ny, C, m = 3, 20, 16, 3, 250
    coords = rng.uniform(-0.5, 0.4999, size=(T * m, 2))
    sens = random_complex(rng, (C, nx, ny)) * 0.3
    truth = random_complex(rng, (T, nx, ny))
    data = O.Operator(coords, sens, T).forward(truth)
    kw = dict(lam=1e-3, beta=1e-2, admm_rtol=1e-150, admm_max_iters=5, cg_atol=1e-150,
              cg_max_iters=5)
    ref, _ = O.admm(data, coords, sens, O.Params(lam_t=5e-3, **kw), n_frames=T)
    ds = _dataset(coords, data, T)
    params = P.ReconParams(lam_t=5e-3, **kw)
    plain, _ = P.admm_reconstruct(ds, sens, params, shard="frame", compute_objectives=False)
    img, rep = P.admm_reconstruct(ds, sens, params, shard="frame", collective="nccl",
                                  compute_objectives=False)
    assert rep.timing["shard"] == "frame"
    assert rel_err(img, plain) <= 1e-6
    assert rel_err(img, ref) <= 1e-4


def test_comm_allreduce_entry(cuda):
    import torch
    from paper_2006_14080_b200.sharding import NcclComm
    comm = NcclComm(0, 1, 0)
    t = torch.arange(10, dtype=torch.float32, device="cuda").to(torch.complex64)
    out = comm.allreduce_(t.clone(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(out, t)
    comm.close()


def test_small_fixture_through_every_collective_mode(cuda):
    g = golden("admm_small.npz")
    lam, beta, rtol, na, atol, ncg = g["fixed_params"]
    params = P.ReconParams(lam=lam, beta=beta, admm_rtol=rtol, admm_max_iters=int(na),
                           cg_atol=atol, cg_max_iters=int(ncg))
    ds = _dataset(g["coords"], g["data"])
    for shard in ("coil", "split", "sample"):
        img, _ = P.admm_reconstruct(ds, g["sens"], params, compute_objectives=False,
                                    shard=shard, collective="nccl")
        assert rel_err(img, g["fixed_double_image"]) <= 1e-4, shard
