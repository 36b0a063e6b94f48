"""World-size-2 tests of the multi-GPU decomposition on CPU (gloo).

The device loop shards coils (static problems: one image allreduce per CG
iteration) or frames (2-D+t: halo exchange (all-gather of boundary frames) for the temporal
differences, allreduced CG/ADMM scalars).  These tests run the same
decomposition with the f64 oracle as the per-rank compute stand-in and gloo
as the interconnect, and check it reproduces the unsharded solve; they also
exercise the host-side shard planning and the NCCL unique-id broadcast.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import csrecon_oracle as O
from paper_2006_14080_b200.sharding import broadcast_unique_id
from paper_2006_14080_b200.solver import plan_shard, shard_inputs

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(T, seed=11, nx=12, ny=10, C=4, m=90):
    rng = np.random.default_rng(seed)
    coords = rng.uniform(-0.5, 0.4999, size=(T * m, 2))
    sens = (rng.standard_normal((C, nx, ny)) + 1j * rng.standard_normal((C, nx, ny))) * 0.4
    truth = rng.standard_normal((T, nx, ny)) + 1j * rng.standard_normal((T, nx, ny))
    op = O.Operator(coords, sens, T)
    data = op.forward(truth if T > 1 else truth[0])
    params = O.Params(lam=1e-3, beta=1e-2, admm_rtol=1e-150, admm_max_iters=4,
                      cg_atol=1e-150, cg_max_iters=5, lam_t=5e-3)
    return coords, sens, data, params


def _allreduce(arr):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.is_complex():
        v = torch.view_as_real(t).clone()
        dist.all_reduce(v)
        return torch.view_as_complex(v).numpy()
    v = t.clone()
    dist.all_reduce(v)
    return v.numpy()


def _ring_exchange(first, last, rank, world):
    """hprev <- previous rank's last frame, hnext <- next rank's first frame,
    as the device loop's halo_exchange does it: every rank contributes its
    [first | last] pair to one all-gather and reads its neighbours' slots
    (csrecon_b200.cu halo_exchange / csr_plan_set_comm)."""
    pair = torch.view_as_real(torch.from_numpy(np.ascontiguousarray(
        np.stack([first, last])))).clone()
    gathered = [torch.empty_like(pair) for _ in range(world)]
    dist.all_gather(gathered, pair)
    prev = torch.view_as_complex(gathered[(rank - 1) % world][1].contiguous()).numpy()
    nxt = torch.view_as_complex(gathered[(rank + 1) % world][0].contiguous()).numpy()
    return prev, nxt


def _theta_h(v, prev):
    """theta of a frame block with the temporal difference at frame 0 taken
    against the halo frame (k_admm_mu / theta_at with hprev)."""
    out = np.empty((3,) + v.shape, v.dtype)
    out[0] = v - np.roll(v, 1, axis=1)
    out[1] = v - np.roll(v, 1, axis=2)
    out[2][1:] = v[1:] - v[:-1]
    out[2][0] = v[0] - prev
    return out


def _theta_adj_h(u, u2_next):
    """theta^H with the temporal component of frame T taken from the halo
    (theta_adj_at in halo mode)."""
    d0, d1, d2 = u
    out = (d0 - np.roll(d0, -1, axis=1)) + (d1 - np.roll(d1, -1, axis=2))
    d2n = np.concatenate([d2[1:], u2_next[None]], axis=0)
    return out + (d2 - d2n)


def _frame_sharded_admm(rank, world, coords, sens, data, params, T):
    """The device loop's frame decomposition (csrecon_b200.cu
    enqueue_admm_iteration, frame mode) with the oracle as the compute."""
    spec = plan_shard(T, sens.shape[0], rank, world, "frame")
    lc, ld, lm = shard_inputs(coords, data, sens, T, spec)
    tl = spec.frames[1] - spec.frames[0]
    op = O.Operator(lc, lm, tl)
    fhd = op.adjoint(ld).reshape(tl, *sens.shape[1:])
    rho = fhd.copy()
    mu = np.zeros((3,) + rho.shape, complex)
    eta = mu.copy()
    hb = params.beta / 2
    t_s, t_t = params.lam / params.beta, params.lam_t / params.beta

    def apply_a(d):
        prev, nxt = _ring_exchange(d[0], d[-1], rank, world)
        th = _theta_h(d, prev)
        th2_next = nxt - d[-1]
        ff = op.adjoint(op.forward(d)).reshape(d.shape)
        return ff + hb * _theta_adj_h(th, th2_next)

    for _ in range(params.admm_max_iters):
        prev, _unused = _ring_exchange(rho[0], rho[-1], rank, world)
        v = _theta_h(rho, prev) + eta
        mu = O.shrink_stack(v, t_s, t_t)
        me0 = mu[2][0] - eta[2][0]
        _unused, me_next = _ring_exchange(me0, me0, rank, world)
        rhs = fhd + hb * _theta_adj_h(mu - eta, me_next)
        x = np.zeros_like(rhs)
        r = rhs.copy()
        d = r.copy()
        tau = float(_allreduce(np.array([np.vdot(r, r).real]))[0])
        for _ in range(params.cg_max_iters):
            ad = apply_a(d)
            dad = _allreduce(np.array([np.vdot(d, ad)]))[0]
            alpha = tau / dad
            x = x + alpha * d
            r = r - alpha * ad
            tn = float(_allreduce(np.array([np.vdot(r, r).real]))[0])
            d = r + (tn / tau) * d
            tau = tn
        prev, _unused = _ring_exchange(x[0], x[-1], rank, world)
        eta = eta + (_theta_h(x, prev) - mu)
        rho = x
    return spec, rho


def _coil_sharded_admm(rank, world, coords, sens, data, params, T, mode="coil"):
    spec = plan_shard(T, sens.shape[0], rank, world, mode, n_samples=coords.shape[0])
    lc, ld, lm = shard_inputs(coords, data, sens, T, spec)
    op = O.Operator(lc, lm, T)
    img, recs = O.admm(ld, lc, lm, params, "double", T, allreduce=_allreduce, op=op)
    return spec, img


def _chunked_partials(coords, sens, v, chunks, data=None):
    """Per-chunk F^H F v (or F^H d) partials, each from its own samples only
    (ChunkedDftOperator, operators.py:206-272)."""
    out = []
    for a, b in chunks:
        p0, p1 = O.build_factors(coords[a:b], *sens.shape[1:])
        d = data[a:b] if data is not None else O.forward_sep(p0, p1, sens, v)
        out.append(O.adjoint_sep(p0, p1, sens, d))
    return np.stack(out)


def _ordered_admm(rank, world, coords, sens, data, params, chunk, gather):
    """The device loop's order-stable sample decomposition
    (CSR_PLAN_ORDERED_SAMPLES): each rank computes its chunks' partials, the
    stacks are all-gathered and folded in global chunk order; everything
    else is replicated."""
    from paper_2006_14080_b200.sharding import make_shard_plan, ordered_chunk_sum
    plan = make_shard_plan(coords.shape[0], world, chunk_size=chunk)
    ids, ranges = plan.worker_chunks(rank)

    def reduce(stack):
        return ordered_chunk_sum(gather((ids, stack)))

    fhd = reduce(_chunked_partials(coords, sens, None, ranges, data))
    rho = fhd.copy()
    mu = np.zeros((2,) + rho.shape, complex)
    eta = mu.copy()
    hb, t = params.beta / 2, params.lam / params.beta
    for _ in range(params.admm_max_iters):
        mu = O.soft_threshold(O.theta(rho) + eta, t)
        rhs = fhd + hb * O.theta_adjoint(mu - eta)
        x = np.zeros_like(rhs)
        r = rhs.copy()
        d = r.copy()
        tau = np.vdot(r, r).real
        for _ in range(params.cg_max_iters):
            ad = reduce(_chunked_partials(coords, sens, d, ranges)) + \
                hb * O.theta_adjoint(O.theta(d))
            alpha = tau / np.vdot(d, ad)
            x = x + alpha * d
            r = r - alpha * ad
            tn = np.vdot(r, r).real
            d = r + (tn / tau) * d
            tau = tn
        eta = eta + (O.theta(x) - mu)
        rho = x
    return plan, rho


def _gather_objects(obj):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, obj)
    return parts


def _worker(rank, world, port, mode, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode == "uid":
            uid = broadcast_unique_id(rank, make_id=lambda: bytes(range(128)))
            res = {"uid": np.frombuffer(uid, np.uint8)}
        elif mode == "sample":
            coords, sens, data, params = _problem(1, m=150)
            plan, img = _ordered_admm(rank, world, coords, sens, data, params, 32,
                                      _gather_objects)
            res = {"img": img, "bounds": np.array(plan.bounds[rank])}
        else:
            T = 4 if mode.startswith("frame") else (4 if mode == "coil_dyn" else 1)
            coords, sens, data, params = _problem(T)
            if mode.startswith("frame"):
                spec, img = _frame_sharded_admm(rank, world, coords, sens, data, params, T)
            else:
                spec, img = _coil_sharded_admm(rank, world, coords, sens, data, params, T,
                                               "split" if mode == "split" else "coil")
            res = {"img": img, "frames": np.array(spec.frames), "coils": np.array(spec.coils)}
        np.savez(out_path.format(rank=rank), **res)
    finally:
        dist.destroy_process_group()


def _run(mode, tmp_path):
    out = str(tmp_path / ("res_{rank}_" + mode + ".npz"))
    mp.spawn(_worker, args=(WORLD, _free_port(), mode, out), nprocs=WORLD, join=True)
    return [np.load(out.format(rank=r)) for r in range(WORLD)]


def test_unique_id_broadcast(tmp_path):
    res = _run("uid", tmp_path)
    for r in res:
        assert np.array_equal(r["uid"], np.arange(128, dtype=np.uint8))


@pytest.mark.parametrize("mode", ["coil", "coil_dyn", "split"])
def test_coil_sharded_admm_matches_unsharded(mode, tmp_path):
    T = 4 if mode == "coil_dyn" else 1
    coords, sens, data, params = _problem(T)
    ref, _ = O.admm(data, coords, sens, params, "double", T)
    res = _run(mode, tmp_path)
    if mode == "split":  # every rank holds all coils and half the samples
        assert tuple(res[0]["coils"]) == (0, 4) and tuple(res[1]["coils"]) == (0, 4)
    else:
        assert tuple(res[0]["coils"]) == (0, 2) and tuple(res[1]["coils"]) == (2, 4)
    for r in res:  # replicated image on every rank
        img = r["img"]
        assert np.linalg.norm(img - ref) <= 1e-10 * np.linalg.norm(ref)


def test_frame_sharded_admm_matches_unsharded(tmp_path):
    T = 4
    coords, sens, data, params = _problem(T)
    ref, _ = O.admm(data, coords, sens, params, "double", T)
    res = _run("frame", tmp_path)
    img = np.concatenate([r["img"] for r in res], axis=0)
    assert tuple(res[0]["frames"]) == (0, 2) and tuple(res[1]["frames"]) == (2, 4)
    assert np.linalg.norm(img - ref) <= 1e-10 * np.linalg.norm(ref)


def test_sample_sharded_admm_bitwise_independent_of_world(tmp_path):
    # order-stable sample sharding (sharding.py:173-208): two ranks reproduce
    # the one-rank result bit for bit
    coords, sens, data, params = _problem(1, m=150)
    _, ref = _ordered_admm(0, 1, coords, sens, data, params, 32, lambda o: [o])
    res = _run("sample", tmp_path)
    assert tuple(res[0]["bounds"]) == (0, 96) and tuple(res[1]["bounds"]) == (96, 150)
    for r in res:
        assert np.array_equal(r["img"], ref)
    full, _ = O.admm(data, coords, sens, params, "double", 1)
    assert np.linalg.norm(ref - full) <= 1e-10 * np.linalg.norm(full)


def test_plan_shard_rules():
    assert plan_shard(64, 16, 3, 8).mode == "frame"
    assert plan_shard(64, 16, 3, 8).frames == (24, 32)
    assert plan_shard(1, 16, 3, 8).mode == "coil"
    assert plan_shard(1, 16, 3, 8).coils == (6, 8)
    # fewer than 4 coils per rank (the operator pads coils to 4): sample split
    assert plan_shard(1, 32, 3, 8, n_samples=16384).mode == "coil"
    sp = plan_shard(1, 8, 3, 8, n_samples=16384)
    assert sp.mode == "split" and sp.samples == (6144, 8192) and sp.coils == (0, 8)
    assert plan_shard(1, 8, 1, 2, n_samples=16384).mode == "coil"
    assert plan_shard(4, 3, 0, 1, "frame").frames == (0, 4)
    with pytest.raises(ValueError):
        plan_shard(4, 3, 0, 1, "tiles")
