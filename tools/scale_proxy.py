"""Single-GPU proxy of one rank of a P-GPU sharded run.  2-D+t configs
(3 / 4): the first T/P frames of the config as their own problem,
frame-shard mode with a one-rank NCCL communicator attached, so the plan
takes exactly the code path of a rank of the P-GPU run (frame-split CG
kernels, halo all-gather, fp64 scalar allreduces, its GEMM grids for T/P
frames) — only the NCCL transfers go to self instead of over NVLink.
Device time of K ADMM iterations (CUDA events, L2 flushed between
iterations, as bench.py).  The P-GPU rate is bounded by one rank's rate,
so  efficiency(P) ~= rate(T/P frames) / (P * rate(T frames, 1 GPU)).
Static configs (0-2): the rank's coils (coil shard, >= 4 coils per rank) or
its 1/P of the samples (sample split), with the shard mode's per-CG-iteration
image allreduce through the one-rank communicator.

    python tools/scale_proxy.py [config=4] [steps=10]
prints one JSON line per P in 1, 2, 4, 8 plus the plain 1-GPU run."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_14080_b200 as P  # noqa: E402
from paper_2006_14080_b200 import _native  # noqa: E402
from paper_2006_14080_b200.solver import _Shard  # noqa: E402
from bench import ClockSampler, input_encoder  # noqa: E402
from harness.configs import make_problem  # noqa: E402


def rate(prob, frames, steps, shard, collective, dev, samples=None, coils=None):
    m = prob.coords.shape[0] // prob.n_frames
    coords, data = prob.coords[:frames * m], prob.data[:frames * m]
    sens = prob.sens
    if samples is not None:  # static sample split: this rank's run of samples
        coords, data = coords[:samples], data[:samples]
    if coils is not None:    # static coil split: this rank's coils
        sens, data = sens[:coils], data[:, :coils]
    traj = P.Trajectory(coords, coords.shape[0], 1)
    ds = P.KSpaceDataset(data, traj, n_frames=frames)
    sh = _Shard(ds, sens, 1, "auto", dev, shard=shard, collective=collective)
    op, lib = sh.op, _native.load()

    def run(n, iter_ms=None, flush=None):
        params = P.ReconParams(**dict(prob.params, admm_max_iters=n))
        rho = torch.empty(op.image_shape, dtype=torch.complex64, device=dev)
        log = (_native.IterLog * n)()
        stats = _native.RunStats()
        if iter_ms is not None:
            _native.call("csr_plan_set_timing", op.plan, flush.data_ptr(), flush.numel(), iter_ms)
        _native.check(lib.csr_admm_run(op.plan, ctypes.byref(params.native()),
                                       sh.data.data_ptr(), rho.data_ptr(), log,
                                       ctypes.byref(stats),
                                       torch.cuda.current_stream(dev).cuda_stream, None))
        _native.call("csr_plan_set_timing", op.plan, None, 0, None)
        return stats

    run(3)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    iter_ms = (ctypes.c_float * steps)()
    clk = ClockSampler(dev.index)
    torch.cuda.synchronize()
    clk.start()
    st = run(steps, iter_ms, flush)
    torch.cuda.synchronize()
    c = clk.stop()
    del sh
    torch.cuda.empty_cache()
    return steps / (st.solve_ms / 1e3), st.kernels_per_iter, c


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    prob = make_problem(cfg, encoder=input_encoder(cfg))
    T = prob.n_frames
    r1, k1, c1 = rate(prob, T, steps, "auto", "auto", dev)
    print(json.dumps({"config": cfg, "mode": "1 GPU, no communicator", "frames": T,
                      "iters_per_s": r1, "kernels_per_iter": k1, "clocks": c1}), flush=True)
    for p in (1, 2, 4, 8):
        if T > 1:
            if T % p:
                continue
            r, k, c = rate(prob, T // p, steps, "frame", "nccl", dev)
            what, size = "frame shard", {"frames": T // p}
        else:
            # bench.py's static split: coils while >= 4 per rank, else samples
            C, M = prob.n_coils, prob.coords.shape[0]
            if C // p >= 4:
                r, k, c = rate(prob, 1, steps, "coil", "nccl", dev, coils=C // p)
                what, size = "coil shard", {"coils": C // p}
            else:
                r, k, c = rate(prob, 1, steps, "split", "nccl", dev, samples=M // p)
                what, size = "sample split", {"samples": M // p}
        print(json.dumps({"config": cfg, "mode": f"one rank of {p} ({what}, 1-rank NCCL)", **size,
                          "iters_per_s": r, "kernels_per_iter": k,
                          "proxy_efficiency_vs_1gpu": r / (p * r1), "clocks": c}), flush=True)


if __name__ == "__main__":
    main()
