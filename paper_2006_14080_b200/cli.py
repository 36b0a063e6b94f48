"""Command-line front end for the reconstruction path (mirror of the
`reconstruct` and `benchmark` commands of csrecon/cli.py:172-283).

    python -m paper_2006_14080_b200.cli reconstruct --data DIR --out IMG [...]
    python -m paper_2006_14080_b200.cli benchmark --data DIR --out CSV [...]

Same flags, defaults and report document as the reference; exit codes 0
success, 1 runtime failure, 2 usage error (cli.py:1-4).  Differences: the
arithmetic is single precision on the GPU (`--precision f32` is the
default; `f64` is a runtime error, there is no CPU fallback), and a worker
is one GPU (one process per GPU): `--workers N` > 1 must be launched under
torchrun, and `benchmark` runs each worker count as its own torchrun job.
"""

import argparse
import csv
import json
import os
import subprocess
import sys
import time

PRECISION_FLAGS = {"f32": "single", "f64": "double"}


def _positive_int(text):
    try:
        v = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected an integer, got {text!r}")
    if v < 1:
        raise argparse.ArgumentTypeError(f"expected a positive integer, got {v}")
    return v


def _workers_list(text):
    items = [s.strip() for s in text.split(",") if s.strip()]
    if not items:
        raise argparse.ArgumentTypeError("worker list must not be empty")
    return [_positive_int(s) for s in items]


def _solver_flags(p):
    # defaults of cli.py:55-67
    p.add_argument("--lambda", dest="lam", type=float, default=1e-7)
    p.add_argument("--beta", type=float, default=1.0)
    p.add_argument("--admm-rtol", type=float, default=1e-4)
    p.add_argument("--admm-iters", type=_positive_int, default=5)
    p.add_argument("--cg-atol", type=float, default=1e-6)
    p.add_argument("--cg-iters", type=_positive_int, default=20)
    p.add_argument("--lambda-t", dest="lam_t", type=float, default=None,
                   help="temporal weight for 2-D+t datasets (default: --lambda)")


def _run_flags(p):
    p.add_argument("--precision", choices=sorted(PRECISION_FLAGS), default="f32")
    p.add_argument("--op-mode", choices=("auto", "materialized", "separable"),
                   default="auto")
    p.add_argument("--memory-budget-gib", type=float, default=None)
    p.add_argument("--shard", choices=("auto", "coil", "frame", "sample", "split"), default="auto",
                   help="work split across GPU workers; 'sample' is the reference's "
                        "order-stable split (bitwise the same image for any --workers)")


def build_parser():
    parser = argparse.ArgumentParser(
        prog="paper_2006_14080_b200",
        description="B200 ADMM reconstruction of radial multi-coil k-space")
    sub = parser.add_subparsers(dest="command", required=True)
    rec = sub.add_parser("reconstruct", help="reconstruct an image from a dataset")
    rec.add_argument("--data", required=True)
    rec.add_argument("--out", required=True)
    rec.add_argument("--report", default=None)
    rec.add_argument("--method", choices=("admm", "adjoint"), default="admm")
    rec.add_argument("--workers", type=_positive_int, default=1)
    _solver_flags(rec)
    _run_flags(rec)
    rec.set_defaults(func=cmd_reconstruct)
    ben = sub.add_parser("benchmark", help="strong-scaling wall-time table")
    ben.add_argument("--data", required=True)
    ben.add_argument("--out", required=True)
    ben.add_argument("--workers-list", type=_workers_list, default=[1, 2, 4])
    ben.add_argument("--repeat", type=_positive_int, default=3)
    _solver_flags(ben)
    _run_flags(ben)
    ben.set_defaults(func=cmd_benchmark)
    wk = sub.add_parser("_bench-worker", help=argparse.SUPPRESS)
    wk.add_argument("--data", required=True)
    wk.add_argument("--repeat", type=_positive_int, default=3)
    _solver_flags(wk)
    _run_flags(wk)
    wk.set_defaults(func=cmd_bench_worker)
    return parser


def _memory_budget(args):
    from .operators import DEFAULT_MEMORY_BUDGET
    if args.memory_budget_gib is None:
        return DEFAULT_MEMORY_BUDGET
    if args.memory_budget_gib <= 0:
        raise ValueError("memory budget must be positive")
    return int(args.memory_budget_gib * 1024 ** 3)


def _params(args):
    from .solver import ReconParams
    return ReconParams(lam=args.lam, beta=args.beta, admm_rtol=args.admm_rtol,
                       admm_max_iters=args.admm_iters, cg_atol=args.cg_atol,
                       cg_max_iters=args.cg_iters, lam_t=args.lam_t)


def _init_dist(workers):
    """One process per GPU: under torchrun join the group (gloo carries the
    NCCL id; the solver's NCCL comm does the data path)."""
    if workers == 1:
        return
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))


def cmd_reconstruct(args):
    from .io import load_dataset, write_tensor
    from .solver import admm_reconstruct, adjoint_reconstruct
    _init_dist(args.workers)
    _, sens, dataset, _ = load_dataset(args.data)
    precision = PRECISION_FLAGS[args.precision]
    budget = _memory_budget(args)
    if args.method == "admm":
        image, report = admm_reconstruct(dataset, sens, _params(args),
                                         n_workers=args.workers, precision=precision,
                                         op_mode=args.op_mode, memory_budget=budget,
                                         shard=args.shard)
    else:
        image, report = adjoint_reconstruct(dataset, sens, n_workers=args.workers,
                                            precision=precision, op_mode=args.op_mode,
                                            memory_budget=budget, shard=args.shard)
    rank = int(os.environ.get("RANK", "0"))
    report_path = args.report or f"{args.out}.report.json"
    if rank == 0:
        write_tensor(args.out, image)
        doc = report.to_dict()
        doc["dataset"] = str(args.data)
        doc["image"] = str(args.out)
        with open(report_path, "w") as f:
            json.dump(doc, f, indent=2, sort_keys=True)
            f.write("\n")
        print(f"wrote {args.out} ({report.grid[0]}x{report.grid[1]} {precision}, "
              f"{args.method}, {len(report.iterations)} outer iterations); "
              f"report: {report_path}")
    return 0


def _best_time(args, workers):
    from .io import load_dataset
    from .solver import admm_reconstruct
    _, sens, dataset, _ = load_dataset(args.data)
    best = None
    for _ in range(args.repeat):
        t0 = time.perf_counter()
        admm_reconstruct(dataset, sens, _params(args), n_workers=workers,
                         precision=PRECISION_FLAGS[args.precision], op_mode=args.op_mode,
                         memory_budget=_memory_budget(args), compute_objectives=False,
                         shard=args.shard)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


def cmd_bench_worker(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    _init_dist(world)
    best = _best_time(args, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([best], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = float(t.item())
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"best_seconds": best}))
    return 0


def _flags_for_worker(args):
    out = ["--data", str(args.data), "--repeat", str(args.repeat),
           "--lambda", repr(args.lam), "--beta", repr(args.beta),
           "--admm-rtol", repr(args.admm_rtol), "--admm-iters", str(args.admm_iters),
           "--cg-atol", repr(args.cg_atol), "--cg-iters", str(args.cg_iters),
           "--precision", args.precision, "--op-mode", args.op_mode, "--shard", args.shard]
    if args.lam_t is not None:
        out += ["--lambda-t", repr(args.lam_t)]
    if args.memory_budget_gib is not None:
        out += ["--memory-budget-gib", repr(args.memory_budget_gib)]
    return out


def run_benchmark(args):
    """Best-of-repeat wall time per worker count (cli.py:223-262): each
    count is its own one-process-per-GPU job; counts above the visible GPUs
    are reported with a note instead of a time."""
    import socket

    import torch
    avail = torch.cuda.device_count()
    times = {}
    for p in args.workers_list:
        if p > avail:
            times[p] = None
            continue
        if p == 1:
            times[p] = _best_time(args, 1)
            continue
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={p}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), "-m", "paper_2006_14080_b200.cli",
               "_bench-worker"] + _flags_for_worker(args)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            raise RuntimeError(f"{p}-GPU benchmark job failed: {res.stderr[-400:]}")
        times[p] = json.loads(res.stdout.strip().splitlines()[-1])["best_seconds"]
    measured = [p for p in args.workers_list if times[p] is not None]
    if not measured:
        raise RuntimeError(f"no worker count fits the {avail} visible GPU(s)")
    base = min(measured)
    rows, prev = [], None
    for p in args.workers_list:
        if times[p] is None:
            rows.append({"workers": p, "best_seconds": None, "speedup": None,
                         "ideal_speedup": p / base,
                         "note": f"needs {p} GPUs, {avail} visible"})
            continue
        note = "slower than previous worker count" if prev is not None and times[p] > prev else ""
        rows.append({"workers": p, "best_seconds": times[p], "speedup": times[base] / times[p],
                     "ideal_speedup": p / base, "note": note})
        prev = times[p]
    return rows


def cmd_benchmark(args):
    rows = run_benchmark(args)
    with open(args.out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["workers", "best_seconds", "speedup",
                                          "ideal_speedup", "note"])
        w.writeheader()
        for r in rows:
            w.writerow({"workers": r["workers"],
                        "best_seconds": "" if r["best_seconds"] is None else f"{r['best_seconds']:.6f}",
                        "speedup": "" if r["speedup"] is None else f"{r['speedup']:.3f}",
                        "ideal_speedup": f"{r['ideal_speedup']:.3f}", "note": r["note"]})
    for r in rows:
        if r["best_seconds"] is None:
            print(f"workers {r['workers']:>3}: skipped ({r['note']})")
            continue
        flag = f"  [{r['note']}]" if r["note"] else ""
        print(f"workers {r['workers']:>3}: {r['best_seconds']:.3f} s  speedup "
              f"{r['speedup']:.2f} (ideal {r['ideal_speedup']:.2f}){flag}")
    return 0


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except BrokenPipeError:
        return 1
    except Exception as exc:  # runtime failures -> 1 (cli.py:286-295)
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
