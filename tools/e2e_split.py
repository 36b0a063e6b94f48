"""Where the end-to-end call loses against the timed device loop (config C):
(a) csr_admm_run on one plan with per-iteration events + L2 flush (bench
'value'), (b) the same plan without timing (wall clock around the call),
(c) admm_reconstruct with host arrays (plan build included)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from paper_2006_14080_b200.solver import _Shard
from harness.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg)
traj = P.Trajectory(prob.coords, prob.coords.shape[0], 1)
ds = P.KSpaceDataset(prob.data, traj, n_frames=prob.n_frames)
n = prob.params["admm_max_iters"]
params = P.ReconParams(**prob.params)
dev = torch.device("cuda", 0)
sh = _Shard(ds, prob.sens, 1, "auto", dev)
lib = _native.load()
rho = torch.empty(sh.op.image_shape, dtype=torch.complex64, device=dev)
log = (_native.IterLog * n)()
st = torch.cuda.current_stream(dev).cuda_stream
def run(timing=False):
    stats = _native.RunStats()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ims = (ctypes.c_float * n)()
    if timing:
        _native.call("csr_plan_set_timing", sh.op.plan, flush.data_ptr(), flush.numel(), ims)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.check(lib.csr_admm_run(sh.op.plan, ctypes.byref(params.native()), sh.data.data_ptr(),
                                   rho.data_ptr(), log, ctypes.byref(stats), st, None))
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    _native.call("csr_plan_set_timing", sh.op.plan, None, 0, None)
    return wall * 1e3, stats.solve_ms, stats.setup_ms
for i in range(3): run()
for i in range(3):
    w, s, su = run(True); print(f"(a) timed+flush: wall {w:.2f} ms, solve_ms {s:.2f} ({1e3 * s / n:.1f} us/it)")
for i in range(3):
    w, s, su = run(False); print(f"(b) untimed:     wall {w:.2f} ms, solve_ms {s:.2f}, setup {su:.3f}")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
dsp = P.KSpaceDataset(pin(prob.data), traj, n_frames=prob.n_frames)
sp = pin(prob.sens)
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    img, rep = P.admm_reconstruct(dsp, sp, params, compute_objectives=False, device=dev)
    torch.cuda.synchronize(); w = 1e3 * (time.perf_counter() - t0)
    print(f"(c) admm_reconstruct: wall {w:.2f} ms, solve {1e3 * rep.timing['solve_seconds']:.2f}, setup {1e3 * rep.timing['setup_seconds']:.2f}")
