"""Device timeline of one timed ADMM iteration (probed kernels): start/end
of every launch and the gaps between them (csr_debug_timeline)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from paper_2006_14080_b200.solver import _Shard
from harness.configs import make_problem
lib = _native.load()
lib.csr_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg)
traj = P.Trajectory(prob.coords, prob.coords.shape[0], 1)
ds = P.KSpaceDataset(prob.data, traj, n_frames=prob.n_frames)
sh = _Shard(ds, prob.sens, 1, "auto", torch.device("cuda", 0))
op = sh.op
names = ["fwd", "adj", "head", "rhs", "prep", "tail", "post", "snap"]
def run(n, flush=None, iter_ms=None):
    params = P.ReconParams(**dict(prob.params, admm_max_iters=n))
    rho = torch.empty(op.image_shape, dtype=torch.complex64, device="cuda")
    log = (_native.IterLog * n)()
    stats = _native.RunStats()
    if iter_ms is not None:
        _native.call("csr_plan_set_timing", op.plan, flush.data_ptr(), flush.numel(), iter_ms)
    lib.csr_admm_run(op.plan, ctypes.byref(params.native()), sh.data.data_ptr(), rho.data_ptr(),
                     log, ctypes.byref(stats), torch.cuda.current_stream().cuda_stream, None)
    _native.call("csr_plan_set_timing", op.plan, None, 0, None)
run(3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
iter_ms = (ctypes.c_float * 4)()
lib.csr_debug_timeline(op.plan, 1, None, 0)
run(4, flush, iter_ms)
buf = np.zeros(3 * 4096, np.uint64)
n = lib.csr_debug_timeline(op.plan, 0, buf.ctypes.data, 4096)
rec = buf[:3 * n].reshape(n, 3).astype(np.int64)
rec = rec[np.argsort(rec[:, 1])]
print("per-iteration device ms:", [round(v, 4) for v in iter_ms])
# last iteration: the records after the last 'head'
heads = np.where(rec[:, 0] == 2)[0]
it = rec[heads[-2]:heads[-1]] if len(heads) > 1 else rec
t0 = it[0, 1]
prev_end = None
tot_gap = 0
for s, a, b in it:
    gap = (a - prev_end) / 1e3 if prev_end is not None else 0.0
    tot_gap += max(gap, 0)
    print(f"{names[s] if s < len(names) else s:6s} start {(a - t0) / 1e3:8.2f} dur {(b - a) / 1e3:7.2f} gap {gap:6.2f} us")
    prev_end = b
print(f"span {(it[-1, 2] - t0) / 1e3:.2f} us, sum of gaps {tot_gap:.2f} us")
