"""Phase timestamps of the fused CG tail (CSR_TRACE=1): block 0 and the last block."""
import ctypes, os, sys
os.environ["CSR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from harness.configs import make_problem
lib = _native.load()
lib.csr_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
prob = make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
traj = P.Trajectory(prob.coords, prob.coords.shape[0], 1)
ds = P.KSpaceDataset(prob.data, traj, n_frames=prob.n_frames)
params = P.ReconParams(**dict(prob.params, admm_max_iters=3))
import paper_2006_14080_b200.solver as S
sh = S._Shard(ds, prob.sens, 1, "auto", torch.device("cuda", 0))
rho = torch.empty(sh.op.image_shape, dtype=torch.complex64, device="cuda")
log = (_native.IterLog * 3)()
stats = _native.RunStats()
lib.csr_admm_run(sh.op.plan, ctypes.byref(params.native()), sh.data.data_ptr(), rho.data_ptr(),
                 log, ctypes.byref(stats), torch.cuda.current_stream().cuda_stream, None)
torch.cuda.synchronize()
buf = np.zeros(4096 * 32, np.uint64)
lib.csr_debug_trace(sh.op.plan, buf.ctypes.data, buf.size)
st = buf[100000:100032].astype(np.int64)
b0, bl = st[:8], st[16:24]
t0 = min(b0[0], bl[0])
names = ["start", "A done", "barrier1", "totals", "B done", "barrier2", "totals2", "C done"]  # cluster: 2,5 unused
for n, a, b in zip(names, b0, bl):
    print(f"{n:10s} block0 {(a - t0) / 1e3:7.3f} us   last {(b - t0) / 1e3:7.3f} us")
