"""Per-K-block timeline of adjoint CTA 0 (CSR_TRACE=1, variant built with
-DADJ_TIMELINE=1): when the MMA issuer
saw block i generated, when generator warp 4 had its inputs, got its TMEM
stage, and finished writing it."""
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
op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens, n_frames=prob.n_frames)
y = torch.from_numpy(np.ascontiguousarray(prob.data.astype(np.complex64))).cuda()
img = torch.empty(op.image_shape, dtype=torch.complex64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _native.call("csr_adjoint", op.plan, y.data_ptr(), img.data_ptr(), st)
torch.cuda.synchronize()
buf = np.zeros(4096 * 32, np.uint64)
lib.csr_debug_trace(op.plan, buf.ctypes.data, buf.size)
t = buf[65536:65536 + 1024].reshape(256, 4).astype(np.int64)
n = int((t[:, 0] > 0).sum())
t0 = t[0, 1]
print("kb  mma_saw_gen  gen_inputs  gen_got_stage  gen_done   (us from gen kb0 inputs)  d(mma)")
prev = None
for i in range(n):
    r = (t[i] - t0) / 1e3
    d = (t[i, 0] - prev) / 1e3 if prev is not None else 0
    prev = t[i, 0]
    if i < 6 or 20 <= i < 30 or i > n - 4:
        print(f"{i:3d} {r[0]:10.3f} {r[1]:10.3f} {r[2]:10.3f} {r[3]:10.3f}   {d:7.3f}")
dm = np.diff(t[:n, 0]) / 1e3
print("median mma step us", np.median(dm), "mean", dm.mean())
