"""Per-CTA globaltimer trace of the adjoint (CSR_TRACE=1)."""
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
tr = buf.reshape(4096, 32).astype(np.int64)
ctas = tr[tr[:, 0] > 0]
t0 = ctas[:, 0].min()
def rel(c):
    v = ctas[:, c]; v = v[v > 0]; return (v - t0) / 1e3
print("CTAs", len(ctas))
print("mma done med", np.median(rel(1)))
for ch in range(4):
    v = rel(12 + ch)
    if len(v): print(f"chain {ch} committed med {np.median(v):7.2f}")
for i in range(4):
    print(f"kb {8+i}: tma issued {np.median(rel(24+i)):7.2f}  mma saw full {np.median(rel(2+2*i)):7.2f}  gen {np.median(rel(3+2*i)):7.2f}  gen4 done {np.median(rel(16+i)):7.2f} gen8 done {np.median(rel(20+i)):7.2f}")
dt = (ctas[:, 1] - ctas[:, 0]).astype(float)
dc = (ctas[:, 31] - ctas[:, 30]).astype(float)
ok = (dt > 0) & (dc > 0)
print("SM clock during adjoint (MHz): median", np.median(dc[ok] / dt[ok] * 1e3))
# per-CTA phases: start -> MMA loop done (tr[1]) -> end after the coil combine (tr[28])
e = ctas[:, 28]
okp = e > 0
if okp.any():
    print("per CTA (us): start->mma done med", np.median((ctas[okp, 1] - ctas[okp, 0]) / 1e3),
          " mma done->end med", np.median((e[okp] - ctas[okp, 1]) / 1e3),
          " first start->last end", (e[okp].max() - ctas[okp, 0].min()) / 1e3)
