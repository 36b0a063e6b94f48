"""Per-CTA globaltimer trace of the A-stationary forward (CSR_TRACE=1)."""
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
x = torch.from_numpy(np.ascontiguousarray(prob.truth.astype(np.complex64))).cuda()
y = torch.empty((op.n_samples, op.n_coils), dtype=torch.complex64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _native.call("csr_forward", op.plan, x.data_ptr(), y.data_ptr(), st)
torch.cuda.synchronize()
buf = np.zeros(4096 * 32, np.uint64)
lib.csr_debug_trace(op.plan, buf.ctypes.data, buf.size)
tr = buf.reshape(4096, 32).astype(np.int64)
ctas = tr[tr[:, 0] > 0]
t0 = ctas[:, 0].min()
rel = lambda c: (ctas[:, c] - t0) / 1e3
print("CTAs", len(ctas))
for name, c in [("entry", 0), ("setup", 1), ("A0 loaded (epi)", 5), ("mma a_ready 0", 2), ("A1 loaded (epi)", 9), ("mma a_ready 1", 6), ("mma done", 3), ("epi done", 4)]:
    v = ctas[:, c]; v = (v[v > 0] - t0) / 1e3
    if len(v): print(f"{name:16s} n {len(v):4d} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
for i in range(8):
    v = rel(16 + i); w = rel(24 + i); print(f"tile {i} mma-commit med {np.median(v):7.2f}  epi-done med {np.median(w):7.2f} us")
