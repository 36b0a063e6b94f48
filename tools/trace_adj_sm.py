"""Per-CTA adjoint trace (CSR_TRACE=1): duration split and per-SM gaps."""
import ctypes, os, sys
os.environ["CSR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from harness.configs import make_problem
lib = _native.load()
lib.csr_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg, encoder=(lambda i, s, c: P.simulate_kspace(i, s, c).data) if cfg >= 2 else None)
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
print("CTAs", len(ctas), "kernel span us", (ctas[:, 28].max() - t0) / 1e3)
mma = (ctas[:, 1] - ctas[:, 0]) / 1e3
tail = (ctas[:, 28] - ctas[:, 1]) / 1e3
print(f"start->mma done: med {np.median(mma):.2f} min {mma.min():.2f} max {mma.max():.2f} us")
print(f"mma done->CTA end: med {np.median(tail):.2f} min {tail.min():.2f} max {tail.max():.2f} us")
gaps = []
for sm in np.unique(ctas[:, 29]):
    c = ctas[ctas[:, 29] == sm]
    c = c[np.argsort(c[:, 0])]
    gaps += list((c[1:, 0] - c[:-1, 28]) / 1e3)
if gaps:
    g = np.array(gaps)
    print(f"per-SM gap between CTAs: med {np.median(g):.2f} max {g.max():.2f} us, n {len(g)}")
    print("SMs used", len(np.unique(ctas[:, 29])), "CTAs per SM max", np.bincount(ctas[:, 29]).max())
