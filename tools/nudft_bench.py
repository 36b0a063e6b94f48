"""Run the NUDFT forward/adjoint of a BASELINE config a few times (profiling driver)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from harness.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
# geometry only (coil maps, coordinates, phantom): the encode is skipped
prob = make_problem(cfg, encoder=lambda img, s, k: np.zeros((k.shape[0], s.shape[0])))
op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens, n_frames=prob.n_frames)
dev = op.device
x = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(prob.truth, op.image_shape).astype(np.complex64))).to(dev)
y = torch.empty((op.n_samples, op.n_coils), dtype=torch.complex64, device=dev)
img = torch.empty(op.image_shape, dtype=torch.complex64, device=dev)
st = torch.cuda.current_stream().cuda_stream
for i in range(reps):
    _native.call("csr_forward", op.plan, x.data_ptr(), y.data_ptr(), st)
    _native.call("csr_adjoint", op.plan, y.data_ptr(), img.data_ptr(), st)
torch.cuda.synchronize()
print("ok", op.info())
