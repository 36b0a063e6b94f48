"""CUDA-event timing of the public forward / adjoint for a config (warm L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from paper_2006_14080_b200 import _native
from harness.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg, encoder=(lambda img, s, k: np.zeros((k.shape[0], s.shape[0])))
                    if cfg >= 2 else None)
op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens, n_frames=prob.n_frames)
dev = op.device
x = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(prob.truth, op.image_shape).astype(np.complex64))).to(dev)
y = torch.empty((op.n_samples, op.n_coils), dtype=torch.complex64, device=dev)
img = torch.empty(op.image_shape, dtype=torch.complex64, device=dev)
st = torch.cuda.current_stream().cuda_stream
res = {}
for name in ("forward", "adjoint"):
    ts = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if name == "forward":
            _native.call("csr_forward", op.plan, x.data_ptr(), y.data_ptr(), st)
        else:
            _native.call("csr_adjoint", op.plan, y.data_ptr(), img.data_ptr(), st)
        b.record(); b.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b) * 1e3)
    res[name] = np.median(ts)
import ctypes
fm, am, fn, an = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
_native.call("csr_plan_kernel_times", op.plan, ctypes.byref(fm), ctypes.byref(am), ctypes.byref(fn), ctypes.byref(an))
print(f"cfg {cfg} variant={os.environ.get('CSR_VARIANT','product')} narrow={os.environ.get('CSR_ADJ_NARROW','0')} exp={os.environ.get('CSR_EXP','0')} split={op.info()['split_k']} fwd {res['forward']:.1f} us adj {res['adjoint']:.1f} us"
      f" | kernels fwd {fm.value*1e3:.1f} adj {am.value*1e3:.1f} us", flush=True)
