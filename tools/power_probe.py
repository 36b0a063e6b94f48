"""Sustained-load probe of one NUDFT GEMM: back-to-back launches for a few
seconds (the regime of a long ADMM step), per-launch device time and the
SM clock / power nvidia-smi reports meanwhile.

    python tools/power_probe.py CFG {forward,adjoint} [SECONDS]

With a debug variant (CSR_VARIANT, built with CSR_DEBUG=1) the profiling
flags CSR_FEXP / CSR_EXP switch parts of the kernel off, which separates the
energy of data movement from that of the MMAs under the power cap.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_14080_b200 as P  # noqa: E402
from paper_2006_14080_b200 import _dev, _native  # noqa: E402
from harness.configs import make_problem  # noqa: E402
from bench import ClockSampler  # noqa: E402

cfg, kind = int(sys.argv[1]), sys.argv[2]
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
prob = make_problem(cfg, encoder=lambda img, s, k: np.zeros((k.shape[0], s.shape[0])))
op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens,
                         n_frames=prob.n_frames)
dev = op.device
rng = np.random.default_rng(1)
x = torch.from_numpy((rng.standard_normal(op.image_shape) + 1j * rng.standard_normal(
    op.image_shape)).astype(np.complex64)).to(dev)
y = torch.from_numpy((rng.standard_normal((op.n_samples, op.n_coils)) + 1j *
                      rng.standard_normal((op.n_samples, op.n_coils))).astype(np.complex64)).to(dev)
ko = torch.empty((op.n_samples, op.n_coils), dtype=torch.complex64, device=dev)
img = torch.empty(op.image_shape, dtype=torch.complex64, device=dev)
st = _dev.stream_ptr(dev)


def once():
    if kind == "forward":
        _native.call("csr_forward", op.plan, x.data_ptr(), ko.data_ptr(), st)
    else:
        _native.call("csr_adjoint", op.plan, y.data_ptr(), img.data_ptr(), st)


for _ in range(3):
    once()
torch.cuda.synchronize()
clk = ClockSampler(0)
clk.start()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
n = 0
t0 = time.perf_counter()
a.record()
while time.perf_counter() - t0 < secs:
    for _ in range(4):
        once()
        n += 1
    torch.cuda.synchronize()
b.record()
b.synchronize()
c = clk.stop()
ms = a.elapsed_time(b) / n
flops = 8.0 * op.n_coils * op.m_per_frame * op.nx * op.ny * op.n_frames
print(f"cfg {cfg} {kind} variant={os.environ.get('CSR_VARIANT', 'product')} "
      f"fexp={os.environ.get('CSR_FEXP', '0')} exp={os.environ.get('CSR_EXP', '0')}: "
      f"{ms:.3f} ms/launch over {n} launches = {flops / ms / 1e9:.1f} TF/s algorithmic; "
      f"clocks {c}", flush=True)
