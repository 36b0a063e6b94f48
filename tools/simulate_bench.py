"""Time GPU simulate_kspace (f64) on a BASELINE config's shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from harness.configs import CONFIGS, golden_angle_coords
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg]
T, nx, ny, C = c["n_frames"], c["nx"], c["ny"], c["n_coils"]
rng = np.random.default_rng(0)
coords = np.concatenate([golden_angle_coords(c["spokes"], c["readout"], f * c["spokes"]) for f in range(T)])
sens = rng.standard_normal((C, nx, ny)) + 1j * rng.standard_normal((C, nx, ny))
img = rng.standard_normal((T, nx, ny)) + 1j * rng.standard_normal((T, nx, ny))
P.simulate_kspace(img[:1], sens, coords[:coords.shape[0] // T])
torch.cuda.synchronize(); t0 = time.perf_counter()
ds = P.simulate_kspace(img if T > 1 else img[0], sens, coords)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
flops = 8.0 * coords.shape[0] * C * nx * ny
print(f"config {cfg}: simulate_kspace f64 {dt*1e3:.1f} ms, {flops/dt/1e12:.2f} TFLOP/s f64 ({flops/1e12:.2f} TFLOP)")
