"""Break down one admm_reconstruct call (plan build vs solve) for a config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from harness.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg)
traj = P.Trajectory(prob.coords, prob.coords.shape[0], 1)
ds = P.KSpaceDataset(prob.data, traj, n_frames=prob.n_frames)
params = P.ReconParams(**prob.params)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens, n_frames=prob.n_frames)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del op
    img, rep = P.admm_reconstruct(ds, prob.sens, params, compute_objectives=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms  admm_reconstruct {1e3*(t2-t1):.1f} ms  timing {rep.timing}", flush=True)
