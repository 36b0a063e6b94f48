"""cProfile of admm_reconstruct (host side) for a config, after warm-up."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_14080_b200 as P
from harness.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_problem(cfg)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
data, sens = pin(prob.data), pin(prob.sens)
traj = P.Trajectory(prob.coords, prob.coords.shape[0], 1)
ds = P.KSpaceDataset(data, traj, n_frames=prob.n_frames)
params = P.ReconParams(**prob.params)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    img, rep = P.admm_reconstruct(ds, sens, params, compute_objectives=False)
    torch.cuda.synchronize(); print(f"call {1e3*(time.perf_counter()-t0):.2f} ms timing {rep.timing}")
pr = cProfile.Profile()
pr.enable()
img, rep = P.admm_reconstruct(ds, sens, params, compute_objectives=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
