"""Quick tensor-core operator check vs the f64 oracle (dev tool)."""
import sys, time
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2006_14080_b200 as P
from oracle import csrecon_oracle as O

def rc(rng, s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)

rng = np.random.default_rng(1)
cases = [(6, 4, 2, 25, 1), (16, 12, 3, 200, 1), (64, 64, 4, 4096, 1), (128, 128, 8, 16384, 1),
         (13, 7, 1, 64, 1), (24, 20, 3, 300, 4), (64, 48, 12, 1000, 1), (192, 192, 8, 4992, 2),
         (256, 256, 16, 8192, 1), (40, 40, 20, 500, 1)]
for nx, ny, C, m, T in cases:
    coords = rng.uniform(-0.5, 0.4999, size=(T * m, 2))
    sens = rc(rng, (C, nx, ny)) * 0.3
    img = rc(rng, (T, nx, ny)) if T > 1 else rc(rng, (nx, ny))
    y = rc(rng, (T * m, C))
    op = P.DftOperator.build(coords, P.ImageGrid(nx, ny), sens, n_frames=T)
    oo = O.Operator(coords, sens, T)
    t0 = time.time()
    f = op.forward(img.astype(np.complex64))
    a = op.adjoint(y.astype(np.complex64))
    fr = oo.forward(img); ar = oo.adjoint(y)
    ef = np.linalg.norm(f - fr) / np.linalg.norm(fr)
    ea = np.linalg.norm(a - ar) / np.linalg.norm(ar)
    print(f"{nx}x{ny} C={C} M={m} T={T} path={op.info()['gemm_path']} S={op.info()['split_k']} fwd {ef:.2e} adj {ea:.2e}", flush=True)
