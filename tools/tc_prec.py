import sys, os
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2006_14080_b200 as P
from oracle import csrecon_oracle as O
rng = np.random.default_rng(1)
nx, ny, C, m = 256, 256, 16, 8192
coords = rng.uniform(-0.5, 0.4999, size=(m, 2))
sens = (rng.standard_normal((C, nx, ny)) + 1j * rng.standard_normal((C, nx, ny))) * 0.3
y = rng.standard_normal((m, C)) + 1j * rng.standard_normal((m, C))
ar = O.Operator(coords, sens).adjoint(y)
op = P.DftOperator.build(coords, P.ImageGrid(nx, ny), sens)
a = op.adjoint(y.astype(np.complex64))
print(os.environ.get("CSR_TC_SPLIT"), os.environ.get("CSR_DISABLE_TC"), op.info(), np.linalg.norm(a - ar) / np.linalg.norm(ar), flush=True)
