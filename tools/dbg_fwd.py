import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2006_14080_b200 as P
from oracle import csrecon_oracle as O
rng = np.random.default_rng(1)
for (nx, ny, C, M) in [(8, 6, 3, 50), (16, 16, 4, 300), (64, 64, 4, 4096), (128, 128, 8, 16384)]:
    coords = rng.uniform(-0.5, 0.4999, size=(M, 2))
    sens = (rng.standard_normal((C, nx, ny)) + 1j * rng.standard_normal((C, nx, ny)))
    img = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
    op = P.DftOperator.build(coords, P.ImageGrid(nx, ny), sens)
    got = op.forward(img.astype(np.complex64))
    ref = O.forward_direct(img, sens, coords) if M <= 4096 else O.Operator(coords, sens, 1).forward(img)
    err = np.abs(got - ref)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    bad = np.where(err.max(axis=1) > 1e-3 * np.abs(ref).max())[0]
    print(nx, ny, C, M, "rel", rel, "bad rows", len(bad), bad[:10], op.info().get('split_k'))
