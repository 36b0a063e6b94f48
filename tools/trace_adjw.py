"""Per-K-block timeline of wide-adjoint CTA 0 (debug variant built with
-DCSR_DEBUG=1,ADJ_TIMELINE=1; CSR_TRACE=1).  clock64 stamps:
  0 MMA warp saw A stage ready (gen)     1 MMA warp saw B stage (issue start)
  2 generator warp 4 had its inputs      3 ... finished its math
  4 ... got its TMEM stage (aempty)      5 ... arrived on gen
  6 epilogue saw a chain complete        7 ... released the accumulator
usage: CSR_VARIANT=tl python tools/trace_adjw.py CFG
"""
import ctypes
import os
import sys

os.environ["CSR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_14080_b200 as P  # noqa: E402
from paper_2006_14080_b200 import _native  # noqa: E402
from harness.configs import make_problem  # noqa: E402

lib = _native.load()
lib.csr_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = make_problem(cfg, encoder=lambda img, s, k: np.zeros((k.shape[0], s.shape[0])))
op = P.DftOperator.build(prob.coords, P.ImageGrid(prob.nx, prob.ny), prob.sens,
                         n_frames=prob.n_frames)
rng = np.random.default_rng(0)
y = torch.from_numpy((rng.standard_normal((op.n_samples, op.n_coils)) + 1j * rng.standard_normal(
    (op.n_samples, op.n_coils))).astype(np.complex64)).cuda()
img = torch.empty(op.image_shape, dtype=torch.complex64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _native.call("csr_adjoint", op.plan, y.data_ptr(), img.data_ptr(), st)
torch.cuda.synchronize()
buf = np.zeros(4096 * 32, np.uint64)
lib.csr_debug_trace(op.plan, buf.ctypes.data, buf.size)
t = buf[65536:65536 + 8 * 1024].reshape(1024, 8).astype(np.int64)
n = int((t[:, 1] > 0).sum())
t0 = t[0, 2]
rel = (t - t0)
print(f"config {cfg}: {n} K blocks traced (cycles from block 0 inputs)")
print("  kb     gen_seen   issue   g_in   g_math  g_stage  g_arr  | d_issue  wait_gen  wait_b")
issue = t[:n, 1]
d_issue = np.diff(issue)
for i in range(n):
    r = rel[i]
    di = issue[i] - issue[i - 1] if i else 0
    wg = t[i, 0] - issue[i - 1] if i else 0       # gen seen after the previous issue
    wb = t[i, 1] - t[i, 0]                        # B wait after gen seen
    if i < 8 or (20 <= i < 28) or i > n - 4:
        print(f"{i:4d} {r[0]:10d} {r[1]:8d} {r[2]:7d} {r[3]:7d} {r[4]:8d} {r[5]:7d} | "
              f"{di:7d} {wg:8d} {wb:7d}")
print("median issue interval", np.median(d_issue), "mean", d_issue.mean(), "cycles")
wait_b = t[1:n, 1] - t[1:n, 0]
wait_g = t[1:n, 0] - issue[:-1]
print("mean wait for gen after previous issue", wait_g.mean(), " mean wait for B after gen", wait_b.mean())
g_math = t[:n, 3] - t[:n, 2]
g_stage = t[:n, 4] - t[:n, 3]
g_store = t[:n, 5] - t[:n, 4]
print("generator: math", np.median(g_math), "wait stage", np.median(g_stage), "store+arrive",
      np.median(g_store))
ch = [(i, t[i, 6], t[i, 7]) for i in range(n) if t[i, 6] > 0]
if ch:
    drains = [c[2] - c[1] for c in ch if c[2] > 0]
    print("chains", len(ch), "drain (acc_full seen -> acc_empty)", np.median(drains), "cycles")
    # chain ch's end: the epilogue's acc_full seen / release stamps are in row
    # ch * L (slot 6 / 7); the MMAs of block (ch + 1) * L wait for that release
    L = ch[1][0] - ch[0][0] if len(ch) > 1 else n
    stall, after = [], []
    for (i, full, empty) in ch[:-1]:
        nb = i + L
        if nb < n and empty > 0:
            stall.append(issue[nb] - issue[nb - 1])
            after.append(issue[nb] - empty)
    if stall:
        print(f"chain {L}: MMA gap at a chain end (issue of its first block after the previous one)",
              np.median(stall), "cycles; of it after the local release", np.median(after))

# drain rounds (rows 600 + chain, slots 0..3: each TMEM round's wait done)
dr = buf[65536 + 8 * 600: 65536 + 8 * 1024].reshape(-1, 8).astype(np.int64)
rows = [r for r in range(dr.shape[0]) if dr[r, 0] > 0]
if rows and ch:
    seen = {c: f for (c, f, e) in [(i // max(L, 1), full, empty) for (i, full, empty) in ch]}
    d = [[dr[r, 0] - seen.get(r, dr[r, 0])] + list(np.diff(dr[r, :4])) for r in rows if r in seen]
    if d:
        print("drain rounds (cycles: acc_full seen -> round 0 done, then per round):",
              np.median(np.array(d), axis=0))
