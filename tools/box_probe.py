"""Dense box pencil probe: time lt_solve_box_dense on a random n x n pencil (and the
library path with LT_BOX_SYGVD=1). Usage: python tools/box_probe.py n [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3839_b200.api import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(1)
A = rng.uniform(-1, 1, (n, n))
H = 0.5 * (A + A.T)
B = rng.uniform(-1, 1, (n, n))
S = B @ B.T / n + np.eye(n)
ctx = Context(0)
ctx.set_stage_timing(True)
ev = ctx.solve_box_dense(H, S)  # warm-up (handles, workspaces, first-call costs)
base = dict(ctx.stage_times())
t = time.perf_counter()
for r in range(reps):
    ev = ctx.solve_box_dense(H, S)
dt = (time.perf_counter() - t) / reps
print("n", n, "wall ms/call %.3f (host H, S upload included)" % (dt * 1e3))
now = ctx.stage_times()
tot = 0.0
for k, (ms, nl) in sorted(now.items(), key=lambda kv: -kv[1][0]):
    d = (ms - base.get(k, (0.0, 0))[0]) * 1e3 / reps
    tot += d
    print("  %-14s %9.1f us/call" % (k, d))
print("  %-14s %9.1f us/call" % ("sum", tot))
if n <= 2048:
    import scipy.linalg as sl
    ref = sl.eigh(H, S, eigvals_only=True)
    print("max rel err %.3g" % (np.max(np.abs(ev - ref)) / np.max(np.abs(ref))))
