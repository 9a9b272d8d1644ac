"""Host-side time split of the device-resident solve (Context.set_diagnostics(host_timing=True)) and the Python-level
per-call wall time, to separate host overhead from device time."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = Context(0)
s = make_config(cfg)
per = s.notes["periodic"]
d = ctx.upload(s)
eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
info = np.zeros(8, dtype=np.int64)
for _ in range(10):
    d.solve(per, eig.data_ptr(), 0, -1, info)
ctx.set_diagnostics(host_timing=True)  # after warm-up: graph replays only
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    d.solve(per, eig.data_ptr(), 0, -1, info)
    ts.append(time.perf_counter() - t0)
print(f"{cfg}: python-level solve {np.median(ts) * 1e6:.1f} us (median of 200)")
ctx.close()
