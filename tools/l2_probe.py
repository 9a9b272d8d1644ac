"""Cold- vs warm-L2 cost of one device-resident solve (the bench's `value` timing without and with the 256 MB
flush between calls), plus the Python-level call time: how much of the bench number is cold HBM latency."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
ctx = Context(0)
s = make_config(cfg)
per = s.notes["periodic"]
d = ctx.upload(s)
eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
info = np.zeros(8, dtype=np.int64)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(10):
    d.solve(per, eig.data_ptr(), 0, -1, info)
torch.cuda.synchronize()
for mode in ("warm", "cold", "warm", "cold"):
    ms = []
    for i in range(100):
        if mode == "cold":
            flush.fill_(float(i))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        d.solve(per, eig.data_ptr(), 0, -1, info)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"{cfg} {mode}: mean {np.mean(ms) * 1e3:.1f} us  median {np.median(ms) * 1e3:.1f} us")
ts = []
for _ in range(100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.solve(per, eig.data_ptr(), 0, -1, info)
    ts.append(time.perf_counter() - t0)
print(f"{cfg}: host time of the call (returns after the graph launch + readback wait) median {np.median(ts) * 1e6:.1f} us")
ctx.close()
