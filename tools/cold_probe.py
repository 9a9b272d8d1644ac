"""Host-side time split of the cold host-API call (a fresh system every call: eager launches, L0
host round trip) with Context.set_diagnostics(host_timing=True)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from bench import scanned  # noqa: E402
from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
ctx = Context(0)
s = make_config(cfg)
per = s.notes["periodic"]
out = np.empty(s.basis_count)
for i in range(5):
    ctx.solve_core(scanned(s, 100 + i), per, out=out)
ctx.set_diagnostics(host_timing=True)
systems = [scanned(s, i) for i in range(40)]
ts = []
for x in systems:
    t0 = time.perf_counter()
    ctx.solve_core(x, per, out=out)
    ts.append(time.perf_counter() - t0)
print(f"{cfg}: cold host-API call {np.median(ts) * 1e6:.1f} us (median of {len(ts)})")
ctx.close()
