"""Per-call wall times of the host API (Context.solve_core) to diagnose e2e overheads."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

ctx = Context(0)
for cfg in sys.argv[1:] or ["c1", "c2"]:
    s = make_config(cfg)
    per = s.notes["periodic"]
    ts = []
    for i in range(12):
        t0 = time.perf_counter()
        ctx.solve_core(s, per)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(cfg, " ".join(f"{t:.3f}" for t in ts))
