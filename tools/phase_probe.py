"""Phase breakdown of the device path under graph replay (Context.set_diagnostics(phase_timing=True)):
phase_l0 (L0 graph), phase_gap (host sync + planning + uploads), phase_post (post-L0 graph)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

for cfg in sys.argv[1:] or ["c2"]:
    ctx = Context(0)
    ctx.set_diagnostics(phase_timing=True)
    s = make_config(cfg)
    per = s.notes["periodic"]
    d = ctx.upload(s)
    eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
    info = np.zeros(8, dtype=np.int64)
    for _ in range(5):
        d.solve(per, eig.data_ptr(), 0, -1, info)
    ctx.set_stage_timing(False)  # resets totals
    n = 20
    for _ in range(n):
        d.solve(per, eig.data_ptr(), 0, -1, info)
    st = ctx.stage_times()
    print(cfg, " ".join(f"{k} {v[0] / n * 1e3:.1f}us" for k, v in sorted(st.items())))
