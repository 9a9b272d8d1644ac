"""Per-launch timeline of one eager solve with stage timing (main = 0, side branches 1-2)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

for cfg in sys.argv[1:] or ["c2"]:
    ctx = Context(0)
    s = make_config(cfg)
    per = s.notes["periodic"]
    d = ctx.upload(s)
    eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
    info = np.zeros(8, dtype=np.int64)
    for _ in range(3):
        d.solve(per, eig.data_ptr(), 0, -1, info)
    ctx.set_stage_timing(True)
    for _ in range(3):
        d.solve(per, eig.data_ptr(), 0, -1, info)
    tl = sorted(ctx.stage_timeline(), key=lambda r: r[2])
    print(f"--- {cfg}")
    for name, st, t0, t1 in tl:
        print(f"  s{st} {t0 * 1e3:8.1f} {t1 * 1e3:8.1f}  {(t1 - t0) * 1e3:7.1f} us  {name}")
    ctx.set_stage_timing(False)
