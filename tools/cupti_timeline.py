"""Device timeline of replayed solves via CUPTI activity records (tools/cupti/liblt_cupti.so):
exact kernel start/end per stream inside the CUDA graphs, no event overhead.

    python tools/cupti_timeline.py c2 [solves] [cold]

`cold`: a 256 MB L2 flush before every solve, as the bench's timed iterations.
"""
import ctypes
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nsol = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cold = len(sys.argv) > 3 and sys.argv[3] == "cold"
cup = ctypes.CDLL(os.path.join("tools", "cupti", "liblt_cupti.so"))
cup.lt_cupti_stop.argtypes = [ctypes.c_char_p]
ctx = Context(0)
s = make_config(cfg)
per = s.notes["periodic"]
d = ctx.upload(s)
eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
info = np.zeros(8, dtype=np.int64)
for _ in range(6):
    d.solve(per, eig.data_ptr(), 0, -1, info)
torch.cuda.synchronize()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda") if cold else None
assert cup.lt_cupti_start() == 0
for i in range(nsol):
    if cold:
        flush.fill_(float(i))
        torch.cuda.synchronize()
    d.solve(per, eig.data_ptr(), 0, -1, info)
torch.cuda.synchronize()
out = f"gpurun_out/cupti_{cfg}.csv"
cup.lt_cupti_stop(out.encode())
rows = [ln.split(",", 4) for ln in open(out).read().splitlines()[1:]]
rows = [(int(k), int(st), int(a), int(b), n) for k, st, a, b, n in rows if "at::native" not in n and "elementwise" not in n]
rows.sort(key=lambda r: r[2])
# split into solves at the spectrum's last kernel (pencils, or the box tridiagonal
# eigenvalues): the records after the second-to-last one form the last solve
ends = [i for i, r in enumerate(rows) if "k_pencil" in r[4] or "tridiag_eig" in r[4]]
last = rows[ends[-2] + 1:] if len(ends) >= 2 else rows
t0 = last[0][2]
streams = sorted({r[1] for r in last})
print(f"--- {cfg}{' (L2 flushed before each solve)' if cold else ''}: last solve, {len(last)} records, span {(last[-1][3] - t0) / 1e3:.1f} us")
for k, st, a, b, n in last:
    nm = n.split("(")[0].replace("void ", "").replace("lt::", "")
    print(f"  s{streams.index(st)} {(a - t0) / 1e3:8.2f} {(b - t0) / 1e3:8.2f} {(b - a) / 1e3:7.2f} us  {nm[:60]}")
