import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1408_3839_b200.api import Context
from paper_1408_3839_b200.system import make_config
cfg = sys.argv[1]
ctx = Context(0)
s = make_config(cfg); per = s.notes["periodic"]
d = ctx.upload(s)
eig = torch.empty(s.basis_count, dtype=torch.float64, device="cuda")
info = np.zeros(8, dtype=np.int64)
for _ in range(10): d.solve(per, eig.data_ptr(), 0, -1, info)
torch.cuda.synchronize()
# (a) event bracket like bench: e0 on idle GPU, then the host call
ms=[]; host=[]
for i in range(50):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); t0=time.perf_counter(); d.solve(per, eig.data_ptr(), 0, -1, info); host.append(time.perf_counter()-t0); e1.record(); e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(cfg, "event-bracketed solve %.1f us, host call %.1f us" % (np.median(ms)*1e3, np.median(host)*1e6))
# (b) back-to-back: 50 solves between two events
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(50): d.solve(per, eig.data_ptr(), 0, -1, info)
e1.record(); e1.synchronize()
print(cfg, "back-to-back per solve %.1f us" % (e0.elapsed_time(e1)*1e3/50))
