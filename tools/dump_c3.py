import sys, numpy as np
sys.path.insert(0, '.')
from paper_1408_3839_b200.system import make_config
from paper_1408_3839_b200.api import Context
ctx = Context(0)
s = make_config("c3")
ev = ctx.solve_core(s, False)
H, S = ctx.assemble_core(s, False)
np.savez_compressed("gpurun_out/c3_gpu.npz", H=H.dense(), S=S.dense(), ev=ev)
print("ok")
