import sys, numpy as np
sys.path.insert(0, '.')
from paper_1408_3839_b200.api import Context
m0, cnt, cplx = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(m0)
A = rng.standard_normal((cnt, m0, m0)) + (1j if cplx else 0) * rng.standard_normal((cnt, m0, m0))
H = A + np.conj(np.transpose(A, (0, 2, 1)))
S = np.stack([np.eye(m0)] * cnt) * 3.0 + 0j
ctx = Context(0)
ev = ctx.pencil_eig(H, S)
import scipy.linalg as sl
print(m0, cnt, cplx, "err", max(np.abs(ev[j] - sl.eigh(H[j], S[j], eigvals_only=True)).max() for j in range(cnt)), flush=True)
