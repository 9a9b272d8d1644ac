"""GPU side of the parity report: solve the five BASELINE configs through the C-ABI and
dump eigenvalues plus the separately assembled Laplace, Nuclear, Mass and core H, S to
gpurun_out/parity_gpu_<cfg>.npz. tools/parity_report.py compares them with Oracle-X here
(where the oracle and the committed fixtures live) and writes profiles/rNN_parity.json.

    python tools/parity_dump.py [c1 c2 ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402


def payload(op):
    if op.periodic:
        k, b = op.blocks()
        return {"kidx": k, "blocks": b}
    return {"dense": np.ascontiguousarray(op.dense())}


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    ctx = Context(0)
    for name in names:
        s = make_config(name)
        per = s.notes["periodic"]
        info = np.zeros(8, dtype=np.int64)
        ev = ctx.solve_core(s, per, info)
        d = {"eig": ev, "info": info}
        H, S = ctx.assemble_core(s, per)
        for tag, op in (("H", H), ("S", S), ("Lap", ctx.assemble(s, per, "laplace")),
                        ("Nuc", ctx.assemble(s, per, "nuclear")), ("Mass", ctx.assemble(s, per, "mass"))):
            for k, v in payload(op).items():
                d[f"{tag}_{k}"] = v
        np.savez_compressed(os.path.join(out, f"parity_gpu_{name}.npz"), **d)
        print(name, "L0", int(info[0]), "eig", ev.shape, flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
