"""One host-API solve of each named BASELINE config (no torch), for compute-sanitizer:
    compute-sanitizer --tool memcheck python tools/sanitize_solve.py c1 c2 c3
Runs each system three times (eager, capture, graph replay) so the graph paths are covered."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1408_3839_b200.api import Context  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:] or ["c1", "c2"]:
    s = make_config(name)
    per = s.notes["periodic"]
    for _ in range(3):
        ev = ctx.solve_core(s, per)
    print(name, "ok", float(ev.min()), float(ev.max()), flush=True)
ctx.close()
