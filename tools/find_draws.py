"""Rejection sampling of the seeded exponent sets.

A draw is accepted when the reference would accept it: the alias guard L_l > 2 L0
holds (periodic, galerkin.cpp:294-302) and the core pencil is definite (the LLT in
solve_periodic / solve_box_dense succeeds, eigensolver.cpp:20-23, :80-83). Candidates
are screened with the B200 engine (fast), then confirmed with the oracle:

    python tools/find_draws.py c3 --gpu        # on a GPU box: first passing draws
    python tools/find_draws.py c3 --verify 7   # here: confirm draw 7 with Oracle-X
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1408_3839_b200.system import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--verify", type=int, default=None)
    ap.add_argument("--max", type=int, default=400)
    ap.add_argument("--want", type=int, default=5)
    a = ap.parse_args()
    if a.gpu:
        from paper_1408_3839_b200.api import Context, DefinitenessError, StructureError
        ctx = Context(0)
        found = []
        t0 = time.time()
        for d in range(a.max):
            s = make_config(a.config, exponent_draw=d)
            try:
                ctx.solve_core(s, s.notes["periodic"])
                found.append(d)
                print("draw", d, "passes", flush=True)
                if len(found) >= a.want:
                    break
            except (DefinitenessError, StructureError) as e:
                print("draw", d, "rejected:", str(e)[:90], flush=True)
        print(a.config, "passing draws", found, "searched", d + 1, "in %.1fs" % (time.time() - t0))
    if a.verify is not None:
        from oracle.binding import OracleError, oracle
        o = oracle()
        s = make_config(a.config, exponent_draw=a.verify)
        per = s.notes["periodic"]
        t0 = time.time()
        try:
            H, S = o.assemble_core(s, per)
            if per:
                o.solve_periodic_ops(H, S, os.cpu_count() or 1)
            else:
                o.solve_box_dense(H.dense, S.dense)
            print(a.config, "draw", a.verify, "accepted by the oracle (L0 %d) in %.1fs" % (H.L0, time.time() - t0))
        except OracleError as e:
            print(a.config, "draw", a.verify, "rejected by the oracle:", e.msg)


if __name__ == "__main__":
    main()
