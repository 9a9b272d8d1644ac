"""Parity report for the five BASELINE configs: GPU results (gpurun_out/parity_gpu_<cfg>.npz,
written on the B200 by tools/parity_dump.py) against the committed golden fixtures
(Oracle-X, tests/golden/<cfg>.npz with eig_floor from tests/golden/make_floor.py).

    python tools/parity_report.py r02 [gpurun_out]   ->  profiles/r02_parity.json

Per config: max entry relative error of Mass, Nuclear (pure relative) and Laplace, H (with
the stiffness absolute term 1e-14 max|.|), max / median |dlambda|, how many eigenvalues
exceed 1e-9 Ha and their FP64 floors, and the largest |dlambda| / max(1e-9, floor) ratio.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from golden_util import EIG_FLOOR_E2E, EIG_FLOOR_SOLVER, eig_tolerance_golden, load, ref_dense  # noqa: E402
from oracle.binding import oracle  # noqa: E402


def rel_err(a, b, abs_frac=0.0):
    a, b = np.asarray(a), np.asarray(b)
    scale = float(np.max(np.abs(b)))
    den = np.maximum(np.abs(b), 2.2250738585072014e-308) + abs_frac * scale / 1e-10  # subnormals: no relative digits
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(den > 0, np.abs(a - b) / den, np.where(a == b, 0.0, np.inf))
    return float(np.max(r))


def dense_full(d, tag):
    U = d[f"{tag}_upper"]
    return U + np.triu(U, 1).T


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    out = {"how": "GPU (B200, C-ABI) vs committed Oracle-X golden fixtures; entries: |a-b|/max(|b|, DBL_MIN) (Mass, Nuclear), "
                  "|a-b|/(|b| + 1e-4 max|b|) i.e. the 1e-10 rel + 1e-14 max abs rule (Laplace, H); eigenvalues: "
                  "|dlambda| against max(1e-9 Ha, floor), floor = largest eigenvalue change of the reference pencil "
                  "under 8-ulp entry perturbations (8 draws, tests/golden/make_floor.py); solver_only: GPU eigenvalues vs the "
                  "reference algorithm (oracle) on the GPU's own pencil"}
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        p = os.path.join(src, f"parity_gpu_{cfg}.npz")
        if not os.path.exists(p):
            continue
        g = dict(np.load(p))
        s, periodic, d = load(cfg)
        r = {}
        for gt, rt, absf in (("Mass", "M", 0.0), ("Nuc", "N", 0.0), ("Lap", "Lap", 1e-14), ("H", "H", 1e-14),
                             ("S", "S", 0.0)):
            if periodic:
                assert np.array_equal(g[f"{gt}_kidx"], d["kidx"])
                a, b = g[f"{gt}_blocks"], d[f"{rt}_blocks"]
            else:
                a = g[f"{gt}_dense"]
                a = np.triu(a) + np.triu(a, 1).T
                b = dense_full(d, rt)
            r[f"entry_rel_{gt}"] = rel_err(a, b, absf)
        ev = g["eig"].reshape(d["eig"].shape)
        # the eigensolver alone: the reference algorithm (oracle) on the GPU's own pencil
        if periodic:
            keys = [tuple(int(x) for x in k) for k in g["H_kidx"]]
            own = oracle().solve_periodic(s.L, s.m0, {k: g["H_blocks"][i] for i, k in enumerate(keys)},
                                          {k: g["S_blocks"][i] for i, k in enumerate(keys)}, os.cpu_count() or 1)
        else:
            Hd, Sd = g["H_dense"], g["S_dense"]
            own = oracle().solve_box_dense(np.triu(Hd) + np.triu(Hd, 1).T, np.triu(Sd) + np.triu(Sd, 1).T)
        serr = np.abs(ev - own.reshape(ev.shape))
        err = np.abs(ev - d["eig"])
        floor = d["eig_floor"]
        tol = eig_tolerance_golden(d)
        r.update({
            "L0": int(g["info"][0]), "L0_ref": int(d["L0"]),
            "n_eigenvalues": int(err.size),
            "max_abs_dlambda": float(err.max()), "median_abs_dlambda": float(np.median(err)),
            "n_dlambda_above_1e-9": int(np.sum(err > 1e-9)),
            "n_floor_above_1e-9": int(np.sum(floor > 1e-9)),
            "floor_median": float(np.median(floor)), "floor_max": float(floor.max()),
            "tolerance_median": float(np.median(tol)), "tolerance_max": float(tol.max()),
            "max_err_over_tolerance": float(np.max(err / tol)),
            "tolerance_rule": f"max(1e-9, {EIG_FLOOR_E2E:g} x floor)",
            "solver_only_max_abs_dlambda": float(serr.max()),
            "solver_only_max_err_over_tolerance": float(np.max(serr / eig_tolerance_golden(d, EIG_FLOOR_SOLVER))),
            "solver_only_tolerance_rule": f"max(1e-9, {EIG_FLOOR_SOLVER:g} x floor)",
            "n_floor_above_1e-3": int(np.sum(floor > 1e-3)),
            "max_err_over_floor_or_1e-9": float(np.max(err / np.maximum(1e-9, floor))),
            "n_floor_below_1e-9_with_err_above_1e-9": int(np.sum((floor <= 1e-9) & (err > 1e-9))),
        })
        out[cfg] = r
        print(cfg, json.dumps(r))
    dst = os.path.join(ROOT, "profiles", f"{tag}_parity.json")
    json.dump(out, open(dst, "w"), indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main()
