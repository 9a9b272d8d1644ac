"""Augment the committed golden fixtures with (run here, where the oracle is built):

* ``eig_floor`` — each reference eigenvalue's FP64 floor: the largest change of that
  eigenvalue when every H and S entry of the reference pencil is perturbed by a random
  relative amount of up to ``ULPS`` units of rounding (symmetry kept), re-solved by the
  same oracle, over ``TRIALS`` independent draws. Two FP64 implementations whose entries
  differ only in summation order cannot agree more closely than this; well-conditioned
  eigenvalues sit far below 1e-9 Ha, the near-linearly-dependent BASELINE bases have some
  eigenvalues above it.
* ``N_upper`` / ``N_blocks`` (and ``Lap_*``, ``M_*``) — the reference Nuclear, Laplace and
  Mass operators on their own, so the entry rules can hold nuclear and mass entries to a
  pure 1e-10 relative and keep the absolute term for the cancelling stiffness entries only.

    python tests/golden/make_floor.py [names...]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_util import load, names as all_names, ref_dense  # noqa: E402
from oracle.binding import oracle, reference  # noqa: E402

ULPS = 8
TRIALS = 8
SEED = 20260


def floor_box(o, H, S, ev_ref, rng):
    eps = ULPS * 2.0 ** -52
    worst = np.zeros_like(ev_ref)
    for _ in range(TRIALS):
        def pert(a):
            p = a * (1 + eps * rng.uniform(-1.0, 1.0, size=a.shape))
            return np.triu(p) + np.triu(p, 1).T
        ev = o.solve_box_dense(pert(H), pert(S))
        worst = np.maximum(worst, np.abs(ev - ev_ref))
    return worst


def floor_periodic(o, L, m0, kidx, Hb, Sb, ev_ref, rng):
    eps = ULPS * 2.0 ** -52
    worst = np.zeros_like(ev_ref)
    keys = [tuple(int(x) for x in k) for k in kidx]
    for _ in range(TRIALS):
        def pert(blocks):
            g = {k: blocks[i] for i, k in enumerate(keys)}
            out = {}
            for k, v in g.items():
                m = tuple((L[l] - k[l]) % L[l] for l in range(3))
                if m in out:  # circulant symmetry B_{-k} = B_k^T is kept exactly
                    out[k] = out[m].T.copy()
                    continue
                p = v * (1 + eps * rng.uniform(-1.0, 1.0, size=v.shape))
                out[k] = 0.5 * (p + p.T) if m == k else p
            return out
        ev = o.solve_periodic(L, m0, pert(Hb), pert(Sb), os.cpu_count() or 1).reshape(ev_ref.shape)
        worst = np.maximum(worst, np.abs(ev - ev_ref))
    return worst


def augment(name):
    t0 = time.time()
    s, periodic, d = load(name)
    src = str(d["source"])
    impl = reference() if src.startswith("Oracle-R") else oracle()
    o = oracle()
    rng = np.random.default_rng(SEED)
    ev_ref = np.asarray(d["eig"], dtype=np.float64)
    L = tuple(int(x) for x in d["L"])
    m0 = int(d["bf_alpha"].shape[0])
    if periodic:
        d["eig_floor"] = floor_periodic(o, L, m0, d["kidx"], d["H_blocks"], d["S_blocks"], ev_ref, rng)
    else:
        d["eig_floor"] = floor_box(o, ref_dense(d, "H"), ref_dense(d, "S"), ev_ref, rng)
    d["eig_floor_ulps"] = ULPS
    d["eig_floor_trials"] = TRIALS
    for kind, tag in (("nuclear", "N"), ("laplace", "Lap"), ("mass", "M")):
        op = impl.assemble(s, periodic, kind)
        if periodic:
            assert np.array_equal(op.kidx, d["kidx"])
            d[f"{tag}_blocks"] = op.blocks
        else:
            d[f"{tag}_upper"] = np.triu(op.dense)
        impl.free(op)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    f = d["eig_floor"]
    print(f"{name}: floor median {np.median(f):.2e} max {np.max(f):.2e}, above 1e-9: {int(np.sum(f > 1e-9))}"
          f"/{f.size}, {time.time() - t0:.1f}s", flush=True)


def main():
    for name in sys.argv[1:] or all_names():
        augment(name)


if __name__ == "__main__":
    main()
