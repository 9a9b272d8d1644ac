import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1408_3839_b200.system import LatticeSystem  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import oracle as _o
    return _o()


@pytest.fixture(scope="session")
def ctx():
    from paper_1408_3839_b200.api import Context
    c = Context(0)
    yield c
    c.close()


# ---------------------------------------------------------------------------
# small systems shaped like the reference's tests (test_galerkin.cpp:23-34)
# ---------------------------------------------------------------------------
def chain_system(L, alpha, n=8, nbar=8, M=10, b=8.0) -> LatticeSystem:
    alphas = alpha if isinstance(alpha, (list, tuple)) else [alpha]
    return LatticeSystem(b=b, L=(L, 1, 1), n=n, nbar=nbar, quad_M=M, nuc_pos=[(0.0, 0.0, 0.0)], nuc_charge=[1.0],
                         bf_center=[(0.0, 0.0, 0.0)] * len(alphas), bf_alpha=alphas, name=f"chain{L}")


def two_nuclei_system(L=(6, 1, 1), n=(16, 8, 8), nbar=None, M=8, b=2.0, alphas=(0.9, 2.5, 0.6, 4.0),
                      deg=None) -> LatticeSystem:
    pos = [(-0.5, 0.1, 0.0), (0.5, 0.0, -0.2)]
    centers = [pos[i % 2] for i in range(len(alphas))]
    return LatticeSystem(b=b, L=L, n=n, nbar=nbar if nbar is not None else n, quad_M=M, nuc_pos=pos,
                         nuc_charge=[1.0, 2.0], bf_center=centers, bf_alpha=list(alphas), bf_deg=deg,
                         name="two_nuclei")


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(1e-300, float(np.max(np.abs(b))))
    return float(np.max(np.abs(a - b))) / scale


def eig_tolerance(oracle, periodic, H, S, ev_ref, trials=3, seed=7, ulps=32):
    """Per-eigenvalue parity bound: max(1e-9 Hartree, 2x the eigenvalue's summation-order floor).

    The floor is measured on the reference pencil itself: perturb every H and S entry by
    a random relative amount of up to `ulps` units of rounding (32 ulps: the measured
    entry-level spread between two FP64 summation orders over the ~10^3-10^4-term grid
    contractions, e.g. 16 ulps for c3), re-solve with the oracle and take each
    eigenvalue's largest change over `trials` perturbations. Two FP64 implementations
    whose entries differ only in summation order cannot agree more closely than that.
    Well-conditioned eigenvalues keep the 1e-9 bound; the near-linear-dependent BASELINE
    bases (cond(S) up to ~1e9-1e13) have a few eigenvalues whose floor is far above it.
    Returns an array shaped like ev_ref.
    """
    rng = np.random.default_rng(seed)
    eps = ulps * 2.0 ** -52
    worst = np.zeros_like(np.asarray(ev_ref, dtype=np.float64))
    for _ in range(trials):
        if periodic:
            L = H.L

            def pert(g):
                out = {}
                for k, v in g.items():
                    m = tuple((L[l] - k[l]) % L[l] for l in range(3))
                    if m in out:
                        out[k] = out[m].T.copy()
                        continue
                    p = v * (1 + eps * rng.uniform(-1.0, 1.0, size=v.shape))
                    out[k] = 0.5 * (p + p.T) if m == k else p
                return out

            ev = oracle.solve_periodic(L, H.m0, pert(H.gen_dict()), pert(S.gen_dict()))
        else:
            def pert(a):
                p = a * (1 + eps * rng.uniform(-1.0, 1.0, size=a.shape))
                return np.triu(p) + np.triu(p, 1).T

            ev = oracle.solve_box_dense(pert(H.dense), pert(S.dense))
        worst = np.maximum(worst, np.abs(ev - ev_ref))
    return np.maximum(1e-9, 2.0 * worst)


def entries_close(gpu, ref, rel=1e-10, abs_frac=1e-14, scale=None):
    """North-star entry rule: |a-b| <= rel |b| + abs_frac max|H|."""
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    s = float(np.max(np.abs(ref))) if scale is None else scale
    bad = np.abs(gpu - ref) > rel * np.abs(ref) + abs_frac * s
    return not bad.any(), float(np.max(np.abs(gpu - ref) / (np.abs(ref) + abs_frac * s / rel + 1e-300)))
