"""Loading the committed golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py)
and the parity checks against them."""
import glob
import os

import numpy as np

from paper_1408_3839_b200.system import LatticeSystem

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EPS = 2.0 ** -52


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    d = dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))
    s = LatticeSystem(b=float(d["b"]), L=tuple(int(x) for x in d["L"]), n=tuple(int(x) for x in d["n"]),
                      nbar=tuple(int(x) for x in d["nbar"]), quad_M=int(d["quad_M"]), nuc_pos=d["nuc_pos"],
                      nuc_charge=d["nuc_charge"], bf_center=d["bf_center"], bf_alpha=d["bf_alpha"],
                      bf_deg=d["bf_deg"], eps_ov=float(d["eps_ov"]), name=name)
    return s, bool(d["periodic"]), d


def ref_dense(d, which):
    """Full reference box matrix from the stored upper triangle (the reference's H is
    symmetric to d['H_sym_dev']; the lower triangle is mirrored)."""
    U = d[f"{which}_upper"]
    return U + np.triu(U, 1).T


def entries_ok(a, b, rel=1e-10, abs_frac=1e-14):
    """|a-b| <= 1e-10 |b| + 1e-14 max|b| (north-star entry rule)."""
    scale = float(np.max(np.abs(b)))
    bad = np.abs(a - b) > rel * np.abs(b) + abs_frac * scale
    return not bad.any()


def check_entries(H, S, d):
    """Compare assembled H, S (dense [N,N] or (kidx, blocks)) with the fixture; returns the
    measured discrepancies (||dH||, ||dS||) for the eigenvalue bound."""
    if bool(d["periodic"]):
        (kH, bH), (kS, bS) = H, S
        assert np.array_equal(kH, d["kidx"]) and np.array_equal(kS, d["kidx"])
        assert entries_ok(bH, d["H_blocks"]) and entries_ok(bS, d["S_blocks"])
        # exact ||dH_k||_2 per k-point: DFT of the block differences over the lattice
        L = tuple(int(x) for x in d["L"])
        return kspace_norms(bH - d["H_blocks"], d["kidx"], L), kspace_norms(bS - d["S_blocks"], d["kidx"], L)
    Hr, Sr = ref_dense(d, "H"), ref_dense(d, "S")
    lo = np.tril_indices(Hr.shape[0], -1)
    Hu, Su = np.triu(H) + np.triu(H, 1).T, np.triu(S) + np.triu(S, 1).T
    assert entries_ok(Hu, Hr) and entries_ok(Su, Sr)
    # the lower triangle must mirror the upper one to rounding (the reference's symmetry level)
    assert np.max(np.abs(H[lo] - H.T[lo])) <= 1e-13 * np.max(np.abs(Hr))
    return float(np.linalg.norm(H - Hr, 2)), float(np.linalg.norm(S - Sr, 2))


def kspace_norms(blocks, kidx, L):
    """||sum_k omega^{<j,k>} B_k||_2 for every lattice frequency j (lexicographic), i.e. the
    spectral norms of the Fourier blocks the pencils are solved on."""
    m0 = blocks.shape[1]
    A = np.zeros(L + (m0, m0), dtype=np.complex128)
    for i, k in enumerate(kidx):
        A[tuple(int(x) for x in k)] = blocks[i]
    F = np.fft.fftn(A, axes=(0, 1, 2)).reshape(-1, m0, m0)
    return np.linalg.norm(F, ord=2, axis=(1, 2))[:, None]


def eig_bound(d, dH, dS, solver_rel=1e-13):
    """First-order bound per eigenvalue: |dlambda_i| <= kappa_i (||dH|| + |lambda_i| ||dS||)
    with kappa_i = ||x_i||^2 (S-normalised reference eigenvectors), doubled, plus both
    solvers' backward errors (solver_rel ||.||) and the 1e-9 Hartree floor."""
    lam = d["eig"]
    kap = d["kappa"]
    if bool(d["periodic"]):
        L = tuple(int(x) for x in d["L"])
        nH = kspace_norms(d["H_blocks"], d["kidx"], L)
        nS = kspace_norms(d["S_blocks"], d["kidx"], L)
    else:
        nH = float(np.linalg.norm(ref_dense(d, "H"), 2))
        nS = float(np.linalg.norm(ref_dense(d, "S"), 2))
    return 1e-9 + 2.0 * kap * ((dH + np.abs(lam) * dS) + solver_rel * (nH + np.abs(lam) * nS))


def check_eigs(ev, d, dH=0.0, dS=0.0):
    ev = np.asarray(ev).reshape(d["eig"].shape)
    err = np.abs(ev - d["eig"])
    tol = eig_bound(d, dH, dS)
    assert np.all(err <= tol), (float(np.max(err / tol)), float(np.max(err)))
    return float(np.max(err)), float(np.max(err / tol))
