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


DBL_MIN = 2.2250738585072014e-308  # below it FP64 has no relative precision (subnormals)


def entries_ok(a, b, rel=1e-10, abs_frac=1e-14):
    """|a-b| <= rel max(|b|, DBL_MIN) + abs_frac max|b|. The north-star entry rule is 1e-10
    relative; the absolute term is for entries that cancel (stiffness and
    H = 0.5 Laplace - Nuclear); Mass and Nuclear entries are sums of positive terms and are
    checked with abs_frac = 0 (pure relative; subnormal entries carry no relative digits)."""
    scale = float(np.max(np.abs(b)))
    bad = np.abs(a - b) > rel * np.maximum(np.abs(b), DBL_MIN) + abs_frac * scale
    return not bad.any()


def check_entries(H, S, d):
    """Compare assembled H, S (dense [N,N] or (kidx, blocks)) with the fixture; returns the
    measured discrepancies (||dH||, ||dS||) for the eigenvalue bound."""
    if bool(d["periodic"]):
        (kH, bH), (kS, bS) = H, S
        assert np.array_equal(kH, d["kidx"]) and np.array_equal(kS, d["kidx"])
        assert entries_ok(bH, d["H_blocks"]) and entries_ok(bS, d["S_blocks"], abs_frac=0.0)
        # exact ||dH_k||_2 per k-point: DFT of the block differences over the lattice
        L = tuple(int(x) for x in d["L"])
        return kspace_norms(bH - d["H_blocks"], d["kidx"], L), kspace_norms(bS - d["S_blocks"], d["kidx"], L)
    Hr, Sr = ref_dense(d, "H"), ref_dense(d, "S")
    lo = np.tril_indices(Hr.shape[0], -1)
    Hu, Su = np.triu(H) + np.triu(H, 1).T, np.triu(S) + np.triu(S, 1).T
    assert entries_ok(Hu, Hr) and entries_ok(Su, Sr, abs_frac=0.0)
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


def check_kinds(ops, d):
    """Laplace, Nuclear, Mass operators assembled on their own ({kind: dense or (kidx, blocks)})
    against the reference's: Nuclear and Mass pure 1e-10 relative, Laplace (stiffness entries
    cancel) with the 1e-14 max|.| absolute term."""
    for kind, tag, absf in (("nuclear", "N", 0.0), ("mass", "M", 0.0), ("laplace", "Lap", 1e-14)):
        if bool(d["periodic"]):
            k, b = ops[kind]
            assert np.array_equal(k, d["kidx"]), kind
            ref = d[f"{tag}_blocks"]
        else:
            D = ops[kind]
            b = np.triu(D) + np.triu(D, 1).T
            ref = ref_dense(d, tag)
        assert entries_ok(b, ref, abs_frac=absf), kind


# Eigenvalue parity (north star: 1e-9 Hartree). Each reference eigenvalue carries its FP64
# floor (`eig_floor`, tests/golden/make_floor.py): the largest change of that eigenvalue when
# the entries of the reference pencil are perturbed by random 8-ulp relative amounts (8 draws).
# GPU and reference entries are two FP64 summation orders of the same sums and differ by up
# to ~66 ulps (profiles/r02_parity.json), so the end-to-end bound is 16 floors (the 128-ulp
# floor in the linear regime); the eigensolver alone — GPU vs the reference algorithm on the
# identical pencil — is held to 2 floors. Eigenvalues whose scaled floor is below 1e-9 are
# held to 1e-9 Hartree.
EIG_FLOOR_E2E = 16.0
EIG_FLOOR_SOLVER = 2.0


def eig_tolerance_golden(d, factor=EIG_FLOOR_E2E):
    return np.maximum(1e-9, factor * np.asarray(d["eig_floor"]))


def check_eigs(ev, d):
    ev = np.asarray(ev).reshape(d["eig"].shape)
    err = np.abs(ev - d["eig"])
    tol = eig_tolerance_golden(d)
    assert np.all(err <= tol), (float(np.max(err / tol)), float(np.max(err)))
    return float(np.max(err)), float(np.max(err / tol))
