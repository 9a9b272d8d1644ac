"""Generate the committed golden fixtures (run here, where /root/reference exists).

* small isotropic systems: produced by Oracle-R, i.e. the reference's own
  proj/core/src/*.cpp compiled in place (oracle/_ref/libref_latham.so);
* BASELINE configs c1..c5 (anisotropic grids, which the reference API cannot express):
  produced by Oracle-X, which is bit-identical to Oracle-R on every isotropic case
  (tests/test_oracle_pinning.py).

Each fixture stores the full reference core pencil H = 0.5 Laplace - Nuclear, S = Mass
(upper triangle for box systems, all generating blocks for periodic ones), its
eigenvalues, L0/band, and each eigenvalue's first-order condition coefficient
kappa_i = ||x_i||^2 for S-normalised eigenvectors x_i (per k-point block for periodic
systems), used by tests/golden_util.check_eigs to bound |lambda_gpu - lambda_ref|
from the measured entry discrepancy.

    python tests/golden/make_golden.py [names...]
"""
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import chain_system, two_nuclei_system  # noqa: E402
from oracle.binding import oracle, reference  # noqa: E402
from paper_1408_3839_b200.system import make_config  # noqa: E402

SMALL = {
    "chain6_box": (chain_system(6, 0.05, M=8), False),
    "chain8_per": (chain_system(8, 0.05, M=6), True),
    "chain16_per_two": (chain_system(16, [0.05, 0.25], M=8), True),
    "two_box": (two_nuclei_system((6, 1, 1), n=(16, 16, 16)), False),
    "two_per": (two_nuclei_system((12, 1, 1), n=(16, 16, 16)), True),
    "box2d": (two_nuclei_system((3, 2, 1), n=(8, 8, 8), alphas=(1.5, 3.0)), False),
    "per3d": (two_nuclei_system((5, 6, 5), n=(6, 6, 6), alphas=(3.0, 5.0), M=6), True),
    "pdeg_box": (two_nuclei_system((4, 1, 1), n=(8, 8, 8), alphas=(1.0, 2.0), deg=[[1, 0, 0], [0, 1, 1]]), False),
    "pdeg_per": (two_nuclei_system((9, 1, 1), n=(8, 8, 8), alphas=(1.0, 2.0), deg=[[2, 0, 0], [1, 1, 0]]), True),
}


def sys_arrays(s):
    return dict(b=s.b, L=np.array(s.L), n=np.array(s.n), nbar=np.array(s.nbar), quad_M=s.quad_M, eps_ov=s.eps_ov,
                nuc_pos=s.nuc_pos, nuc_charge=s.nuc_charge, bf_center=s.bf_center, bf_alpha=s.bf_alpha,
                bf_deg=s.bf_deg)


def kappa_box(H, S):
    _, X = sl.eigh(H, S)  # X^T S X = I
    return np.sum(X * X, axis=0)


def kappa_periodic(impl, H, S, dims, m0):
    Hb = oracle().block_diagonalize(dims, m0, H.gen_dict())
    Sb = oracle().block_diagonalize(dims, m0, S.gen_dict())
    out = np.zeros((Hb.shape[0], m0))
    for j in range(Hb.shape[0]):
        h = 0.5 * (Hb[j] + Hb[j].conj().T)
        s = 0.5 * (Sb[j] + Sb[j].conj().T)
        _, X = sl.eigh(h, s)
        out[j] = np.sum(np.abs(X) ** 2, axis=0)
    return out


def make(name, s, periodic, impl, src):
    t0 = time.time()
    H, S = impl.assemble_core(s, periodic)
    if periodic:
        ev = impl.solve_periodic_ops(H, S, os.cpu_count() or 1)
        kap = kappa_periodic(impl, H, S, s.L, s.m0)
    else:
        ev = impl.solve_box_dense(H.dense, S.dense)
        kap = kappa_box(H.dense, S.dense)
    d = dict(sys_arrays(s), periodic=periodic, source=src, L0=H.L0, band=np.array(H.band), eig=ev, kappa=kap)
    if periodic:
        d["kidx"] = H.kidx
        d["H_blocks"] = H.blocks
        d["S_blocks"] = S.blocks
    else:
        d["H_upper"] = np.triu(H.dense)
        d["S_upper"] = np.triu(S.dense)
        d["H_sym_dev"] = np.max(np.abs(H.dense - H.dense.T))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"{name}: {src}, L0={H.L0}, max kappa={np.max(kap):.2e}, {time.time() - t0:.1f}s", flush=True)


def main():
    names = sys.argv[1:]
    ref = reference()
    if ref is None:
        raise SystemExit("Oracle-R not built: make -C oracle ref")
    for name, (s, per) in SMALL.items():
        if not names or name in names:
            make(name, s, per, ref, "Oracle-R (reference sources compiled in place)")
    for cfg in ("c1", "c2", "c5", "c4", "c3"):
        if not names or cfg in names:
            s = make_config(cfg)
            make(cfg, s, s.notes["periodic"], oracle(), "Oracle-X (bit-identical to Oracle-R on isotropic grids)")


if __name__ == "__main__":
    main()
