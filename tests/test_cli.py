"""The latham_b200 command-line front end: the reference CLI's wire formats and exit codes
(tests restate proj/tests/test_cli.cpp; parity of the written spectra against Oracle-X)."""
import os
import subprocess

import numpy as np
import pytest

from paper_1408_3839_b200.system import LatticeSystem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1408_3839_b200", "_lib", "latham_b200")

CHAIN = """
cell.b = 8.0
grid.n = 8
grid.nbar = 8
quad.M = 10
lattice.L = 4 1 1
boundary = both
nucleus = 0 0 0 1.0
basis = 0 0 0 0.3
n_occ = 1
"""


def need_cli():
    if not os.path.exists(CLI):
        pytest.skip("latham_b200 CLI not built")


def run(tmp_path, sub, body, out="out", name="exp.cfg"):
    need_cli()
    cfg = tmp_path / name
    if body is not None:
        cfg.write_text(body)
    p = subprocess.run([CLI, sub, "--config", str(cfg), "--out", str(tmp_path / out)], capture_output=True, text=True)
    return p.returncode


def data_lines(path):
    return [ln for ln in open(path).read().splitlines() if ln and not ln.startswith("#")]


# ---- configuration errors: no device needed (parsing precedes any GPU work) ----------
def test_config_errors_exit_two(tmp_path):
    assert run(tmp_path, "solve", "nonsense\n") == 2
    assert run(tmp_path, "solve", "unknown.key = 3\n") == 2
    assert run(tmp_path, "solve", None, name="missing.cfg") == 2
    assert run(tmp_path, "solve", "cell.b = 8\nnucleus = 7 0 0 1\nbasis = 0 0 0 0.3\n") == 2  # outside the cell
    assert run(tmp_path, "kernel", CHAIN + "lattice.L = 1 1 1\n") == 2  # duplicate key
    assert run(tmp_path, "solve", CHAIN + "caps.dense = 9000\n") == 2  # raised cap without acknowledgement


def test_usage_errors(tmp_path):
    need_cli()
    assert subprocess.run([CLI], capture_output=True).returncode == 2
    assert subprocess.run([CLI, "frobnicate", "--config", "x", "--out", "y"], capture_output=True).returncode == 2


# ---- GPU runs ----------------------------------------------------------------------------
@pytest.mark.gpu
def test_kernel_smoke_and_quadrature_convergence(tmp_path):
    def err(M):
        body = f"cell.b = 8\ngrid.n = 8\nquad.M = {M}\nlattice.L = 1 1 1\nnucleus = 0 0 0 1\nbasis = 0 0 0 0.3\n"
        assert run(tmp_path, "kernel", body, out=f"m{M}", name=f"m{M}.cfg") == 0
        lines = data_lines(tmp_path / f"m{M}" / "kernel_report.csv")
        assert len(lines) == 2 and "rank_bound" in lines[0]
        return float(lines[1].split(",")[5])
    e10, e20, e40 = err(10), err(20), err(40)
    assert e20 < e10 and e40 < e20


@pytest.mark.gpu
def test_solve_periodic_rows(tmp_path):
    assert run(tmp_path, "solve", CHAIN.replace("boundary = both", "boundary = periodic")) == 0
    rows = data_lines(tmp_path / "out" / "spectrum_periodic.csv")
    assert len(rows) == 5 and rows[0] == "k1,k2,k3,band,eigenvalue"
    for r in rows[1:]:
        float(r.split(",")[4])


@pytest.mark.gpu
def test_solve_both_files_defect_and_byte_identical_reruns(tmp_path, oracle):
    assert run(tmp_path, "solve", CHAIN, out="a") == 0
    assert run(tmp_path, "solve", CHAIN, out="b") == 0
    for f in ("spectrum_box.csv", "spectrum_periodic.csv", "bands_box.csv", "bands_periodic.csv", "defect.csv",
              "bands.gp"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f
    rows = data_lines(tmp_path / "a" / "defect.csv")
    assert "nuclear_defect_rel_fro" in rows[0] and len(rows) == 2
    head = (tmp_path / "a" / "spectrum_box.csv").read_text().splitlines()
    assert head[0] == "# latham solve" and "# cell.b = 8" in head and "# eps_ov = 1e-08" in head
    # the written spectra against the oracle's solve of the same system
    s = LatticeSystem(b=8.0, L=(4, 1, 1), n=(8,) * 3, nbar=(8,) * 3, quad_M=10, nuc_pos=[(0, 0, 0)],
                      nuc_charge=[1.0], bf_center=[(0, 0, 0)], bf_alpha=[0.3])
    H, S = oracle.assemble_core(s, True)
    ref = np.sort(oracle.solve_periodic_ops(H, S).reshape(-1))
    got = np.sort([float(r.split(",")[4]) for r in data_lines(tmp_path / "a" / "spectrum_periodic.csv")[1:]])
    assert np.max(np.abs(got - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))
    Hb, Sb = oracle.assemble_core(s, False)
    refb = oracle.solve_box_dense(Hb.dense, Sb.dense)
    gotb = np.array([float(r.split(",")[4]) for r in data_lines(tmp_path / "a" / "spectrum_box.csv")[1:]])
    assert np.max(np.abs(gotb - refb)) <= 1e-9 * max(1.0, np.max(np.abs(refb)))


@pytest.mark.gpu
def test_solve_eigenvectors_files(tmp_path, oracle):
    """solve.eigenvectors = true (commands.cpp:183-205): eigenvectors_box.csv holds the
    S-orthonormal pencil eigenvectors, eigenvectors_periodic.csv the reconstructed
    lattice eigenvectors; both satisfy the generalised eigenproblem of the dense matrices."""
    assert run(tmp_path, "solve", CHAIN + "solve.eigenvectors = true\n", out="v") == 0
    assert run(tmp_path, "solve", CHAIN + "solve.eigenvectors = true\n", out="w") == 0
    for f in ("eigenvectors_box.csv", "eigenvectors_periodic.csv", "spectrum_box.csv"):
        assert (tmp_path / "v" / f).read_bytes() == (tmp_path / "w" / f).read_bytes(), f
    s = LatticeSystem(b=8.0, L=(4, 1, 1), n=(8,) * 3, nbar=(8,) * 3, quad_M=10, nuc_pos=[(0, 0, 0)],
                      nuc_charge=[1.0], bf_center=[(0, 0, 0)], bf_alpha=[0.3])
    Hb, Sb = oracle.assemble_core(s, False)
    rows = data_lines(tmp_path / "v" / "eigenvectors_box.csv")
    assert rows[0] == "index,component,value" and len(rows) == 1 + 16
    X = np.zeros((4, 4))
    for r in rows[1:]:
        c, i, v = r.split(",")
        X[int(i), int(c)] = float(v)
    lam = np.array([float(r.split(",")[4]) for r in data_lines(tmp_path / "v" / "spectrum_box.csv")[1:]])
    assert np.max(np.abs(X.T @ Sb.dense @ X - np.eye(4))) < 1e-9
    assert np.max(np.abs(Hb.dense @ X - Sb.dense @ X * lam)) < 1e-9 * max(1.0, np.max(np.abs(Hb.dense)))
    rows = data_lines(tmp_path / "v" / "eigenvectors_periodic.csv")
    assert rows[0] == "index,component,re,im" and len(rows) == 1 + 16
    U = np.zeros((4, 4), dtype=complex)
    for r in rows[1:]:
        c, i, re, im = r.split(",")
        U[int(i), int(c)] = float(re) + 1j * float(im)
    H, S = oracle.assemble_core(s, True)
    ev = oracle.solve_periodic_ops(H, S).reshape(-1)
    from test_gpu_vectors import bc_to_dense
    Hd, Sd = bc_to_dense(H.gen_dict(), (4, 1, 1), 1), bc_to_dense(S.gen_dict(), (4, 1, 1), 1)
    assert np.max(np.abs(U.conj().T @ Sd @ U - np.eye(4))) < 1e-9
    assert np.max(np.abs(Hd @ U - (Sd @ U) * ev)) < 1e-9 * max(1.0, np.max(np.abs(Hd)))


@pytest.mark.gpu
def test_energy_sweep(tmp_path):
    assert run(tmp_path, "energy", CHAIN + "energy.L_list = 4 8\n") == 0
    rows = data_lines(tmp_path / "out" / "energy.csv")
    assert len(rows) == 5 and rows[0] == "L1,L2,L3,boundary,E_per_cell"


@pytest.mark.gpu
def test_bench_timings_and_exponents(tmp_path):
    assert run(tmp_path, "bench", CHAIN + "bench.L_list = 4 8\n") == 0
    assert len(data_lines(tmp_path / "out" / "bench.csv")) == 5
    assert len(data_lines(tmp_path / "out" / "bench_exponents.csv")) == 3


@pytest.mark.gpu
def test_resource_cap_exits_four(tmp_path):
    body = """cell.b = 8.0
grid.n = 4
grid.nbar = 4
quad.M = 5
lattice.L = 4 1 1
boundary = box
nucleus = 0 0 0 1.0
basis = 0 0 0 0.3
caps.dense = 2
caps.acknowledge = false
"""
    assert run(tmp_path, "solve", body) == 4


@pytest.mark.gpu
def test_wrap_alias_exits_numerical(tmp_path):
    body = """cell.b = 8.0
grid.n = 8
grid.nbar = 8
quad.M = 6
lattice.L = 2 1 1
boundary = periodic
nucleus = 0 0 0 1.0
basis = 0 0 0 0.05
"""
    assert run(tmp_path, "solve", body) == 3
