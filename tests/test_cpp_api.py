"""The C++ mirror of the reference API (include/latham_b200.hpp): a reference-style client
(tests/cpp/core_solve.cpp) compiles and links against the C-ABI library on CPU; on the GPU
it reproduces the Python API bitwise and the reference's exception classes."""
import os
import subprocess

import numpy as np
import pytest

from paper_1408_3839_b200.system import LatticeSystem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1408_3839_b200", "_lib")


def build(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "liblatham_b200.so")):
        pytest.skip("C-ABI library not built")
    exe = str(tmp_path / "core_solve")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "core_solve.cpp"), "-L" + LIBDIR, "-llatham_b200",
           "-Wl,-rpath," + LIBDIR, "-Wl,-rpath-link,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_client_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


def chain(Lx, two):
    pos = [[-0.5, 0, 0], [0.5, 0, 0]] if two else [[0, 0, 0]]
    centers = [p for p in pos for _ in range(2)]
    alphas = [a for _ in pos for a in (1.3, 3.1)]
    return LatticeSystem(b=2.0, L=(Lx, 1, 1), n=(32,) * 3, nbar=(32,) * 3, quad_M=8, nuc_pos=pos,
                         nuc_charge=[1.0] * len(pos), bf_center=centers, bf_alpha=alphas)


@pytest.mark.gpu
def test_cpp_client_matches_python_api(tmp_path, ctx):
    out = subprocess.run([build(tmp_path)], check=True, capture_output=True, text=True).stdout.splitlines()
    # (NCCL may print its version banner on communicator creation: keep the client's lines)
    res = {ln.split()[0]: ln.split()[1:] for ln in out if ln.split() and not ln.startswith("NCCL")}
    vals = {k: np.array([float(x) for x in v[1:]]) for k, v in res.items() if not k.startswith(("error", "resid"))}
    per = np.sort(ctx.solve_core(chain(16, True), True).reshape(-1))
    box = ctx.solve_core(chain(6, False), False)
    assert np.array_equal(vals["periodic_core"], per)
    assert np.array_equal(vals["box_core"], box)
    # lt_solve_core_multi (NCCL communicator over the listed devices): k-point split bitwise,
    # rank-term split (partial H summed by the all-reduce) to rounding
    assert np.array_equal(vals["periodic_multi_k"], per)
    assert np.max(np.abs(vals["periodic_multi_r"] - per)) < 1e-10 * max(1.0, np.max(np.abs(per)))
    # the separate-operator route (assemble x3, combine, solve) agrees to rounding
    assert np.max(np.abs(vals["periodic_ops"] - per)) < 1e-10 * max(1.0, np.max(np.abs(per)))
    assert np.max(np.abs(vals["box_ops"] - box)) < 1e-10 * max(1.0, np.max(np.abs(box)))
    assert np.max(np.abs(vals["periodic_factorized"] - per)) < 1e-10 * max(1.0, np.max(np.abs(per)))
    assert float(res["residual"][0]) < 1e-12
    assert np.max(np.abs(vals["periodic_vec_eig"] - per)) < 1e-10 * max(1.0, np.max(np.abs(per)))
    assert np.max(np.abs(vals["box_vec_eig"] - box)) < 1e-10 * max(1.0, np.max(np.abs(box)))
    assert float(res["recon_col_dev"][0]) < 1e-15
    n = box.size
    X = vals["box_vec"].reshape(n, n).T
    assert X.shape == (n, n) and np.all(np.isfinite(X))
    assert res["error_alias"][0] == "StructureError"
    assert res["error_cap"][0] == "ResourceCapError"
