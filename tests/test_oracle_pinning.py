"""Oracle-X pinned to the reference itself (CPU only).

Oracle-R is the reference's own proj/core/src/*.cpp compiled in place against the
Eigen-subset shim (make -C oracle ref). On isotropic grids (the only ones the reference
accepts) Oracle-X must reproduce it bit for bit: every assembled operator, every stage,
every eigenvalue.
"""
import numpy as np
import pytest

from conftest import chain_system, two_nuclei_system
from oracle.binding import reference

SYSTEMS = {
    "chain6_box": (chain_system(6, 0.05, M=8), False),
    "chain8_per": (chain_system(8, 0.05, M=6), True),
    "chain4_two": (chain_system(4, [0.1, 0.4], M=6), False),
    "two_box": (two_nuclei_system((6, 1, 1), n=(16, 16, 16)), False),
    "two_per": (two_nuclei_system((12, 1, 1), n=(16, 16, 16)), True),
    "box2d": (two_nuclei_system((3, 2, 1), n=(8, 8, 8), alphas=(1.5, 3.0)), False),
    "per3d": (two_nuclei_system((5, 6, 5), n=(6, 6, 6), alphas=(3.0, 5.0), M=6), True),
    "pdeg_box": (two_nuclei_system((4, 1, 1), n=(8, 8, 8), alphas=(1.0, 2.0), deg=[[1, 0, 0], [0, 1, 1]]), False),
    "pdeg_per": (two_nuclei_system((9, 1, 1), n=(8, 8, 8), alphas=(1.0, 2.0), deg=[[2, 0, 0], [1, 1, 0]]), True),
    "unit_box": (two_nuclei_system((1, 1, 1), n=(10, 10, 10), alphas=(0.8, 1.6)), False),
}


@pytest.fixture(scope="module")
def ref():
    r = reference()
    if r is None:
        pytest.skip("Oracle-R not built (needs /root/reference: make -C oracle ref)")
    return r


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_assembly_and_spectrum_bitwise(oracle, ref, name):
    s, per = SYSTEMS[name]
    assert oracle.overlap_constant(s) == ref.overlap_constant(s)
    for kind in ("mass", "laplace", "nuclear"):
        a, b = oracle.assemble(s, per, kind), ref.assemble(s, per, kind)
        assert (a.L0, a.coefficient_rank) == (b.L0, b.coefficient_rank)
        if per:
            assert np.array_equal(a.kidx, b.kidx) and np.array_equal(a.blocks, b.blocks)
        else:
            assert np.array_equal(a.dense, b.dense)
    H, S = oracle.assemble_core(s, per)
    H2, S2 = ref.assemble_core(s, per)
    if per:
        assert np.array_equal(oracle.solve_periodic_ops(H, S), ref.solve_periodic_ops(H2, S2))
    else:
        assert np.array_equal(oracle.solve_box_dense(H.dense, S.dense), ref.solve_box_dense(H2.dense, S2.dense))


def test_stages_bitwise(oracle, ref):
    for M in (1, 3, 12, 20):
        t1, w1 = oracle.sinc_quadrature(M)
        t2, w2 = ref.sinc_quadrature(M)
        assert np.array_equal(t1, t2) and np.array_equal(w1, w2)
    for ncells, h, M in ((64, 0.25, 10), (301, 2.0 / 64, 16)):
        assert np.array_equal(oracle.newton_master_column(ncells, h, M), ref.newton_master_column(ncells, h, M))
    rng = np.random.default_rng(3)
    m = rng.uniform(0.1, 1.0, size=(200, 5))
    for shifts in ([10 + 7 * k for k in range(9)], [17], [5, 9, 20]):
        assert np.array_equal(oracle.assembled_window_sum(m, shifts, 60), ref.assembled_window_sum(m, shifts, 60))
    for name in ("two_box", "two_per", "per3d", "unit_box"):
        s, per = SYSTEMS[name]
        for margin in (2, 5):
            p1, w1, t1 = oracle.potential(s, per, margin)
            p2, w2, t2 = ref.potential(s, per, margin)
            assert t1 == t2 and np.array_equal(w1, w2)
            for l in range(3):
                assert np.array_equal(p1[l], p2[l])
    for args in (((0.3, -0.2, 0.1), 0.7, (0, 0, 0), 0, 80, 0.25, 3, 8, 2.0, 0.5, 1e-280),
                 ((0.3, -0.2, 0.1), 1.1, (2, 1, 0), 1, 80, 0.25, 2, 8, 2.0, 0.0, 1e-280),
                 ((0.0, 0.0, 0.0), 0.005, (0, 0, 0), 2, 64, 1.0, 3, 8, 8.0, 0.5, 0.0)):
        o1, v1 = oracle.sample_gto_1d(*args)
        o2, v2 = ref.sample_gto_1d(*args)
        assert o1 == o2 and np.array_equal(v1, v2)
    u = rng.uniform(-1, 1, 9)
    v = rng.uniform(-1, 1, 7)
    for h in (0.25, 2.0 / 64):
        assert oracle.tri_form(3, u, 5, v, -1 / h, 2 / h) == ref.tri_form(3, u, 5, v, -1 / h, 2 / h)
        assert abs(oracle.tri_form(3, u, 5, v, h / 6, 4 * h / 6) - ref.tri_form(3, u, 5, v, h / 6, 4 * h / 6)) <= 1e-15


def test_error_behaviour_matches(oracle, ref):
    from oracle.binding import OracleError
    for call in (lambda o: o.assemble(chain_system(2, 0.05), True, "mass"),
                 lambda o: o.solve_box_dense(np.eye(3), np.diag([1.0, 1.0, -1.0])),
                 lambda o: o.solve_box_dense(np.eye(8), np.eye(8), cap=4),
                 lambda o: o.solve_periodic((3, 1, 1), 1, {(0, 0, 0): np.array([[1.0]])},
                                            {(0, 0, 0): np.array([[-1.0]])})):
        with pytest.raises(OracleError) as e1:
            call(oracle)
        with pytest.raises(OracleError) as e2:
            call(ref)
        assert e1.value.kind == e2.value.kind and e1.value.msg == e2.value.msg


def test_factorized_path_matches_fft_path(ref):
    # solve_periodic_factorized (eigensolver.cpp:143-162) vs solve_periodic on the same operators
    s, _ = SYSTEMS["two_per"]
    H, S = ref.assemble_core(s, True)
    a = ref.solve_periodic_ops(H, S)
    b = ref.solve_periodic_factorized_ops(H, S)
    assert np.max(np.abs(a - b)) < 1e-9
