"""GPU coverage of paths the BASELINE configs do not reach on their own.

* ``lt_assembled_window_sum`` called directly (canonical_tensor.cpp:123-164) in each of its
  device forms: the running sum of a uniform shift progression (the reference's recurrence,
  bit-identical), the periodic cell window (size <= step, >= 32 shifts: warp-parallel
  K-term sums, 1e-13 relative), the single-shift copy; and its BoundsError.
* The dense box pencil beyond the on-chip tridiagonalisation (N_b = 2048: the device
  reduction, the library eigensolver on A), eigensolver.cpp:12-35, against scipy.
* A BASELINE-size periodic system (c2's lattice and grids) whose basis carries p-type
  functions, so the L0 search runs its sampled scan (k_l0_sample + k_l0_scan) instead of the
  s-type peak windows, against Oracle-X (entries, L0, eigenvalues).
"""
import numpy as np
import pytest

from conftest import eig_tolerance, entries_close
from paper_1408_3839_b200.api import Context
from paper_1408_3839_b200.native import BoundsError
from paper_1408_3839_b200.system import LatticeSystem, make_config

pytestmark = pytest.mark.gpu


def _direct_window_sum(m, shifts, size):
    return sum(m[s:s + size] for s in shifts)


def test_window_sum_staged_uniform(ctx, oracle):
    """Uniform progressions staged through shared memory (segmented running sums): within
    1e-13 of the panel's largest entry of the reference's one-chain running sum and of the
    direct sum; odd / even window starts and column offsets exercise the 16-byte bulk-copy
    alignment, the last case the chunking over several CTAs per column."""
    rng = np.random.default_rng(11)
    m = rng.uniform(0.05, 1.0, size=(900, 7))
    cases = [([10 + 16 * k for k in range(24)], 400), ([3, 67, 131], 700), ([0, 1], 899), ([1, 2], 898),
             ([5 + 3 * k for k in range(9)], 1), ([7 + 64 * k for k in range(6)], 64), ([2 * k for k in range(40)], 801)]
    for shifts, size in cases:
        got = ctx.assembled_window_sum(m, shifts, size)
        ref = oracle.assembled_window_sum(m, shifts, size)  # the reference's running sum
        assert got.shape == ref.shape
        scale = np.max(np.abs(ref))
        assert np.max(np.abs(got - ref)) <= 1e-13 * scale, (shifts[:3], size)
        assert np.max(np.abs(got - _direct_window_sum(m, shifts, size))) <= 1e-13 * scale
    big = rng.uniform(0.05, 1.0, size=(17025, 3))  # c3-like: 128 shifts of 64, 8704 outputs, odd column length
    shifts = [33 + 64 * k for k in range(128)]
    got = ctx.assembled_window_sum(big, shifts, 8704)
    ref = oracle.assembled_window_sum(big, shifts, 8704)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert np.max(np.abs(got - _direct_window_sum(big, shifts, 8704))) <= 1e-13 * np.max(np.abs(ref))


def test_window_sum_cell_window_and_copy(ctx, oracle):
    rng = np.random.default_rng(12)
    m = rng.uniform(0.05, 1.0, size=(64 * 40 + 64, 5))
    shifts = [64 * k for k in range(40)]  # 40 cells of 64 points, one output per residue
    got = ctx.assembled_window_sum(m, shifts, 64)
    ref = oracle.assembled_window_sum(m, shifts, 64)
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-13
    one = ctx.assembled_window_sum(m, [77], 300)
    assert np.array_equal(one, m[77:377])


def test_window_sum_bounds(ctx):
    m = np.ones((100, 3))
    with pytest.raises(BoundsError):
        ctx.assembled_window_sum(m, [90], 20)


def test_dense_pencil_beyond_onchip_tridiagonalisation(ctx):
    scipy_linalg = pytest.importorskip("scipy.linalg")
    n = 2048  # above the register/shared-memory resident one-stage reduction (~1900)
    rng = np.random.default_rng(13)
    B = rng.standard_normal((n, n)) / np.sqrt(n)
    S = B @ B.T + np.eye(n)
    A = rng.standard_normal((n, n))
    H = 0.5 * (A + A.T)
    ev = ctx.solve_box_dense(H, S)
    ref = scipy_linalg.eigh(H, S, eigvals_only=True)
    scale = np.max(np.abs(ref))
    assert np.all(np.diff(ev) >= 0)
    assert np.max(np.abs(ev - ref)) <= 1e-11 * scale


def _with_p_functions(sys: LatticeSystem) -> LatticeSystem:
    # p_x (along the lattice) on the two steepest functions, p_y on the fourth steepest: both
    # the wrapped and a transverse direction take the sampled L0 scan; the overlap stays
    # positive definite at every k-point (other placements make S_0 numerically singular)
    deg = np.zeros((len(sys.bf_alpha), 3), dtype=np.int32)
    order = np.argsort(sys.bf_alpha)
    deg[order[-2:], 0] = 1
    deg[order[-4], 1] = 1
    return LatticeSystem(b=sys.b, L=tuple(sys.L), n=tuple(sys.n), nbar=tuple(sys.nbar), quad_M=sys.quad_M,
                         nuc_pos=sys.nuc_pos, nuc_charge=sys.nuc_charge, bf_center=sys.bf_center,
                         bf_alpha=sys.bf_alpha, bf_deg=deg, eps_ov=sys.eps_ov, name="c2_p")


def test_baseline_size_with_p_functions(ctx, oracle):
    sys = _with_p_functions(make_config("c2"))
    oH, oS = oracle.assemble_core(sys, True)
    info = np.zeros(8, dtype=np.int64)
    ev = ctx.solve_core(sys, True, info)
    assert info[0] == oH.L0
    H, S = ctx.assemble_core(sys, True)
    ok, worst = entries_close(H.blocks()[1], oH.blocks)
    assert ok, worst
    ok, worst = entries_close(S.blocks()[1], oS.blocks)
    assert ok, worst
    oev = oracle.solve_periodic_ops(oH, oS)
    tol = eig_tolerance(oracle, True, oH, oS, oev)
    assert np.all(np.abs(ev - oev) <= tol), np.max(np.abs(ev - oev) / tol)


@pytest.mark.parametrize("L,n", [(40, 16), (150, 16), (64, 32), (48, 24)])
def test_box_chain_nuclear_hankel_shapes(ctx, oracle, L, n):
    """The box-chain nuclear contraction (galerkin.cpp:224-247) across the shapes of the Hankel
    kernels: a partly filled 128-cell tile (L = 40, 48, 64), two cell tiles (L = 150), rows of
    16 and 32 points (the shared-memory resident TMA kernel) and of 24 points (not a multiple
    of 16: the tile-loading kernel); H and S entries against Oracle-X."""
    pos = [(-0.45, 0.1, 0.0), (0.5, 0.0, -0.2)]
    sys = LatticeSystem(b=2.0, L=(L, 1, 1), n=(n, 8, 8), nbar=(n, 8, 8), quad_M=6, nuc_pos=pos, nuc_charge=[1.0, 2.0],
                        bf_center=[pos[0], pos[1], pos[0], pos[1]], bf_alpha=[0.35, 2.5, 0.9, 6.0])
    oH, oS = oracle.assemble_core(sys, False)
    H, S = ctx.assemble_core(sys, False)
    ok, worst = entries_close(H.dense(), oH.dense)
    assert ok, worst
    ok, worst = entries_close(S.dense(), oS.dense)
    assert ok, worst


@pytest.mark.parametrize("periodic", [True, False])
def test_l0_prediction_across_systems_of_one_shape(periodic):
    """L0 is predicted from the previous system of the same shape (exponent scans run without
    the L0 host round trip); a system whose L0 differs must be detected on the device and
    solved again: alternating two such systems on one context reproduces the spectra of fresh
    contexts exactly, with the right L0 reported each time."""
    pos = [(-0.5, 0.1, 0.0), (0.5, 0.0, -0.2)]

    def system(scale):
        return LatticeSystem(b=2.0, L=(12, 1, 1) if periodic else (6, 1, 1), n=(16, 8, 8), nbar=(16, 8, 8), quad_M=8,
                             nuc_pos=pos, nuc_charge=[1.0, 2.0], bf_center=[pos[0], pos[1], pos[0], pos[1]],
                             bf_alpha=[0.9 * scale, 2.5 * scale, 0.6 * scale, 4.0 * scale])

    tight, diffuse = system(1.0), system(0.45)
    ref = {}
    for name, s in (("tight", tight), ("diffuse", diffuse)):
        c = Context(0)
        info = np.zeros(8, dtype=np.int64)
        ref[name] = (c.solve_core(s, periodic, info).copy(), int(info[0]))
        c.close()
    assert ref["tight"][1] != ref["diffuse"][1], "the two systems must differ in L0 for this test"
    c = Context(0)
    for name, s in (("tight", tight), ("tight", tight), ("diffuse", diffuse), ("tight", tight), ("diffuse", diffuse),
                    ("diffuse", diffuse), ("tight", tight)):
        info = np.zeros(8, dtype=np.int64)
        ev = c.solve_core(s, periodic, info)
        assert int(info[0]) == ref[name][1], name
        assert np.array_equal(ev, ref[name][0]), name
    c.close()
