"""GPU parity of the spectrum stage: lattice DFT, batched pencils, dense box pencil.

Known-answer tests restate the reference's test_block_circulant.cpp / test_eigensolver.cpp;
random pencils compare with the oracle and with scipy (independent route)."""
import numpy as np
import pytest
import scipy.linalg as sl

from paper_1408_3839_b200.api import DefinitenessError, ResourceCapError

pytestmark = pytest.mark.gpu


def scalar_gen(col):
    return {(k, 0, 0): np.array([[v]]) for k, v in enumerate(col)}


def test_block_diagonalize_kats(ctx):
    # test_block_circulant.cpp:75-79 {3,1}
    bd = ctx.bc_block_diagonalize((2, 1, 1), 1, scalar_gen([2.0, 1.0]))
    assert abs(bd[0, 0, 0] - 3.0) < 1e-14 and abs(bd[1, 0, 0] - 1.0) < 1e-14
    # :81-95 two-level signs {8,4,2,2}
    g = {(0, 0, 0): np.array([[4.0]]), (0, 1, 0): np.array([[1.0]]), (1, 0, 0): np.array([[2.0]]),
         (1, 1, 0): np.array([[1.0]])}
    bd = ctx.bc_block_diagonalize((2, 2, 1), 1, g)
    assert np.allclose(bd[:, 0, 0].real, [8.0, 4.0, 2.0, 2.0], atol=1e-13)


def test_block_diagonalize_vs_oracle(ctx, oracle):
    rng = np.random.default_rng(5)
    for dims, m0 in (((7, 1, 1), 3), ((4, 3, 1), 2), ((3, 2, 5), 4), ((16, 1, 1), 8)):
        gen = {}
        for _ in range(int(np.prod(dims)) // 2 + 1):
            k = tuple(int(rng.integers(0, d)) for d in dims)
            gen[k] = rng.standard_normal((m0, m0))
        g = ctx.bc_block_diagonalize(dims, m0, gen)
        o = oracle.block_diagonalize(dims, m0, gen)
        assert np.max(np.abs(g - o)) < 1e-12 * max(1.0, np.max(np.abs(o)))


def random_pencils(rng, count, m0):
    A = rng.standard_normal((count, m0, m0)) + 1j * rng.standard_normal((count, m0, m0))
    H = A + np.conj(np.transpose(A, (0, 2, 1)))
    B = rng.standard_normal((count, m0, m0)) + 1j * rng.standard_normal((count, m0, m0))
    S = B @ np.conj(np.transpose(B, (0, 2, 1))) + m0 * np.eye(m0)
    return H, S


@pytest.mark.parametrize("m0", [1, 2, 3, 5, 8, 11, 16, 20, 32])
def test_pencils_random(ctx, oracle, m0):
    rng = np.random.default_rng(100 + m0)
    H, S = random_pencils(rng, 37, m0)
    ev = ctx.pencil_eig(H, S)
    for j in range(H.shape[0]):
        ref = sl.eigh(H[j], S[j], eigvals_only=True)
        assert np.max(np.abs(ev[j] - ref)) < 1e-11 * max(1.0, np.max(np.abs(ref)))
        orc = oracle.solve_pencil(H[j], S[j], j)
        assert np.max(np.abs(ev[j] - orc)) < 1e-11 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("m0,count", [(8, 1300), (12, 700), (24, 160), (6, 1100)])
def test_pencils_large_batch(ctx, m0, count):
    # batches too large for the latency layout take the throughput layout (fewer
    # multisection points per eigenvalue); both must agree with scipy
    rng = np.random.default_rng(7 * m0 + count)
    H, S = random_pencils(rng, count, m0)
    ev = ctx.pencil_eig(H, S)
    for j in range(0, count, 7):
        ref = sl.eigh(H[j], S[j], eigvals_only=True)
        assert np.max(np.abs(ev[j] - ref)) < 1e-11 * max(1.0, np.max(np.abs(ref)))


def test_pencil_scalar_kat(ctx):
    # test_eigensolver.cpp:28-34 scalar pencil (-0.3, 0.8) -> -0.375
    ev = ctx.pencil_eig(np.array([[[-0.3 + 0j]]]), np.array([[[0.8 + 0j]]]))
    assert abs(ev[0, 0] + 0.375) < 1e-14


def test_indefinite_overlap_names_kpoint(ctx):
    # test_eigensolver.cpp:133-146: every Fourier block of S is -1
    H = {(0, 0, 0): np.array([[1.0]])}
    S = {(0, 0, 0): np.array([[-1.0]])}
    with pytest.raises(DefinitenessError) as e:
        ctx.solve_periodic_gen((3, 1, 1), 1, H, S)
    assert "k-point 0" in str(e.value)


def test_non_hermitian_block_reported(ctx):
    # non-symmetric circulant -> non-Hermitian Fourier block -> DefinitenessError naming the k-point
    H = {(0, 0, 0): np.array([[1.0, 2.0], [0.0, 1.0]])}
    S = {(0, 0, 0): np.eye(2)}
    with pytest.raises(DefinitenessError) as e:
        ctx.solve_periodic_gen((2, 1, 1), 2, H, S)
    assert "non-Hermitian diagonal block at k-point 0" in str(e.value)


def test_periodic_matches_dense_expansion(ctx):
    # test_eigensolver.cpp:107-123 (1D and 3D) via an independent dense route
    rng = np.random.default_rng(64)
    for dims, m0 in (((4, 1, 1), 2), ((2, 2, 2), 3), ((5, 3, 1), 2)):
        K = int(np.prod(dims))
        H, S = {}, {}
        for k1 in range(dims[0]):
            for k2 in range(dims[1]):
                for k3 in range(dims[2]):
                    k = (k1, k2, k3)
                    mk = tuple((dims[l] - k[l]) % dims[l] for l in range(3))
                    if mk in H:
                        H[k] = H[mk].T.copy()
                        S[k] = S[mk].T.copy()
                        continue
                    a = rng.standard_normal((m0, m0))
                    b = 0.05 * rng.standard_normal((m0, m0))
                    if mk == k:
                        a = 0.5 * (a + a.T)
                        b = 0.5 * (b + b.T)
                    if k == (0, 0, 0):
                        b = b + (1.0 + m0) * np.eye(m0)
                    H[k], S[k] = a, b
        ev = np.sort(ctx.solve_periodic_gen(dims, m0, H, S).reshape(-1))

        def dense(g):
            D = np.zeros((K * m0, K * m0))
            idx = [(a, b_, c) for a in range(dims[0]) for b_ in range(dims[1]) for c in range(dims[2])]
            for i, mi in enumerate(idx):
                for j, mj in enumerate(idx):
                    k = tuple((mi[l] - mj[l]) % dims[l] for l in range(3))
                    if k in g:
                        D[i * m0:(i + 1) * m0, j * m0:(j + 1) * m0] = g[k]
            return D
        ref = sl.eigh(dense(H), dense(S), eigvals_only=True)
        assert np.max(np.abs(ev - ref)) < 1e-10 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("n", [1, 6, 12, 32, 64, 200])
def test_box_dense(ctx, oracle, n):
    rng = np.random.default_rng(61 + n)
    A = rng.standard_normal((n, n))
    H = 0.5 * (A + A.T)
    B = rng.standard_normal((n, n))
    S = B @ B.T + n * np.eye(n)
    ev = ctx.solve_box_dense(H, S)
    ref = sl.eigh(H, S, eigvals_only=True)
    assert np.max(np.abs(ev - ref)) < 1e-11 * max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(ev - oracle.solve_box_dense(H, S))) < 1e-11 * max(1.0, np.max(np.abs(ref)))


def test_box_dense_errors(ctx):
    # test_eigensolver.cpp:62-72: indefinite overlap and the size cap
    H = np.eye(3)
    S = np.eye(3)
    S[2, 2] = -1.0
    with pytest.raises(DefinitenessError):
        ctx.solve_box_dense(H, S)
    big = np.eye(40)
    S = np.eye(40)
    S[39, 39] = -1.0
    with pytest.raises(DefinitenessError):
        ctx.solve_box_dense(big, S)
    with pytest.raises(ResourceCapError):
        ctx.solve_box_dense(np.eye(8), np.eye(8), cap=4)
    ev = ctx.solve_box_dense(np.array([[-0.3]]), np.array([[0.8]]))
    assert abs(ev[0] + 0.375) < 1e-14
