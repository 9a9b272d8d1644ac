"""GPU dense box pencil beyond the library eigensolver (eigensolver.cpp:12-35):
the persistent tridiagonalisation (k_sytrd*) and the Sturm multisection on the tridiagonal
(k_tridiag_eig3), checked against LAPACK (scipy) on matrices that stress each piece —
tridiagonal inputs with S = I pass through the reduction unchanged, so the eigenvalue kernel
sees them exactly; dense pencils exercise the reduction. Bound: max |lambda - lambda_ref|
<= 1e-12 ||T|| (both sides backward stable; n eps ||T|| for n = 1024 is 2.3e-13 ||T||)."""
import numpy as np
import pytest
import scipy.linalg as sl

pytestmark = pytest.mark.gpu


def tridiag_cases(rng, n):
    m = (n - 1) // 2
    yield "random", rng.uniform(-1, 1, n), rng.uniform(-1, 1, n - 1)
    yield "graded", 10.0 ** (-np.arange(n) / (n / 12)), 0.5 * 10.0 ** (-np.arange(n - 1) / (n / 12))
    yield "wilkinson", np.abs(np.arange(n) - m).astype(float), np.ones(n - 1)
    yield "cluster", 1.0 + 1e-10 * rng.uniform(-1, 1, n), 1e-8 * rng.uniform(0, 1, n - 1)
    yield "range", 10.0 ** rng.uniform(-8, 8, n) * rng.choice([-1, 1], n), 10.0 ** rng.uniform(-8, 8, n - 1)
    e = rng.uniform(-1, 1, n - 1)
    e[::7] = 0.0  # split blocks
    yield "split", rng.uniform(-1, 1, n), e
    yield "scaled", 1e150 * rng.uniform(-1, 1, n), 1e150 * rng.uniform(-1, 1, n - 1)
    yield "tiny", 1e-150 * rng.uniform(-1, 1, n), 1e-150 * rng.uniform(-1, 1, n - 1)


@pytest.mark.parametrize("n", [33, 100, 257, 1024])
def test_tridiagonal_eigenvalues(ctx, n):
    rng = np.random.default_rng(n)
    for name, d, e in tridiag_cases(rng, n):
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        ev = ctx.solve_box_dense(T, np.eye(n))
        ref = sl.eigvalsh_tridiagonal(d, e)
        norm = max(np.max(np.abs(d)), np.max(np.abs(e)))
        err = np.max(np.abs(ev - ref)) / norm
        assert err <= 1e-12, (name, err)
        assert np.all(np.diff(ev) >= 0), name


@pytest.mark.parametrize("n", [40, 129, 300, 512, 513, 777, 1024])
def test_dense_pencil_reduction(ctx, oracle, n):
    rng = np.random.default_rng(7 + n)
    A = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (A + A.T)
    B = rng.uniform(-1, 1, (n, n))
    S = B @ B.T / n + np.eye(n)
    ev = ctx.solve_box_dense(H, S)
    ref = sl.eigh(H, S, eigvals_only=True)
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(ev - ref)) / scale < 1e-11
    if n <= 300:
        assert np.max(np.abs(ev - oracle.solve_box_dense(H, S))) / scale < 1e-11


@pytest.mark.parametrize("n", [33, 65, 191, 1000])
def test_dense_pencil_reduction_edges(ctx, n):
    # sizes off the 64-column panel grid (partial leaf blocks, odd pitch -> padded TMA copies)
    rng = np.random.default_rng(100 + n)
    A = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (A + A.T)
    Q, _ = np.linalg.qr(rng.uniform(-1, 1, (n, n)))
    S = (Q * np.logspace(-3, 0, n)) @ Q.T
    S = 0.5 * (S + S.T)
    ev = ctx.solve_box_dense(H, S)
    ref = sl.eigh(H, S, eigvals_only=True)
    assert np.max(np.abs(ev - ref)) <= 1e-12 * np.max(np.abs(ref)) * n


@pytest.mark.parametrize("n", [33, 65])
def test_dense_pencil_ill_conditioned_overlap(ctx, n):
    # cond(S) = 1e10, as near-linear-dependent bases produce: every FP64 algorithm (LAPACK
    # sygvd included) is off the exact eigenvalues by ~cond(L) u ||A||; the GPU must be as
    # close to a 40-digit reference (mpmath) as LAPACK, within a factor 8
    mp = pytest.importorskip("mpmath")
    rng = np.random.default_rng(100 + n)
    A = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (A + A.T)
    Q, _ = np.linalg.qr(rng.uniform(-1, 1, (n, n)))
    S = (Q * np.logspace(-10, 0, n)) @ Q.T
    S = 0.5 * (S + S.T)
    mp.mp.dps = 40
    Lm = mp.cholesky(mp.matrix(S.tolist()))
    Li = mp.inverse(Lm)
    hp = np.array(sorted(float(x) for x in mp.eigsy(Li * mp.matrix(H.tolist()) * Li.T)[0]))
    ev = ctx.solve_box_dense(H, S)
    lap = sl.eigh(H, S, eigvals_only=True)
    assert np.max(np.abs(ev - hp)) <= 8 * np.max(np.abs(lap - hp)), (np.max(np.abs(ev - hp)), np.max(np.abs(lap - hp)))


@pytest.mark.parametrize("n", [40, 700])
def test_dense_pencil_indefinite_overlap_raises(ctx, n):
    # eigensolver.cpp:20-24: LLT fails -> DefinitenessError, as the reference
    from paper_1408_3839_b200.api import DefinitenessError
    rng = np.random.default_rng(n)
    H = np.eye(n)
    Q, _ = np.linalg.qr(rng.uniform(-1, 1, (n, n)))
    d = np.ones(n)
    d[n // 2] = -1e-3
    S = (Q * d) @ Q.T
    with pytest.raises(DefinitenessError, match="not positive definite"):
        ctx.solve_box_dense(H, 0.5 * (S + S.T))
