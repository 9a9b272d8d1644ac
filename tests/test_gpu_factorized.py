"""GPU parity of the factorized Fourier path: separable metadata of the
assembled operators, separable_residual, solve_periodic_factorized, and
factorized_block_diagonalize — against Oracle-X and the reference's own tests restated
(test_factorized.cpp, test_eigensolver.cpp:148-185, test_galerkin.cpp:399-410)."""
import numpy as np
import pytest

from conftest import chain_system, entries_close, two_nuclei_system
from paper_1408_3839_b200.api import StructureError

pytestmark = pytest.mark.gpu


def expand(terms, dims, m0):
    """FactorizedDiagonalizer::expand (factorized_diag.cpp:80-96)."""
    gen = {}
    for k1 in range(dims[0]):
        for k2 in range(dims[1]):
            for k3 in range(dims[2]):
                blk = np.zeros((m0, m0))
                for t in terms:
                    blk = blk + (t[0][k1] * t[1][k2]) * t[2][k3]
                if np.max(np.abs(blk)) > 0:
                    gen[(k1, k2, k3)] = blk
    return gen


def random_terms(rng, dims, m0, n):
    return [[rng.standard_normal((dims[l], m0, m0)) for l in range(3)] for _ in range(n)]


def test_identity_at_zero_lag(ctx):
    # test_factorized.cpp: Factorized.IdentityAtZeroLag
    dims, m0 = (3, 2, 2), 2
    term = []
    for l in range(3):
        seq = np.zeros((dims[l], m0, m0))
        seq[0] = np.eye(m0)
        term.append(seq)
    bd = ctx.factorized_block_diagonalize(3, dims, m0, [term])
    assert np.max(np.abs(bd - np.eye(m0))) <= 1e-14


@pytest.mark.parametrize("rank,dims", [(1, (3, 2, 2)), (3, (4, 3, 2)), (5, (5, 1, 3))])
def test_factorized_matches_general_path(ctx, rank, dims):
    # Factorized.RankOneMatchesGeneralPath / RankThreeMatchesGeneralPath
    rng = np.random.default_rng(40 + rank)
    m0 = 2
    terms = random_terms(rng, dims, m0, rank)
    fact = ctx.factorized_block_diagonalize(3, dims, m0, terms)
    general = ctx.bc_block_diagonalize(dims, m0, expand(terms, dims, m0))
    assert np.max(np.abs(fact - general)) <= 1e-12


def spd_circulant(rng, L, m0):
    gen = {}
    for k in range(L // 2 + 1):
        b = 0.2 * rng.standard_normal((m0, m0))
        if k == 0:
            gen[(0, 0, 0)] = 0.5 * (b + b.T) + (2.0 + m0) * np.eye(m0)
        elif 2 * k == L:
            gen[(k, 0, 0)] = 0.5 * (b + b.T)
        else:
            gen[(k, 0, 0)] = b
            gen[(L - k, 0, 0)] = b.T.copy()
    return gen


def level_terms_from_gen(gen, L, m0):
    seq0 = np.stack([gen.get((k, 0, 0), np.zeros((m0, m0))) for k in range(L)])
    return [[seq0, np.ones((1, m0, m0)), np.ones((1, m0, m0))]]


def test_mass_only_pencil_is_unit(ctx):
    # test_eigensolver.cpp:148-166 FactorizedSolve.MassOnlyPencilIsUnit
    rng = np.random.default_rng(66)
    L, m0 = 4, 2
    gen = spd_circulant(rng, L, m0)
    terms = level_terms_from_gen(gen, L, m0)
    ev = ctx.solve_periodic_factorized_gen((L, 1, 1), m0, gen, gen, terms, terms)
    assert np.max(np.abs(ev - 1.0)) <= 1e-12


def test_metadata_residual_is_checked(ctx):
    # test_eigensolver.cpp:168-185 FactorizedSolve.MetadataResidualIsChecked
    rng = np.random.default_rng(67)
    L, m0 = 4, 2
    gen = spd_circulant(rng, L, m0)
    terms = level_terms_from_gen(gen, L, m0)
    terms[0][0][1][0, 0] += 0.37
    with pytest.raises(StructureError) as e:
        ctx.solve_periodic_factorized_gen((L, 1, 1), m0, gen, gen, terms, terms)
    assert "factorization residual 0.370000 exceeds tolerance" in str(e.value)


def systems():
    return [
        ("chain7", chain_system(7, [0.6, 1.7], n=8, nbar=8, M=6, b=4.0)),
        ("two_nuclei_x", two_nuclei_system(L=(8, 1, 1), n=(16, 8, 8), alphas=(1.2, 3.0, 0.9, 5.0))),
        ("two_nuclei_xy", two_nuclei_system(L=(6, 5, 1), n=(8, 8, 8), alphas=(2.0, 4.0, 3.0, 6.0))),
    ]


@pytest.mark.parametrize("name,s", systems())
def test_operator_metadata_matches_oracle(ctx, oracle, name, s):
    # SeparableMetadataReassembles (test_galerkin.cpp:399-410) and the metadata itself
    for kind, rank in (("mass", 1), ("laplace", 3), ("nuclear", s.rank_total)):
        op = ctx.assemble(s, True, kind)
        ref = oracle.assemble(s, True, kind)
        assert op.coefficient_rank == rank == ref.coefficient_rank
        assert ctx.separable_residual(op) <= 1e-13 * max(1.0, np.max(np.abs(ref.blocks)))
        got, exp = op.separable(), oracle.separable_terms(ref)
        assert len(got) == len(exp) == rank
        scale = max(float(np.max(np.abs(x))) for t in exp for x in t)
        for gt, et in zip(got, exp):
            for l in range(3):
                ok, worst = entries_close(gt[l], et[l], scale=scale)
                assert ok, (name, kind, l, worst)
        oracle.free(ref)


@pytest.mark.parametrize("name,s", systems())
def test_solve_periodic_factorized_matches(ctx, oracle, name, s):
    # the combined H keeps valid metadata (Combine.PeriodicLinearCombination) and the
    # factorized spectrum equals the general path's
    lap, nuc, S = (ctx.assemble(s, True, k) for k in ("laplace", "nuclear", "mass"))
    H = ctx.combine(0.5, lap, -1.0, nuc)
    assert H.coefficient_rank == 3 + s.rank_total
    assert ctx.separable_residual(H) <= 1e-12 * max(1.0, np.max(np.abs(H.blocks()[1])))
    ev = ctx.solve_periodic_factorized(H, S)
    general = ctx.solve_periodic(H, S)
    rH, rS = oracle.assemble_core(s, True)
    ref = oracle.solve_periodic_factorized_ops(rH, rS)
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(ev - general)) <= 1e-10 * scale
    assert np.max(np.abs(ev - ref)) <= 1e-9 * scale
    # assemble_core's H, S carry the same metadata
    Hc, Sc = ctx.assemble_core(s, True)
    assert ctx.separable_residual(Hc) <= 1e-12 * max(1.0, np.max(np.abs(Hc.blocks()[1])))
    assert np.max(np.abs(ctx.solve_periodic_factorized(Hc, Sc) - ref)) <= 1e-9 * scale


def test_factorized_requires_metadata(ctx):
    s = chain_system(7, [0.6, 1.7], n=8, nbar=8, M=6, b=4.0)
    Hb = ctx.assemble(s, False, "mass")
    with pytest.raises(StructureError, match="operators must be periodic assemblies"):
        ctx.solve_periodic_factorized(Hb, Hb)


def test_box_circulant_defect(ctx, oracle):
    # galerkin.cpp:445-454 against the oracle's box and periodic nuclear operators
    s = chain_system(7, [0.6, 1.7], n=8, nbar=8, M=6, b=4.0)
    rel, D = ctx.box_circulant_defect(s, want_defect=True)
    box = oracle.assemble(s, False, "nuclear")
    per = oracle.assemble(s, True, "nuclear")
    L, m0 = per.L, per.m0
    g = per.gen_dict()
    K = L[0] * L[1] * L[2]
    dense = np.zeros((K * m0, K * m0))
    idx = [(a, b, c) for a in range(L[0]) for b in range(L[1]) for c in range(L[2])]
    for i, mi in enumerate(idx):
        for j, mj in enumerate(idx):
            k = tuple((mi[l] - mj[l]) % L[l] for l in range(3))
            if k in g:
                dense[i * m0:(i + 1) * m0, j * m0:(j + 1) * m0] = g[k]
    ref = box.dense - dense
    assert abs(rel - np.linalg.norm(ref) / np.linalg.norm(box.dense)) <= 1e-9 * rel
    assert np.max(np.abs(D - ref)) <= 1e-10 * np.max(np.abs(box.dense))
    oracle.free(box)
    oracle.free(per)
