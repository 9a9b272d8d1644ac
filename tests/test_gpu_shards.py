"""Multi-GPU assembly shards on one GPU: the rank-term shards of the core
Hamiltonian, assembled one after another through lt_assemble_core_dev, sum to the full H
(entries within 1e-10 relative: only the order of the rank sum differs), S is complete on
every shard (bit-exact), and lt_spectrum_dev on the summed pencil — in k-point shards —
reproduces lt_solve_core. The collectives themselves are covered by the gloo tests
(tests/test_dist_cpu.py); no rank here waits on another."""
import numpy as np
import pytest
import torch

from conftest import entries_close, two_nuclei_system
from paper_1408_3839_b200.dist import rank_term_range, shard_kinetic, shard_range, solve_core_sharded
from paper_1408_3839_b200.system import make_config

pytestmark = pytest.mark.gpu

SYSTEMS = {
    "two_per": (lambda: two_nuclei_system((12, 1, 1)), True),
    "two_box": (lambda: two_nuclei_system((6, 1, 1)), False),
    "per3d": (lambda: two_nuclei_system((5, 6, 5), n=(6, 6, 6), alphas=(3.0, 5.0), M=6), True),
    "c2": (lambda: make_config("c2"), True),
    "c4": (lambda: make_config("c4"), True),
    "c1": (lambda: make_config("c1"), False),
    "c3": (lambda: make_config("c3"), False),
}


def _shards(ds, periodic, world):
    info, kidx = ds.layout(periodic)
    count, Rtot = int(info[6]), int(info[5])
    Hs, S0 = [], None
    for q in range(world):
        H = torch.empty(count, dtype=torch.float64, device="cuda")
        S = torch.empty(count, dtype=torch.float64, device="cuda")
        r0, r1 = rank_term_range(Rtot, q, world)
        ds.assemble_shard(periodic, r0, r1, shard_kinetic(q), H.data_ptr(), S.data_ptr())
        Hs.append(H.cpu().numpy())
        s = S.cpu().numpy()
        if S0 is None:
            S0 = s
        else:
            assert np.array_equal(s, S0)
    return info, kidx, Hs, S0


@pytest.mark.parametrize("name", sorted(SYSTEMS))
@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_term_shards_sum_to_full(ctx, name, world):
    mk, periodic = SYSTEMS[name]
    sys = mk()
    ds = ctx.upload(sys)
    info, kidx, full, Sf = _shards(ds, periodic, 1)
    H1 = full[0]
    gH, gS = ctx.assemble_core(sys, periodic)
    if periodic:
        gk, gb = gH.blocks()
        assert np.array_equal(gk, kidx)
        m0 = int(info[4])
        colmajor = lambda a: a.reshape(-1, m0, m0).transpose(0, 2, 1)  # block (mu, nu) at mu + nu m0
        assert np.array_equal(gb, colmajor(H1)) and np.array_equal(gS.blocks()[1], colmajor(Sf))
    else:
        assert np.array_equal(gH.dense().reshape(-1, order="F"), H1)
    _, _, Hs, S = _shards(ds, periodic, world)
    assert np.array_equal(S, Sf)
    Hsum = np.sum(Hs, axis=0)
    ok, worst = entries_close(Hsum, H1)
    assert ok, worst
    # the spectrum of the reduced pencil, in k-point shards, against the fused solve
    ev = ctx.solve_core(sys, periodic)
    K, per_k = int(info[3]), int(info[7])
    Hd = torch.from_numpy(Hsum).cuda()
    Sd = torch.from_numpy(S).cuda()
    eig = torch.zeros((K if periodic else 1) * per_k, dtype=torch.float64, device="cuda")
    for q in range(world if periodic else 1):
        b, e = shard_range(K, q, world) if periodic else (0, 1)
        ds.spectrum(periodic, Hd.data_ptr(), Sd.data_ptr(), eig.data_ptr(), b, e)
    got = eig.cpu().numpy().reshape(ev.shape)
    # first-order bound |dl| <= ||dH||_2 / lambda_min(S) per pencil (dS = 0): the shards change
    # only the order of the rank sum, whose rounding the overlap conditioning amplifies
    dH = Hsum - H1
    if periodic:
        m0 = int(info[4])
        dims = [int(x) for x in sys.L]
        bl = lambda a: a.reshape(-1, m0, m0).transpose(0, 2, 1)
        dB, SB = bl(dH), bl(S)
        ks = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), -1).reshape(-1, 3)
        ph = np.exp(-2j * np.pi * (ks[:, None, :] * kidx[None, :, :] / np.array(dims)).sum(-1))  # [K, nblk]
        dHk = np.einsum("kb,bij->kij", ph, dB)
        Sk = np.einsum("kb,bij->kij", ph, SB)
        bound = np.array([np.linalg.norm(dHk[k], 2) / np.linalg.eigvalsh(Sk[k])[0] for k in range(len(ks))])
        err = np.abs(got - ev).max(axis=1)
    else:
        nb = int(info[2])
        bound = np.linalg.norm(dH.reshape(nb, nb, order="F"), 2) / np.linalg.eigvalsh(S.reshape(nb, nb, order="F"))[0]
        err = np.abs(got - ev).max()
    assert np.all(err <= 2.0 * bound + 1e-9), (float(np.max(err)), float(np.max(bound)))


def test_solve_core_sharded_single_rank(ctx):
    """dist.solve_core_sharded at world = 1 (no process group): identical to lt_solve_core."""
    for name in ("two_per", "c2", "two_box"):
        mk, periodic = SYSTEMS[name]
        sys = mk()
        ev = ctx.solve_core(sys, periodic)
        got = solve_core_sharded(ctx, sys, periodic).cpu().numpy().reshape(ev.shape)
        assert np.array_equal(got, ev)


def test_shard_errors(ctx):
    from paper_1408_3839_b200.native import DimensionError
    sys = two_nuclei_system((12, 1, 1))
    ds = ctx.upload(sys)
    with pytest.raises(DimensionError):
        ds.assemble_shard(True, 0, -1, True, 0, 0)


@pytest.mark.parametrize("name", ["c2", "c5", "c1", "c3"])
def test_gpu_multi_context_matches_single(ctx, name):
    # lt_create_multi / lt_solve_core_multi over the devices of this box (NCCL communicator
    # from ncclCommInitAll): the k-point split is bitwise the single-device spectrum, the
    # rank-term split (partial H per device + ncclAllReduce) within the shard-sum bound
    from golden_util import load

    from paper_1408_3839_b200.api import MultiContext
    s, periodic, d = load(name)
    ref = ctx.solve_core(s, periodic)
    m = MultiContext([0])
    assert m.ndev == 1
    ev_k = m.solve_core(s, periodic, "kpoints")
    assert np.array_equal(ev_k, ref)
    ev_r = m.solve_core(s, periodic, "rankterms")
    tol = np.maximum(1e-9, 2.0 * np.asarray(d["eig_floor"]))
    assert np.all(np.abs(ev_r.reshape(tol.shape) - ref.reshape(tol.shape)) <= tol)
    m.close()
