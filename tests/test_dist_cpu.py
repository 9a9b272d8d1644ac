"""N > 1 host logic on CPU: world_size-2 gloo ranks shard the k-points of a periodic system,
solve their shard (oracle stands in for the device), all-gather, and must reproduce the
single-rank spectrum bit for bit in k-lexicographic order (the determinism contract of
test_eigensolver.cpp:125-131)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1408_3839_b200.dist import pack_shard, padded_shard, shard_range, shard_ranges, unpack_gathered


def test_shard_ranges_partition():
    for K in (1, 2, 7, 32, 512, 4096):
        for world in (1, 2, 3, 4, 8):
            rs = shard_ranges(K, world)
            assert rs[0][0] == 0 and rs[-1][1] == K
            for (b0, e0), (b1, e1) in zip(rs, rs[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
            assert padded_shard(K, world) == max(sizes)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    """dist.solve_core_distributed itself (k-point shards + _gather_k's all-gather) on CPU
    tensors, with the oracle-backed stand-in for the engine (tests/oracle_engine.py)."""
    import sys
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import two_nuclei_system
    from oracle_engine import OracleContext
    from paper_1408_3839_b200.dist import solve_core_distributed
    octx = OracleContext()
    out = []
    for s, periodic in ((two_nuclei_system((13, 1, 1)), True), (two_nuclei_system((5, 6, 5), n=(6, 6, 6), alphas=(3.0, 5.0), M=6), True),
                        (two_nuclei_system((6, 1, 1)), False)):
        full = solve_core_distributed(octx, s, periodic)
        assert isinstance(full, torch.Tensor) and full.device.type == "cpu"
        H, S = octx.o.assemble_core(s, periodic)
        ref = octx.o.solve_periodic_ops(H, S) if periodic else octx.o.solve_box_dense(H.dense, S.dense)
        out.append((full.numpy().copy(), ref))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_kpoint_shards_match_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for full, ref in out:  # k-lexicographic order and values identical to one rank
        assert np.array_equal(full.reshape(ref.shape), ref)


def test_rank_term_ranges_partition():
    from paper_1408_3839_b200.dist import rank_term_range, shard_kinetic
    for Rtot in (50, 58, 66, 132):
        for world in (1, 2, 3, 8):
            rs = [rank_term_range(Rtot, q, world) for q in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == Rtot
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert sum(shard_kinetic(q) for q in range(world)) == 1


def _rank_term_worker(rank, world, port, q):
    """dist.solve_core_sharded itself on CPU tensors: each gloo rank assembles
    the nuclear rank terms rank_term_range(R_tot) (+ 0.5 Laplace on rank 0) into its partial H
    through the engine interface (oracle stand-in: the separable metadata, one term per rank
    term, galerkin.cpp:394-423), dist.py's all-reduce completes H, each rank solves its
    k-range and _gather_k's all-gather returns the k-lexicographic spectrum."""
    import sys
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import two_nuclei_system
    from oracle_engine import OracleContext
    from paper_1408_3839_b200.dist import solve_core_sharded
    octx = OracleContext()
    s = two_nuclei_system((13, 1, 1))
    dsys = octx.upload(s)
    info, kidx = dsys.layout(True)
    n = int(info[6])
    H = torch.zeros(n, dtype=torch.float64)
    S = torch.zeros(n, dtype=torch.float64)
    eig = torch.zeros(s.lattice_count * s.m0, dtype=torch.float64)
    full = solve_core_sharded(octx, s, True, dsys=dsys, buffers=(H, S, eig))
    Href, Sref = octx.o.assemble_core(s, True)
    m0 = s.m0
    Hsum = H.numpy().reshape(-1, m0, m0).transpose(0, 2, 1)  # column-major blocks -> [row, col]
    worst = float(np.max(np.abs(Hsum - Href.blocks)))
    scale = float(np.max(np.abs(Href.blocks)))
    if rank == 0:
        ref = octx.o.solve_periodic_ops(Href, Sref)
        q.put((worst / scale, float(np.max(np.abs(full.numpy() - ref))), int(info[5])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_rank_term_assembly_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_term_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rel, ev_err, Rtot = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert Rtot == 2 * 17  # two nuclei x (2M + 1), M = 8
    assert rel < 1e-13, rel
    assert ev_err < 1e-9, ev_err
