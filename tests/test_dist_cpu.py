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
    import sys
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import two_nuclei_system
    from oracle.binding import oracle
    o = oracle()
    s = two_nuclei_system((13, 1, 1))
    H, S = o.assemble_core(s, True)
    K = s.lattice_count
    Hb = o.block_diagonalize(s.L, s.m0, H.gen_dict())
    Sb = o.block_diagonalize(s.L, s.m0, S.gen_dict())
    b, e = shard_range(K, rank, world)
    mine = np.zeros((K, s.m0))
    for j in range(b, e):
        mine[j] = o.solve_pencil(Hb[j], Sb[j], j)
    slot = padded_shard(K, world)
    send = torch.from_numpy(pack_shard(mine, b, e, slot))
    recv = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    full = unpack_gathered(torch.stack(recv).numpy(), K, world)
    if rank == 0:
        ref = np.stack([o.solve_pencil(Hb[j], Sb[j], j) for j in range(K)])
        q.put((full, ref))
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
    full, ref = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert np.array_equal(full, ref)


def test_rank_term_ranges_partition():
    from paper_1408_3839_b200.dist import rank_term_range, shard_kinetic
    for Rtot in (50, 58, 66, 132):
        for world in (1, 2, 3, 8):
            rs = [rank_term_range(Rtot, q, world) for q in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == Rtot
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert sum(shard_kinetic(q) for q in range(world)) == 1


def _rank_term_worker(rank, world, port, q):
    """SURVEY §8(e) assembly sharding on CPU: each gloo rank forms its partial H from the
    nuclear rank terms rank_term_range(R_tot) (the oracle's separable metadata: one term per
    rank term r, weight folded into level 0, galerkin.cpp:394-423) plus 0.5 Laplace on rank 0;
    one all-reduce completes H; then the k-point shards and the all-gather."""
    import sys
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import two_nuclei_system
    from oracle.binding import oracle
    from paper_1408_3839_b200.dist import rank_term_range, shard_kinetic
    o = oracle()
    s = two_nuclei_system((13, 1, 1))
    lap = o.assemble(s, True, "laplace").gen_dict()
    nuc_op = o.assemble(s, True, "nuclear")
    terms = o.separable_terms(nuc_op)
    keys = sorted(nuc_op.gen_dict())
    Rtot = len(terms)
    r0, r1 = rank_term_range(Rtot, rank, world)
    part = np.zeros((len(keys), s.m0, s.m0))
    for i, k in enumerate(keys):
        acc = np.zeros((s.m0, s.m0))
        for t in range(r0, r1):
            acc += terms[t][0][k[0]] * terms[t][1][k[1]] * terms[t][2][k[2]]
        part[i] = (0.5 * lap[k] if shard_kinetic(rank) else 0.0) - acc
    Ht = torch.from_numpy(part)
    dist.all_reduce(Ht)
    Hsum = {k: Ht[i].numpy() for i, k in enumerate(keys)}
    Href, Sref = o.assemble_core(s, True)
    hd = Href.gen_dict()
    worst = max(float(np.max(np.abs(Hsum[k] - hd[k]))) for k in keys)
    scale = max(float(np.max(np.abs(v))) for v in hd.values())
    K = s.lattice_count
    Hb = o.block_diagonalize(s.L, s.m0, Hsum)
    Sb = o.block_diagonalize(s.L, s.m0, Sref.gen_dict())
    b, e = shard_range(K, rank, world)
    mine = np.zeros((K, s.m0))
    for j in range(b, e):
        mine[j] = o.solve_pencil(Hb[j], Sb[j], j)
    slot = padded_shard(K, world)
    send = torch.from_numpy(pack_shard(mine, b, e, slot))
    recv = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    full = unpack_gathered(torch.stack(recv).numpy(), K, world)
    if rank == 0:
        ref = o.solve_periodic_ops(Href, Sref)
        q.put((worst / scale, float(np.max(np.abs(full - ref))), Rtot))
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
