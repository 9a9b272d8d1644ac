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
