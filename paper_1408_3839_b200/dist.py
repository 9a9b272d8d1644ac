"""Multi-GPU path: one process per GPU, k-point sharding of the periodic spectrum.

The reference parallelises only the k-point loop (parallel_for over solve_pencil,
eigensolver.cpp:95-120, parallel.hpp:15-32) and requires results independent of the
thread count (test_eigensolver.cpp:125-131). Here each rank assembles the (small)
generating tensors and runs the lattice DFT redundantly, solves the pencils of its
contiguous k-range, and one all-gather of eigenvalues (k-lexicographic, identical to
the single-GPU order) completes the spectrum. Box systems do not shard (the dense
pencil is one factorisation): every rank computes the same spectrum (replicas).

The partitioning helpers are pure Python so the N > 1 logic is testable on CPU with
the gloo backend (tests/test_dist_cpu.py).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def shard_range(K: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous k-range [begin, end) of `rank`; shards differ in size by at most one."""
    base, extra = divmod(K, world)
    begin = rank * base + min(rank, extra)
    end = begin + base + (1 if rank < extra else 0)
    return begin, end


def shard_ranges(K: int, world: int) -> List[Tuple[int, int]]:
    return [shard_range(K, r, world) for r in range(world)]


def padded_shard(K: int, world: int) -> int:
    """Per-rank slot count of the all-gather buffer (max shard size)."""
    return max(e - b for b, e in shard_ranges(K, world))


def pack_shard(eig_full_rows: np.ndarray, begin: int, end: int, slot: int):
    """Rows [begin, end) of a [K, m0] array copied into a zero-padded [slot, m0] buffer."""
    m0 = eig_full_rows.shape[1]
    out = np.zeros((slot, m0), dtype=eig_full_rows.dtype)
    out[: end - begin] = eig_full_rows[begin:end]
    return out


def unpack_gathered(gathered: np.ndarray, K: int, world: int) -> np.ndarray:
    """[world, slot, m0] gathered shards -> [K, m0] in k-lexicographic order."""
    parts = [gathered[r, : e - b] for r, (b, e) in enumerate(shard_ranges(K, world))]
    return np.concatenate(parts, axis=0)


def solve_core_distributed(ctx, sys, periodic: bool, group=None, dsys=None, eig_dev=None, info=None):
    """All ranks of `group` cooperate on one system; every rank returns the full
    eigenvalue array on the host (the public multi-GPU entry point)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = torch.device("cuda", ctx.device)
    if dsys is None:
        dsys = ctx.upload(sys)
    K = sys.lattice_count if periodic else 1
    m0 = sys.m0 if periodic else sys.basis_count
    if not periodic or world == 1:
        if eig_dev is None:
            eig_dev = torch.empty(K * m0, dtype=torch.float64, device=dev)
        dsys.solve(periodic, eig_dev.data_ptr(), 0, -1, info)
        return eig_dev.view(K, m0) if periodic else eig_dev
    b, e = shard_range(K, rank, world)
    slot = padded_shard(K, world)
    if eig_dev is None:
        eig_dev = torch.empty(K * m0, dtype=torch.float64, device=dev)
    dsys.solve(periodic, eig_dev.data_ptr(), b, e, info)
    send = torch.zeros(slot * m0, dtype=torch.float64, device=dev)
    send[: (e - b) * m0] = eig_dev[b * m0: e * m0]
    recv = torch.empty(world * slot * m0, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    parts = [recv[r * slot * m0: (r * slot + (ee - bb)) * m0] for r, (bb, ee) in enumerate(shard_ranges(K, world))]
    return torch.cat(parts).view(K, m0)
