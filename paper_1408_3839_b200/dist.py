"""Multi-GPU path: one process per GPU; rank-term sharding of the assembly and k-point
sharding of the periodic spectrum.

The reference parallelises only the k-point loop (parallel_for over solve_pencil,
eigensolver.cpp:95-120, parallel.hpp:15-32) and requires results independent of the
thread count (test_eigensolver.cpp:125-131). Here each rank assembles the (small)
generating tensors and runs the lattice DFT redundantly, solves the pencils of its
contiguous k-range, and one all-gather of eigenvalues (k-lexicographic, identical to
the single-GPU order) completes the spectrum. Box systems do not shard (the dense
pencil is one factorisation): every rank computes the same spectrum (replicas).

The functions take any context whose `upload(sys)` returns an object with the
DeviceSystem methods (solve / layout / assemble_shard / spectrum, writing through buffer
pointers) and whose `torch_device` names where the buffers live, so the N > 1 paths run
unchanged on CPU tensors with the gloo backend (tests/test_dist_cpu.py, with an
oracle-backed stand-in for the engine).
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
    dev = ctx.torch_device
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
    if eig_dev is None:
        eig_dev = torch.empty(K * m0, dtype=torch.float64, device=dev)
    dsys.solve(periodic, eig_dev.data_ptr(), b, e, info)
    return _gather_k(eig_dev, K, m0, b, e, world, group)


def _gather_k(eig_dev, K: int, m0: int, b: int, e: int, world: int, group=None):
    """One all-gather of the padded k-shards -> [K, m0] in k-lexicographic order."""
    import torch
    import torch.distributed as dist

    slot = padded_shard(K, world)
    send = torch.zeros(slot * m0, dtype=torch.float64, device=eig_dev.device)
    send[: (e - b) * m0] = eig_dev[b * m0: e * m0]
    recv = torch.empty(world * slot * m0, dtype=torch.float64, device=eig_dev.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
    else:  # gloo (CPU tests): list form into views of the same buffer
        dist.all_gather(list(recv.view(world, slot * m0).unbind(0)), send, group=group)
    parts = [recv[r * slot * m0: (r * slot + (ee - bb)) * m0] for r, (bb, ee) in enumerate(shard_ranges(K, world))]
    return torch.cat(parts).view(K, m0)


def rank_term_range(Rtot: int, rank: int, world: int) -> Tuple[int, int]:
    """Nuclear rank terms [r0, r1) assembled by `rank` (contiguous, sizes differ by <= 1)."""
    return shard_range(Rtot, rank, world)


def shard_kinetic(rank: int) -> bool:
    """The Laplace part (0.5 Laplace) enters H on the leading shard only."""
    return rank == 0


def solve_core_sharded(ctx, sys, periodic: bool, group=None, dsys=None, buffers=None):
    """Assembly sharded by rank terms across the ranks of `group`, then the spectrum sharded
    by k-points. The nuclear operator is a rank-R_tot sum (galerkin.cpp:
    275-283): rank q assembles the terms rank_term_range(R_tot, q, P) (plus 0.5 Laplace on
    q = 0) into a partial H, one NCCL all-reduce (sum) of H completes it, S = Mass is complete
    on every rank; each rank then solves its k-range and one all-gather returns the full
    k-lexicographic spectrum to every rank. Box systems all-reduce the dense H and solve the
    dense pencil on every rank (replicas). Returns eigenvalues on the device ([K, m0] or [N_b])."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = ctx.torch_device
    if dsys is None:
        dsys = ctx.upload(sys)
    info, _ = dsys.layout(periodic)
    count, Rtot, K, per_k = int(info[6]), int(info[5]), int(info[3]), int(info[7])
    if buffers is None:
        buffers = (torch.empty(count, dtype=torch.float64, device=dev), torch.empty(count, dtype=torch.float64, device=dev),
                   torch.empty((K if periodic else 1) * per_k, dtype=torch.float64, device=dev))
    H, S, eig = buffers
    r0, r1 = rank_term_range(Rtot, rank, world)
    dsys.assemble_shard(periodic, r0, r1, shard_kinetic(rank), H.data_ptr(), S.data_ptr())
    if world > 1:
        dist.all_reduce(H, op=dist.ReduceOp.SUM, group=group)  # ordered on the caller's stream
    if not periodic:
        dsys.spectrum(False, H.data_ptr(), S.data_ptr(), eig.data_ptr())
        return eig
    b, e = shard_range(K, rank, world) if world > 1 else (0, K)
    dsys.spectrum(True, H.data_ptr(), S.data_ptr(), eig.data_ptr(), b, e)
    if world == 1:
        return eig.view(K, per_k)
    return _gather_k(eig, K, per_k, b, e, world, group)
