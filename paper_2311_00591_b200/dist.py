"""Multi-GPU plumbing for the Coop hot path: one process per GPU over torch.distributed.

The path shards with no exchange step: the batched search owns
independent pools, the replay sweep owns independent (trace, budget) cells.  The only
collective is the gather of per-shard result records to every rank (NCCL all-gather
over NVLink on B200; gloo in the CPU tests), done outside the timed region.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def pool_range(pools_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns global pools [r * P, (r + 1) * P)."""
    return rank * pools_per_rank, (rank + 1) * pools_per_rank


def cyclic_cells(n_cells: int, rank: int, world: int) -> list[int]:
    """Replay sweep: cell c -> rank c mod world (low-budget, slow cells spread evenly)."""
    return list(range(rank, n_cells, world))


def gather_bytes(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather equal-sized uint8 record buffers -> [world, nbytes] on every rank."""
    if world == 1:
        return local.reshape(1, -1)
    out = torch.empty((world, local.numel()), dtype=torch.uint8, device=local.device)
    if local.device.type == "cuda":
        dist.all_gather_into_tensor(out.view(-1), local.contiguous().view(-1), group=group)
    else:
        parts = list(out.unbind(0))
        dist.all_gather(parts, local.contiguous().view(-1), group=group)
    return out


def assemble_cyclic(per_rank, n_cells: int, world: int):
    """Records of rank r's cyclic cells (rank-major, [len(cyclic_cells(n, r, world)), ...]
    each, extra padding rows ignored) -> all records in global cell order."""
    first = per_rank[0]
    shape = (n_cells,) + tuple(first.shape[1:])
    out = first.new_empty(shape) if isinstance(first, torch.Tensor) else np.empty(shape, first.dtype)
    for r in range(world):
        cells = cyclic_cells(n_cells, r, world)
        if cells:
            out[cells] = per_rank[r][:len(cells)]
    return out


def gather_cells(local: torch.Tensor, n_cells: int, rec_bytes: int, world: int, group=None) -> torch.Tensor:
    """Gather per-rank cyclic cell records (padded to ceil(n_cells / world) records per
    rank) and return them in global cell order as [n_cells, rec_bytes] uint8."""
    per = (n_cells + world - 1) // world
    buf = torch.zeros(per * rec_bytes, dtype=torch.uint8, device=local.device)
    buf[:local.numel()] = local.view(-1)
    allr = gather_bytes(buf, world, group).view(world, per, rec_bytes)
    return assemble_cyclic([allr[r] for r in range(world)], n_cells, world)
