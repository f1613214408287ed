"""Multi-GPU plumbing for the data-parallel decode path (host logic only).

The path shards by sequence with no exchange step (independent
data-parallel replicas scale linearly): each rank owns a
contiguous block of sequences and its own KV caches.  torch.distributed is
used for the barrier, the max-over-ranks timing reduction and (optionally) an
all-gather of outputs for reporting -- never inside the timed data path.
"""
from __future__ import annotations

import torch


def shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Sequences [begin, end) owned by `rank` when `batch` sequences are split
    over `world` ranks in contiguous blocks of ceil(batch / world)."""
    per = (batch + world - 1) // world
    begin = min(batch, rank * per)
    end = min(batch, begin + per)
    return begin, end


def owner(batch: int, world: int, row: int) -> int:
    """The rank whose shard holds global sequence `row`."""
    return row // ((batch + world - 1) // world)


def rank_batch(global_batch: int, world: int, rank: int, scaling: str) -> int:
    """Sequences processed by `rank`: the full per-GPU batch for weak scaling,
    its shard of the fixed global batch for strong scaling."""
    if scaling == "weak":
        return global_batch
    b, e = shard(global_batch, world, rank)
    return e - b


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over the process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_outputs(out: torch.Tensor, global_batch: int) -> torch.Tensor:
    """All-gather each rank's [B_rank, ...] output block into [global_batch, ...]
    (blocks padded to ceil(global_batch / world) rows for the collective)."""
    import torch.distributed as dist
    world = dist.get_world_size()
    per = (global_batch + world - 1) // world
    pad = torch.zeros((per,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pad[: out.shape[0]] = out
    full = torch.empty((per * world,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    dist.all_gather_into_tensor(full, pad)
    return full[:global_batch]
