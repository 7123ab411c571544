"""Batch data-parallel helpers.

Independent registrations shard across ranks (one process per GPU); the only
collective is a final all-gather of the per-pair CostReport rows.  Single
volumes are not split (a semi-Lagrangian back-trace has no bounded halo):
replicas only.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_pairs", "gather_terms", "sharded_cost_and_grad"]


def shard_pairs(n_pairs: int, rank: int, world: int) -> list:
    """Contiguous, balanced split of pair indices (pair p keeps seed base+p on any rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    lo = (n_pairs * rank) // world
    hi = (n_pairs * (rank + 1)) // world
    return list(range(lo, hi))


def gather_terms(local: torch.Tensor, n_pairs: int) -> torch.Tensor:
    """All-gather [B_local, 4] CostReport rows into [n_pairs, 4] in pair order."""
    world = dist.get_world_size()
    counts = [len(shard_pairs(n_pairs, r, world)) for r in range(world)]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def sharded_cost_and_grad(compute, n_pairs: int):
    """Run ``compute(pairs) -> (grad [b,...], terms [b,4])`` on this rank's shard and
    gather every pair's terms.  ``compute`` is the device path in production."""
    rank, world = dist.get_rank(), dist.get_world_size()
    pairs = shard_pairs(n_pairs, rank, world)
    g, terms = compute(pairs)
    return pairs, g, gather_terms(terms, n_pairs)
