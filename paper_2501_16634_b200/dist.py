"""Multi-GPU plumbing: one process per GPU, the plan space
partitioned into contiguous index ranges, one exchange step -- an all-gather
of the fixed 64-byte winner records -- followed by the deterministic
total-order reduce (objective_less, estimator.hpp:93-116).  Because the order
is strict (the identifier rank breaks every tie) the result is independent of
the number of ranks and of the gather order.

torch.distributed is the plumbing: NCCL over NVLink on the GPU box, gloo in
the CPU tests.
"""
from __future__ import annotations

import ctypes as C

from . import loom


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) slice of [0, total) for `rank` of `world`."""
    return total * rank // world, total * (rank + 1) // world


def shard_jobs(n_jobs: int, rank: int, world: int) -> tuple[int, int]:
    return n_jobs * rank // world, n_jobs * (rank + 1) // world


def _to_bytes(w: dict) -> bytes:
    return bytes(loom.winner_from_dict(w))


def _from_bytes(b: bytes) -> dict:
    return loom.Winner.from_buffer_copy(b).as_dict()


def allgather_winners(winner: dict, group=None, device=None) -> list[dict]:
    """All-gather one winner record per rank (64 bytes each)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    raw = torch.frombuffer(bytearray(_to_bytes(winner)), dtype=torch.uint8)
    if device is not None:
        raw = raw.to(device)
    out = [torch.empty_like(raw) for _ in range(world)]
    dist.all_gather(out, raw, group=group)
    return [_from_bytes(t.cpu().numpy().tobytes()) for t in out]


def combine(winners: list[dict], objective: loom.Objective) -> dict:
    """Deterministic reduce of per-rank winners; raises NoFeasibleConfigError
    when no rank found a feasible plan (optimizer.hpp:184-186)."""
    return loom.winner_reduce([loom.winner_from_dict(w) for w in winners], objective)


def empty_winner() -> dict:
    return loom.Winner().as_dict()


__all__ = ["shard_range", "shard_jobs", "allgather_winners", "combine", "empty_winner", "C"]
