"""Multi-GPU plumbing: one process per GPU, the plan space
partitioned into contiguous index ranges, one exchange step -- an all-gather
of the fixed 64-byte winner records -- followed by the deterministic
total-order reduce (objective_less, estimator.hpp:93-116); for the Pareto
frontier, an all-gather of the per-rank frontiers and one device filter of
their union.  Because the order
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


def search_shard(ctx, problem, objective, rank: int, world: int) -> dict:
    """This rank's shard search: argmin of its plan-index range plus the
    greedy seed as a common incumbent (loom_search_argmin_shard), so every
    rank prunes like a whole-space search.  Returns an empty (found == 0)
    record when nothing in the shard, nor the incumbent, is feasible."""
    lw_total = C.c_uint64()
    loom._check(loom.lib().loom_problem_total(C.byref(problem), C.byref(lw_total)))
    begin, end = shard_range(lw_total.value, rank, world)
    try:
        return loom.search_argmin_shard(ctx, problem, objective, begin, end)
    except loom.NoFeasibleConfigError:
        return empty_winner()


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


# ---- Pareto (config 5): per-rank frontiers -> one frontier ---------------
def _points_bytes(points: list[dict]) -> bytes:
    arr = (loom.Point * max(1, len(points)))()
    for i, p in enumerate(points):
        for k in ("plan_index", "dollars", "gpu_wh", "latency_us", "quality"):
            setattr(arr[i], k, p[k])
    return bytes(arr)[: 40 * len(points)]


def allgather_frontiers(points: list[dict], group=None, device=None) -> list[list[dict]]:
    """All-gather every rank's local frontier (40-byte loom_point records):
    one all-gather of the counts, then one padded all-gather of the points."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = torch.tensor([len(points)], dtype=torch.int64, device=device)
    counts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    width = 40 * max(1, max(counts))
    raw = bytearray(width)
    mine = _points_bytes(points)
    raw[: len(mine)] = mine
    t = torch.frombuffer(raw, dtype=torch.uint8)
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    res = []
    for k, o in enumerate(out):
        b = o.cpu().numpy().tobytes()
        res.append([loom.Point.from_buffer_copy(b, 40 * i).as_dict() for i in range(counts[k])])
    return res


def combine_frontiers(frontiers: list[list[dict]], keep_fn) -> list[dict]:
    """Global frontier from per-shard frontiers.  A point that no plan of the
    whole space dominates is not dominated inside its own shard either, so the
    union of the shard frontiers holds the global frontier; keep_fn (the
    device filter, loom.pareto_filter_points bound to a ctx) removes the
    points another shard dominates.  Output in enumeration (index) order,
    like pareto_filter's stable input order (optimizer.hpp:163-170)."""
    union = [p for f in frontiers for p in f]
    keep = keep_fn(union) if union else []
    return sorted((p for p, k in zip(union, keep) if k), key=lambda p: p["plan_index"])


__all__ = ["shard_range", "shard_jobs", "allgather_winners", "combine", "empty_winner", "allgather_frontiers",
           "combine_frontiers", "C"]
