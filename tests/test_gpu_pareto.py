"""GPU Pareto frontier (pareto_filter over every plan in enumeration order,
optimizer.hpp:153-171) against the reference goldens and the oracle."""
import random

import pytest

from conftest import cpu_threads
from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu


def _front(ctx, w, begin=0, end=None):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    return lw, loom.search_pareto_points(ctx, lw.problem, begin, end)


def test_c1_frontier(ctx, golden):
    ref = [r["plan_index"] for r in golden("c1/results.json")["pareto"]["frontier"]]
    lw, f = _front(ctx, W.config1())
    assert [p["plan_index"] for p in f] == ref == [42, 162]
    for p in f:
        e = lw.evaluate(p["plan_index"])
        assert (p["dollars"], p["gpu_wh"], p["latency_us"], p["quality"]) == (
            e["dollars"], e["gpu_wh"], e["latency_us"], e["quality"])
    assert loom.search_pareto(ctx, lw.problem) == [42, 162]


def test_random_scenario_frontiers(ctx, golden):
    gold = golden("random/results.json")
    n = 0
    for seed, entry in gold.items():
        if "pareto" not in entry:
            continue
        _, f = _front(ctx, W.random_scenario(int(seed), max_nodes=4))
        assert [p["plan_index"] for p in f] == entry["pareto"], seed
        n += 1
    assert n > 50


def test_c5_reduced_frontiers(ctx, golden):
    for k, entry in golden("c5/reduced_pareto.json").items():
        _, f = _front(ctx, W.config5(n_nodes=int(k)))
        assert [p["plan_index"] for p in f] == entry["frontier"]


def test_c5_slices_vs_oracle(ctx):
    w = W.config5()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for b, e in [(0, 3_000_000), (123_456_789, 126_456_789), (lw.total - 2_500_001, lw.total)]:
        ora = O.pareto(p, b, e, threads=cpu_threads())
        got = loom.search_pareto_points(ctx, lw.problem, b, e)
        assert [g["plan_index"] for g in got] == [o["index"] for o in ora]
        for g, o in zip(got, ora):
            assert (g["dollars"], g["gpu_wh"], g["latency_us"], g["quality"]) == (
                o["dollars"], o["gpu_wh"], o["latency_us"], o["quality"])


def test_c5_full_space_properties(ctx):
    """1e9 plans: the frontier is mutually non-dominated, every point is the
    exact estimate of its plan, and random plans are each dominated by or
    equal to some frontier point."""
    w = W.config5()
    lw, f = _front(ctx, w)
    assert lw.total == 1_000_000_000 and len(f) > 10
    assert all(loom.pareto_filter_points(ctx, f))
    idx = [p["plan_index"] for p in f]
    assert idx == sorted(idx)
    rng = random.Random(1)
    for p in rng.sample(f, min(50, len(f))):
        e = lw.evaluate(p["plan_index"])
        assert (p["dollars"], p["gpu_wh"], p["latency_us"]) == (e["dollars"], e["gpu_wh"], e["latency_us"])
    P = O.problem(w.dag, w.library, w.bounds)
    import numpy as np
    F = np.array([(p["dollars"], p["gpu_wh"], p["latency_us"]) for p in f])
    for i in [rng.randrange(lw.total) for _ in range(3000)]:
        e = O.estimates(P, i, i + 1)[0]
        x = np.array([e["dollars"], e["gpu_wh"], e["latency_us"]])
        le = (F <= x).all(axis=1)
        assert le.any(), i  # some frontier point is no worse on every axis


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_frontier_merge(ctx, world):
    """per-rank frontiers of contiguous index shards, merged by
    one device filter of their union, equal the whole-space frontier (C5 with
    7 tasks: 1e7 plans, every shard boundary inside a group)."""
    from paper_2501_16634_b200 import dist as D
    w = W.config5(n_nodes=7)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    whole = loom.search_pareto_points(ctx, lw.problem)
    shards = [loom.search_pareto_points(ctx, lw.problem, *D.shard_range(lw.total, r, world)) for r in range(world)]
    merged = D.combine_frontiers(shards, lambda pts: loom.pareto_filter_points(ctx, pts))
    assert merged == whole and len(whole) > 10
