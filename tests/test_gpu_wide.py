"""The frontier search's other instantiations: bfs_kernel<32, int64_t, 0>
runs for DAGs of more than 16 nodes and for any DAG whose latencies can
exceed 2^30 us, with the criteria read from the parameters.  Wide random
DAGs (17-22 nodes, 1e10-1e14 plans) against the oracle's C branch and bound
(validated against the flat loop, tests/test_oracle.py); long-wall DAGs
(work scaled so walls reach hours) against the flat oracle."""
import json

import pytest

from conftest import cpu_threads
from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
METRICS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")
WIDE_SEEDS = [2, 5, 10, 15, 17, 25, 37, 57]


def _objectives(p):
    fastest = O.argmin_bnb(p, {"constraint": "MIN_LATENCY"}, cpu_threads())[0]["latency_us"]
    return [{"constraint": "MIN_COST"}, {"constraint": "MIN_LATENCY"}, {"constraint": "MAX_QUALITY"},
            {"constraint": "MIN_DOLLARS"},
            {"constraint": "MIN_COST", "latency_slo_us": fastest * 115 // 100},
            {"constraint": "MAX_QUALITY", "latency_slo_us": fastest * 130 // 100},
            {"criteria": ["min_latency", "min_cost_dollars"]}]


def _same(got, ref, tag):
    assert got["plan_index"] == ref["index"], tag
    for k in METRICS:
        assert got[k] == ref[k], (tag, k)


@pytest.mark.parametrize("seed", WIDE_SEEDS)
def test_wide_dags_vs_oracle_branch_and_bound(ctx, seed):
    w = W.random_scenario(seed, max_nodes=22, max_fanout=1, max_paths=1)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    assert lw.problem.n_nodes > 16
    p = O.problem(w.dag, w.library, w.bounds)
    for o in _objectives(p):
        ref, _ = O.argmin_bnb(p, o, cpu_threads())
        ob = loom.objective(o)
        got = loom.search_argmin(ctx, lw.problem, ob)
        _same(got, ref, (seed, o, "one-shot"))
        dp = loom.DeviceProblem(ctx, lw.problem, ob)
        dp.search_async(0, None)
        _same(dp.result(), ref, (seed, o, "graph"))
        dp.close()
    lw.close()


def _long(seed):
    w = W.random_scenario(seed, max_nodes=6)
    dag = json.loads(json.dumps(w.dag))
    for node in dag["nodes"]:  # walls of hours: latencies beyond 2^30 us
        node["work_units"] *= 300.0
        if node.get("min_chunk"):
            node["min_chunk"] *= 300.0
    return dag, w


@pytest.mark.parametrize("seed", [1, 4, 7, 11, 13, 21])
def test_long_walls_vs_flat_oracle(ctx, seed):
    dag, w = _long(seed)
    lw = loom.Lowered(dag, w.library, w.bounds)
    p = O.problem(dag, w.library, w.bounds)
    if lw.total == 0:
        pytest.skip("empty space")
    for o in ({"constraint": "MIN_COST"}, {"constraint": "MIN_LATENCY"}, {"constraint": "MAX_QUALITY"}):
        ref = O.argmin(p, o, threads=cpu_threads())
        got = loom.search_argmin(ctx, lw.problem, loom.objective(o))
        _same(got, ref, (seed, o))
    lw.close()
