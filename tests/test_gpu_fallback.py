"""The default search's fallback chain, forced: a frontier that overflows its
buffer hands over to the depth-first kernel (bnb.cuh), and a depth-first
search over its evaluation budget hands over to the every-plan sweep
(DESIGN.md §3b).  Device-problem searches run the chain as one CUDA graph
whose conditional node only the frontier kernel opens; one-shot searches
launch the three kernels in order.  Every path must return the full-space
golden answer of C3 (tests/golden/c3/full_space.json).

Each case runs in a fresh process: the knobs (LOOM_BFS_CAP, LOOM_BNB_BUDGET,
LOOM_NO_GRAPH) are read once per process."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_2501_16634_b200 import loom, workloads as W
cases = json.loads(sys.argv[2])
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
ctx = loom.Context(0)
out = []
for o in cases:
    ob = loom.objective(o)
    one = loom.search_argmin(ctx, lw.problem, ob)           # one-shot: three launches
    s1 = loom.bnb_last_stats()
    dp = loom.DeviceProblem(ctx, lw.problem, ob)            # device problem: the search graph
    dp.search_async(0, None)
    two = dp.result()
    s2 = loom.bnb_last_stats()
    dp.search_async(0, None)                                # graph relaunch, same parameters
    three = dp.result()
    dp.close()
    out.append({"one": one, "two": two, "three": three, "s1": s1, "s2": s2})
print(json.dumps(out))
'''

OBJECTIVES = [{"constraint": "MIN_COST", "latency_slo_us": 40000000}, {"constraint": "MIN_LATENCY"},
              {"constraint": "MIN_DOLLARS", "latency_slo_us": 40000000}]


def _run(env_extra, cases):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), json.dumps(cases)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def _golden(golden, o):
    return next(c for c in golden("c3/full_space.json")["cases"] if c["objective"] == o)["winner"]


def _same(got, win):
    assert got["plan_index"] == win["index"]
    for k in ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality"):
        assert got[k] == win[k], k


@pytest.mark.parametrize("graph", [True, False])
def test_frontier_overflow_hands_over_to_depth_first(golden, graph):
    env = {"LOOM_BFS_CAP": "64"}
    if not graph:
        env["LOOM_NO_GRAPH"] = "1"
    for o, r in zip(OBJECTIVES, _run(env, OBJECTIVES)):
        win = _golden(golden, o)
        for key in ("one", "two", "three"):
            _same(r[key], win)
        if o["constraint"] != "MIN_LATENCY":  # MIN_LATENCY's frontier stays one entry wide
            assert r["s1"]["depth_first"] and r["s2"]["depth_first"], (o, r["s1"], r["s2"])


def test_depth_first_budget_hands_over_to_sweep(golden):
    o = OBJECTIVES[0]
    r = _run({"LOOM_BFS_CAP": "64", "LOOM_BNB_BUDGET": "4096"}, [o])[0]
    win = _golden(golden, o)
    for key in ("one", "two", "three"):
        _same(r[key], win)
    assert r["s1"]["aborted"] and r["s2"]["aborted"], (r["s1"], r["s2"])


def test_graph_and_plain_launches_agree(golden):
    """No knobs: the graph path and the plain path (LOOM_NO_GRAPH) return the
    same records on every objective of the full-space golden."""
    cases = [c["objective"] for c in golden("c3/full_space.json")["cases"] if c["winner"] is not None][:8]
    a = _run({}, cases)
    b = _run({"LOOM_NO_GRAPH": "1"}, cases)
    for o, x, y in zip(cases, a, b):
        win = _golden(golden, o)
        for r in (x, y):
            for key in ("one", "two", "three"):
                _same(r[key], win)
        assert not x["s2"]["depth_first"] and not x["s2"]["aborted"]
