"""greedy_search (optimizer.hpp:227-291) on the GPU against the compiled
reference's greedy_search: same selected ConfigPoint, bit-identical metrics,
same errors (empty DAG, no option meeting the floor)."""
import pytest

from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
TOKENS = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]
METRICS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")


def _same(got, ref):
    assert got["identifier"] == ref["identifier"]
    for k in METRICS:
        assert got[k] == ref[k], k


def _run(ctx, w, obj, ref):
    if ref.get("error"):
        with pytest.raises(loom.LoomError) as ei:
            loom.greedy_search(w.dag, w.library, obj, w.bounds, ctx=ctx)
        assert ei.value.code == ref["error"]
        assert str(ei.value) == ref["message"]
    else:
        _same(loom.greedy_search(w.dag, w.library, obj, w.bounds, ctx=ctx), ref)


@pytest.mark.parametrize("token", TOKENS)
def test_c1(ctx, golden, token):
    _run(ctx, W.config1(), {"constraint": token}, golden("c1/results.json")["tokens"][token]["greedy"])


def test_random_scenarios(ctx, golden):
    g = golden("greedy/results.json")["random"]
    for seed, entry in g.items():
        w = W.random_scenario(int(seed), max_nodes=5)
        for t in TOKENS:
            _run(ctx, w, {"constraint": t}, entry[t])
        _run(ctx, w, {"constraint": w.objective["constraint"], "quality_floor": 2}, entry["floor2"])


def test_c2_c3_c4(ctx, golden):
    g = golden("greedy/results.json")
    w = W.config2()
    for t in TOKENS:
        _run(ctx, w, {"constraint": t}, g["c2"][t])
    _run(ctx, w, w.objective, g["c2"]["config"])
    w = W.config3(slo_us=None)
    for t in TOKENS:
        _run(ctx, w, {"constraint": t}, g["c3"][t])
    for j, w in enumerate(W.config4(16)):
        _run(ctx, w, w.objective, g["c4"][str(j)])


def test_empty_dag(ctx):
    w = W.config1()
    with pytest.raises(loom.NoFeasibleConfigError, match="cannot search an empty dag"):
        loom.greedy_search({"nodes": [], "edges": []}, w.library, "MIN_COST", w.bounds, ctx=ctx)
