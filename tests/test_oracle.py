"""The CPU oracle (oracle/lower.py + oracle/flat_oracle.c) pinned against the
golden vectors produced by the compiled reference (tests/golden/make_golden.py)
and, where they are published, against the reference's own known answers
(test_fixture.cpp, test_cli.cpp)."""
import pytest

from conftest import cpu_threads
from oracle import oracle as O
from paper_2501_16634_b200 import workloads as W

TOKENS = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]


def _same(oracle_row: dict, ref: dict, p) -> None:
    assert O.identifier(p, oracle_row["index"]) == ref["identifier"]
    for k in ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality"):
        assert oracle_row[k] == ref[k], k  # bit-exact doubles


@pytest.fixture(scope="module")
def c1():
    w = W.config1()
    return w, O.problem(w.dag, w.library, w.bounds)


def test_c1_lowering_matches_reference(c1, golden):
    w, p = c1
    low = golden("c1/results.json")["lowered"]
    assert p.lowered.radix == [len(n["options"]) for n in low["nodes"]] == [1, 14, 1, 12]
    for i, node in enumerate(low["nodes"]):
        for k, o in enumerate(node["options"]):
            plan = p.lowered.plans[i][k]
            assert (plan["wall_us"], plan["gpu_wh"], plan["cpu_wh"], plan["dollars"]) == (
                o["wall_us"], o["gpu_wh"], o["cpu_wh"], o["dollars"])
            assert p.lowered.tokens[i][k] == o["identifier"]
            assert p.lowered.quality[i][k] == o["quality"]
    assert [p.lowered.node_ids[i] for i in p.lowered.topo] == low["topological_order"]


def test_c1_every_estimate_matches_reference(c1, golden):
    w, p = c1
    ref = golden("c1/results.json")["estimates"]
    mine = O.estimates(p, 0, 168)
    for r, m in zip(ref, mine):
        assert tuple(r[1:]) == (m["latency_us"], m["gpu_wh"], m["cpu_wh"], m["total_wh"], m["dollars"],
                                m["quality"])


@pytest.mark.parametrize("token", TOKENS)
def test_c1_argmin_matches_reference(c1, golden, token):
    w, p = c1
    ref = golden("c1/results.json")["tokens"][token]["exhaustive"]
    _same(O.argmin(p, {"constraint": token}, threads=1), ref, p)
    _same(O.argmin(p, {"constraint": token}, threads=7), ref, p)


def test_c1_known_answers(c1):
    """SURVEY.md §8c / test_cli.cpp:73,96,154-157 / test_fixture.cpp:56-94."""
    w, p = c1
    cost = O.argmin(p, {"constraint": "MIN_COST"})
    assert O.identifier(p, cost["index"]) == (
        "t0_frame_extraction=opencv-frame-extractor[cpu-epyc:16x1]p1;"
        "t1_speech_to_text=whisper[cpu-epyc:16x4]p1;t2_object_detection=clip[cpu-epyc:16x1]p1;"
        "t3_summarization=nvlm[gpu-a100:2x4]p1;")
    assert cost["latency_us"] == 83_000_000
    assert f"{cost['gpu_wh']:.6f}" == "33.777778"
    lat = O.argmin(p, {"constraint": "MIN_LATENCY"})
    assert lat["latency_us"] == 76_750_000
    assert f"{lat['gpu_wh']:.6f}" == "41.555556"
    assert "whisper[gpu-a100:2x1+cpu-epyc:16x1]p1" in O.identifier(p, lat["index"])


@pytest.mark.parametrize("floor", [0, 1, 2, 3, 4, 5])
def test_c1_quality_floor(c1, golden, floor):
    w, p = c1
    ref = golden("c1/results.json")["floors"][str(floor)]
    got = O.argmin(p, {"constraint": "MIN_COST", "quality_floor": floor})
    if ref.get("error"):
        assert ref["error"] == "NoFeasibleConfigError" and got is None
    else:
        _same(got, ref, p)


def test_c1_pareto_matches_reference(c1, golden):
    w, p = c1
    ref = golden("c1/results.json")["pareto"]["frontier"]
    got = O.pareto(p, threads=3)
    assert [g["index"] for g in got] == [r["plan_index"] for r in ref] == [42, 162]


def test_random_scenarios_match_reference(golden):
    gold = golden("random/results.json")
    import hashlib
    import json
    checked = 0
    for seed, entry in gold.items():
        w = W.random_scenario(int(seed), max_nodes=4)
        assert hashlib.sha256(json.dumps([w.dag, w.library, w.bounds], sort_keys=True).encode()).hexdigest()[
               :16] == entry["digest"], "generator drift"
        p = O.problem(w.dag, w.library, w.bounds)
        assert p.lowered.radix == entry["radix"]
        for token, ref in entry.get("search", {}).items():
            got = O.argmin(p, {"constraint": token}, threads=cpu_threads())
            if ref.get("error"):
                assert got is None
            else:
                _same(got, ref, p)
                checked += 1
        if "floor2" in entry:
            ref = entry["floor2"]
            got = O.argmin(p, {"constraint": w.objective["constraint"], "quality_floor": 2})
            assert (got is None) == bool(ref.get("error"))
            if got:
                _same(got, ref, p)
        if "pareto" in entry:
            assert [g["index"] for g in O.pareto(p, threads=2)] == entry["pareto"]
    assert checked > 200


def test_c4_jobs_match_reference(golden):
    gold = golden("c4/jobs.json")["jobs"]
    for j, w in enumerate(W.config4(len(gold))):
        p = O.problem(w.dag, w.library, w.bounds)
        _same(O.argmin(p, w.objective, threads=cpu_threads()), gold[str(j)]["result"], p)


def test_c5_reduced_pareto_matches_reference(golden):
    gold = golden("c5/reduced_pareto.json")
    for n, entry in gold.items():
        w = W.config5(n_nodes=int(n))
        p = O.problem(w.dag, w.library, w.bounds)
        assert p.total == entry["total"]
        assert [g["index"] for g in O.pareto(p, threads=cpu_threads())] == entry["frontier"]


def test_c3_slices_match_reference(golden):
    gold = golden("c3/slices.json")
    w = W.config3()
    p = O.problem(w.dag, w.library, w.bounds)
    for s in gold["slices"]:
        got = O.argmin(p, gold["objective"], s["begin"], s["end"], threads=cpu_threads())
        ref = s["result"]
        if not ref["found"]:
            assert got is None
        else:
            assert got["index"] == ref["winner"]["plan_index"]
            _same(got, ref["winner"], p)
    s = gold["slice_no_slo"]
    got = O.argmin(p, {"constraint": "MIN_COST"}, s["begin"], s["end"], threads=cpu_threads())
    _same(got, s["result"]["winner"], p)
