"""The CPU oracle (oracle/lower.py + oracle/flat_oracle.c) pinned against the
golden vectors produced by the compiled reference (tests/golden/make_golden.py)
and, where they are published, against the reference's own known answers
(test_fixture.cpp, test_cli.cpp)."""
from pathlib import Path

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


# ---------------------------------------------------------------------------
# The oracle's exact branch and bound (flat_oracle.c: oracle_argmin_bnb), which
# produces the full-space C3 goldens, pinned to the reference's goldens and to
# the flat per-plan loop.
def test_bnb_matches_reference_c1(c1, golden):
    w, p = c1
    res = golden("c1/results.json")
    for token in TOKENS:
        got, _ = O.argmin_bnb(p, {"constraint": token}, threads=3)
        _same(got, res["tokens"][token]["exhaustive"], p)
    for floor, ref in res["floors"].items():
        got, _ = O.argmin_bnb(p, {"constraint": "MIN_COST", "quality_floor": int(floor)})
        if ref.get("error"):
            assert got is None
        else:
            _same(got, ref, p)


def test_bnb_matches_reference_random_and_c2(golden):
    gold = golden("random/results.json")
    checked = 0
    for seed, entry in gold.items():
        w = W.random_scenario(int(seed), max_nodes=4)
        p = O.problem(w.dag, w.library, w.bounds)
        for token, ref in entry.get("search", {}).items():
            got, _ = O.argmin_bnb(p, {"constraint": token}, threads=2)
            if ref.get("error"):
                assert got is None
            else:
                _same(got, ref, p)
                checked += 1
    assert checked > 200
    w = W.config2()
    p = O.problem(w.dag, w.library, w.bounds)
    for o in (w.objective, {"constraint": "MIN_COST"}, {"constraint": "MAX_QUALITY"},
              {"constraint": "MIN_DOLLARS", "latency_slo_us": 300_000_000}):
        got, _ = O.argmin_bnb(p, o)
        ref = O.argmin(p, o, threads=cpu_threads())
        assert got == ref, o
    ref = golden("c2/results.json")
    assert ref  # c2 goldens pin O.argmin (test_c2_* above); bnb == argmin here


C3_RESTRICTIONS = [
    [0, 3, 8, 11, 14],          # 5^10 plans: CPU and GPU options of both sizes
    [1, 6, 9, 15],              # 4^10
    [2, 5, 7, 10, 12, 13],      # 6^10 (~6e7)
]


@pytest.mark.parametrize("keep", C3_RESTRICTIONS)
def test_bnb_matches_flat_loop_on_restricted_c3(keep):
    """Restricted C3 spaces the flat per-plan loop finishes: the branch and
    bound equals it under binding / non-binding SLOs and every token."""
    w = W.config3(slo_us=None)
    full = O.problem(w.dag, w.library, w.bounds)
    p = O.subproblem(full, [keep] * 10)
    objs = [{"constraint": "MIN_COST"}, {"constraint": "MIN_LATENCY"}, {"constraint": "MAX_QUALITY"},
            {"constraint": "MIN_DOLLARS", "latency_slo_us": 45_000_000}]
    lat = O.argmin(p, {"constraint": "MIN_LATENCY"}, threads=cpu_threads())["latency_us"]
    cpu = O.argmin(p, {"constraint": "MIN_COST"}, threads=cpu_threads())["latency_us"]
    for f in (0.2, 0.5, 0.8, 0.97):  # SLOs between the fastest plan and the cheapest
        objs.append({"constraint": "MIN_COST", "latency_slo_us": int(lat + f * (cpu - lat))})
    objs.append({"constraint": "MIN_COST", "latency_slo_us": lat - 1})  # infeasible
    for o in objs:
        got, _ = O.argmin_bnb(p, o)
        ref = O.argmin(p, o, threads=cpu_threads())
        assert got == ref, o


def test_c3_full_space_goldens(golden):
    """The committed full-space C3 answers (make_fullspace.py) are what the
    oracle's branch and bound returns; the binding SLOs do bind."""
    gold = golden("c3/full_space.json")
    w = W.config3(slo_us=None)
    p = O.problem(w.dag, w.library, w.bounds)
    seed = gold["cases"][0]["winner"]["index"]  # MIN_COST: the all-CPU greedy seed
    for case in gold["cases"]:
        got, _ = O.argmin_bnb(p, case["objective"])
        if case["winner"] is None:
            assert got is None
            continue
        assert {k: got[k] for k in case["winner"]} == case["winner"]
        assert O.identifier(p, got["index"]) == case["identifier"]
        slo = case["objective"].get("latency_slo_us")
        if case["objective"]["constraint"] == "MIN_COST" and slo is not None and slo < 47_258_723:
            assert got["index"] != seed and got["gpu_wh"] > 0 and got["latency_us"] <= slo


def test_c3_all_cpu_subspace(golden):
    """MIN_COST ranks on quantize(gpu_wh) first; every C3 option
    lowered onto a GPU has quantize(gpu_wh) >= 1 and every CPU option 0, so the
    full-space argmin lies in the 8^10-plan all-CPU subspace, which the flat
    per-plan loop searches exhaustively (~10 s on 8 threads)."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_fullspace import all_cpu_subspace

    w = W.config3(slo_us=None)
    p = O.problem(w.dag, w.library, w.bounds)
    for plans, opts in zip(p.lowered.plans, p.lowered.options):
        assert sum(pl["gpu_wh"] == 0.0 for pl in plans) == 8
        for pl, op in zip(plans, opts):
            assert pl["gpu_wh"] == 0.0 or pl["gpu_wh"] * op["path_count"] * 1e9 >= 0.5  # llround >= 1
    sub, full_index = all_cpu_subspace(p)
    assert sub.total == 8 ** 10
    r = O.argmin(sub, {"constraint": "MIN_COST"}, threads=cpu_threads())
    gold = golden("c3/full_space.json")
    assert full_index(r["index"]) == gold["all_cpu_subspace"]["full_index"] == gold["cases"][0]["winner"]["index"]
    assert r["latency_us"] == gold["cases"][0]["winner"]["latency_us"] == 47_258_723


def test_c4_all_jobs_golden_pinned_to_reference(golden):
    """The flat oracle's 10,000-job C4 golden agrees with every job the
    compiled reference answered (c4/jobs.json), and re-derives on a sample."""
    allj = golden("c4/all_jobs.json")["objectives"]["MIN_COST"]
    ref = golden("c4/jobs.json")["jobs"]
    jobs = W.config4(10_000)
    for k, r in ref.items():
        p = O.problem(jobs[int(k)].dag, jobs[int(k)].library, jobs[int(k)].bounds)
        assert O.identifier(p, allj[int(k)][0]) == r["result"]["identifier"]
        assert allj[int(k)][1:] == [r["result"]["latency_us"], r["result"]["gpu_wh"], r["result"]["dollars"]]
    lat = golden("c4/all_jobs.json")["objectives"]["MIN_LATENCY"]
    for k in (17, 4321, 9999):
        p = O.problem(jobs[k].dag, jobs[k].library, jobs[k].bounds)
        for token, g in (("MIN_COST", allj[k]), ("MIN_LATENCY", lat[k])):
            r = O.argmin(p, {"constraint": token}, threads=cpu_threads())
            assert [r["index"], r["latency_us"], r["gpu_wh"], r["dollars"]] == g


def test_c5_frontier_golden_properties(golden):
    """The committed 1e9-plan C5 frontier: ascending plan indices, each point
    the oracle's estimate of its plan, no point dominated by another."""
    import numpy as np
    g = golden("c5/frontier.json")["frontier"]
    w = W.config5()
    p = O.problem(w.dag, w.library, w.bounds)
    idx = [r[0] for r in g]
    assert idx == sorted(idx) and len(g) == 2322
    for r in g[::97]:
        e = O.estimates(p, r[0], r[0] + 1)[0]
        assert [e["latency_us"], e["gpu_wh"], e["dollars"], e["quality"]] == r[1:]
    F = np.array([[r[3], r[2], r[1], -r[4]] for r in g], dtype=np.float64)
    for i in range(len(F)):
        le = (F <= F[i]).all(axis=1) & (F < F[i]).any(axis=1)
        assert not le.any(), i
