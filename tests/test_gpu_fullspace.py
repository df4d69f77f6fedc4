"""GPU answers over WHOLE plan spaces against the committed full-space goldens
(tests/golden/make_fullspace.py: the CPU oracle over every plan of C3, C4 and
C5), plus objective edge cases (empty / repeated criteria lists).

Every search algorithm is held to the same answer: LOOM_ALGO_AUTO (branch and
bound with the sweep as fallback, the default), LOOM_ALGO_SWEEP (every plan
tested in the fast path) and, for one binding C3 objective, LOOM_ALGO_FULL
(one plan per thread re-evaluated from scratch: 1.1e12 independent plan
evaluations)."""
import json
import random

import pytest

from conftest import cpu_threads
from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
METRICS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")


@pytest.fixture(scope="module")
def c3(ctx):
    w = W.config3(slo_us=None)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    yield w, lw
    lw.close()


def _greedy_seed(lw, obj) -> int:
    import ctypes as C
    seed = (C.c_int32 * lw.problem.n_nodes)()
    assert loom.lib().loom_greedy_seed(C.byref(lw.problem), C.byref(obj), seed) == 0
    idx = 0
    for d, r in zip(seed, lw.radix):
        idx = idx * r + d
    return idx


def _check(got, case, lw):
    assert got["plan_index"] == case["winner"]["index"], case["objective"]
    for k in METRICS:
        assert got[k] == case["winner"][k], (case["objective"], k)
    assert lw.config(got["plan_index"])["identifier"] == case["identifier"]


@pytest.mark.parametrize("algo", [loom.ALGO_AUTO, loom.ALGO_SWEEP])
def test_c3_full_space(ctx, golden, c3, algo):
    w, lw = c3
    for case in golden("c3/full_space.json")["cases"]:
        obj = loom.objective(case["objective"])
        if case["winner"] is None:
            with pytest.raises(loom.NoFeasibleConfigError):
                loom.search_argmin(ctx, lw.problem, obj, 0, None, algo)
            continue
        _check(loom.search_argmin(ctx, lw.problem, obj, 0, None, algo), case, lw)


def test_c3_binding_slo_is_not_the_greedy_seed(ctx, golden, c3):
    """The bench's headline objective: the SLO binds, so the argmin differs
    from the node-local greedy seed the kernels start from."""
    w, lw = c3
    o = {"constraint": "MIN_COST", "latency_slo_us": W.C3_BINDING_SLO_US}
    case = next(c for c in golden("c3/full_space.json")["cases"] if c["objective"] == o)
    got = loom.search_argmin(ctx, lw.problem, loom.objective(o))
    _check(got, case, lw)
    assert got["plan_index"] != _greedy_seed(lw, loom.objective(o))
    assert got["gpu_wh"] > 0 and got["latency_us"] <= W.C3_BINDING_SLO_US
    dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
    dp.search_async(0, None)
    assert dp.result() == got
    st = loom.bnb_last_stats()
    assert not st["aborted"] and not st["depth_first"] and 0 < st["child_evaluations"] < lw.total // 10 ** 4
    assert 0 < st["leaves"] <= st["child_evaluations"] and st["max_frontier"] > 0
    dp.close()


def test_c3_dropin_json_binding_slo(ctx, golden):
    w = W.config3(slo_us=W.C3_BINDING_SLO_US)
    case = next(c for c in golden("c3/full_space.json")["cases"] if c["objective"] == w.objective)
    est = loom.exhaustive_search(*w.texts(), ctx=ctx)
    assert est["plan_index"] == case["winner"]["index"] and est["identifier"] == case["identifier"]
    for k in METRICS:
        assert est[k] == case["winner"][k]


@pytest.mark.slow
def test_c3_full_space_one_plan_per_thread(ctx, golden, c3):
    """LOOM_ALGO_FULL over all 1.1e12 plans (every plan decoded and evaluated
    from scratch, no bounds): the binding-SLO MIN_COST answer."""
    w, lw = c3
    o = {"constraint": "MIN_COST", "latency_slo_us": W.C3_BINDING_SLO_US}
    case = next(c for c in golden("c3/full_space.json")["cases"] if c["objective"] == o)
    _check(loom.search_argmin(ctx, lw.problem, loom.objective(o), 0, None, loom.ALGO_FULL), case, lw)


def c4_objectives(jobs, token):
    """The objective(s) of a C4 golden column; MIN_COST_SLO: one objective per
    job, its SLO 110 % of the job's fastest plan (loom_latency_floor)."""
    if token != "MIN_COST_SLO":
        return {"constraint": token}
    objs = []
    for j in jobs:
        lw = loom.Lowered(j.dag, j.library, j.bounds)
        objs.append(W.c4_slo_objective(loom.latency_floor(lw.problem)))
        lw.close()
    return objs


@pytest.mark.parametrize("token", ["MIN_COST", "MIN_LATENCY", "MIN_COST_SLO"])
def test_c4_all_jobs(ctx, golden, token):
    """All 10,000 C4 jobs through the multi-tenant JSON call against the flat
    oracle's per-job answers."""
    g_all = golden("c4/all_jobs.json")
    gold = g_all["objectives"][token]
    jobs = W.config4(10_000)
    dags = [json.dumps(j.dag) for j in jobs]
    objs = c4_objectives(jobs, token)
    if token == "MIN_COST_SLO":
        assert [o["latency_slo_us"] for o in objs] == g_all["slo_us"]
    res = loom.exhaustive_search_batch(dags, json.dumps(jobs[0].library), objs, json.dumps(jobs[0].bounds), ctx=ctx)
    assert len(res) == len(gold) == 10_000
    mism = []
    for k, g in enumerate(gold):
        st, got = res[k]
        if g is None:
            assert st == loom.LOOM_INFEASIBLE
            continue
        assert st == 0
        if [got["plan_index"], got["latency_us"], got["gpu_wh"], got["dollars"]] != g:
            mism.append(k)
    assert not mism, mism[:10]


def test_c4_slo_binds(golden):
    """C4's binding objective: under 110 % of its fastest plan most jobs put
    work on GPUs (gpu_wh > 0), so most winners differ from the unconstrained
    MIN_COST winner (an all-CPU plan) and from the node-local greedy seed."""
    g = golden("c4/all_jobs.json")["objectives"]
    slo, cost = g["MIN_COST_SLO"], g["MIN_COST"]
    assert all(r is not None for r in slo)
    assert all(c[2] == 0.0 for c in cost)
    assert sum(1 for r, c in zip(slo, cost) if r[0] != c[0] and r[2] > 0) > 8000
    jobs = W.config4(100)
    differ = 0
    for j, r in zip(jobs, slo):
        lw = loom.Lowered(j.dag, j.library, j.bounds)
        o = loom.objective(W.c4_slo_objective(loom.latency_floor(lw.problem)))
        differ += r[0] != _greedy_seed(lw, o)
        lw.close()
    assert differ > 80


def test_c5_full_frontier(ctx, golden):
    """pareto_filter over all 1e9 C5 plans equals the flat streaming skyline."""
    gold = golden("c5/frontier.json")
    w = W.config5()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    f = loom.search_pareto_points(ctx, lw.problem)
    assert len(f) == len(gold["frontier"])
    for p, g in zip(f, gold["frontier"]):
        assert [p["plan_index"], p["latency_us"], p["gpu_wh"], p["dollars"], p["quality"]] == g


CRITERIA_CASES = [
    [],
    ["min_energy", "min_latency", "min_energy", "min_latency", "max_quality"],
    ["max_quality", "max_quality", "min_cost_dollars"],
    ["min_latency", "min_latency"],
]


def _dedup(cs):
    out = []
    for c in cs:
        if c not in out:
            out.append(c)
    return out


@pytest.mark.parametrize("crit", CRITERIA_CASES)
def test_criteria_lists_vs_oracle(ctx, crit):
    """objective_less (estimator.hpp:93-116) with an empty list orders plans by
    identifier only; repeated criteria never change the order.  Every
    algorithm against the flat oracle on C1, C2, random scenarios and C3
    slices."""
    cases = [(W.config1(), None), (W.config2(), None)]
    cases += [(W.random_scenario(s, max_nodes=4), None) for s in range(0, 40, 3)]
    w3 = W.config3(slo_us=None)
    rng = random.Random(5)
    for _ in range(3):
        b = rng.randrange(w3_total := 16 ** 10)
        cases.append((w3, (b, min(w3_total, b + (1 << 22)))))
    for w, rngs in cases:
        lw = loom.Lowered(w.dag, w.library, w.bounds)
        p = O.problem(w.dag, w.library, w.bounds)
        for extra in ({}, {"latency_slo_us": 45_000_000}):
            o = {"criteria": crit, **extra}
            b, e = rngs or (0, lw.total)
            ref = O.argmin(p, {"criteria": _dedup(crit), **extra}, b, e, threads=cpu_threads())
            for algo in (loom.ALGO_AUTO, loom.ALGO_SWEEP, loom.ALGO_FULL):
                try:
                    got = loom.search_argmin(ctx, lw.problem, loom.objective(o), b, e, algo)
                except loom.NoFeasibleConfigError:
                    got = None
                assert (got is None) == (ref is None), (w.name, o, algo)
                if got:
                    assert got["plan_index"] == ref["index"], (w.name, o, algo)
                    for k in METRICS:
                        assert got[k] == ref[k]
        lw.close()
