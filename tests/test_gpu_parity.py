"""GPU parity: the sm_100a search through the C ABI against the reference's
golden vectors (tests/golden) and the CPU oracle on the same inputs.  The
bar is bit-exact: same selected plan (identifier / plan index), same integer
latency and quality, bit-identical doubles."""
import random

import json

import pytest

from conftest import cpu_threads
from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
TOKENS = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]
METRICS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")


def _check_ref(got: dict, ref: dict, lw: loom.Lowered) -> None:
    assert lw.config(got["plan_index"])["identifier"] == ref["identifier"]
    for k in METRICS:
        assert got[k] == ref[k], k


def _check_oracle(got: dict, ora: dict) -> None:
    assert got["plan_index"] == ora["index"]
    for k in METRICS:
        assert got[k] == ora[k], k


def _search(ctx, w, obj, begin=0, end=None, algo=0):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    return lw, loom.search_argmin(ctx, lw.problem, loom.objective(obj), begin, end, algo)


@pytest.mark.parametrize("token", TOKENS)
@pytest.mark.parametrize("algo", [0, 1])
def test_c1_tokens(ctx, golden, token, algo):
    w = W.config1()
    lw, got = _search(ctx, w, {"constraint": token}, algo=algo)
    _check_ref(got, golden("c1/results.json")["tokens"][token]["exhaustive"], lw)


@pytest.mark.parametrize("floor", range(6))
def test_c1_floors(ctx, golden, floor):
    w = W.config1()
    ref = golden("c1/results.json")["floors"][str(floor)]
    obj = {"constraint": "MIN_COST", "quality_floor": floor}
    if ref.get("error"):
        with pytest.raises(loom.NoFeasibleConfigError, match="no configuration satisfies the quality floor and bounds"):
            _search(ctx, w, obj)
    else:
        lw, got = _search(ctx, w, obj)
        _check_ref(got, ref, lw)


@pytest.mark.parametrize("token", TOKENS)
def test_c1_dropin_json(ctx, golden, token):
    """loom::exhaustive_search on reference-format JSON (the drop-in call)."""
    w = W.config1()
    ref = golden("c1/results.json")["tokens"][token]["exhaustive"]
    got = loom.exhaustive_search(w.dag, w.library, {"constraint": token}, w.bounds, ctx=ctx)
    assert got["identifier"] == ref["identifier"]
    assert got["config"]["nodes"] == ref["config"]["nodes"]
    for k in METRICS:
        assert got[k] == ref[k]
    assert got["plans"] == 168


def test_c1_min_latency_prefers_hybrid(ctx):
    """test_fixture.cpp:72-94: MIN_LATENCY breaks the 77 s tie by energy toward gpu+cpu."""
    w = W.config1()
    got = loom.exhaustive_search(w.dag, w.library, "MIN_LATENCY", w.bounds, ctx=ctx)
    stt = got["config"]["nodes"]["t1_speech_to_text"]["placements"]
    assert {p["sku"] for p in stt} == {"cpu-epyc", "gpu-a100"}
    assert got["latency_us"] == 76_750_000


def test_random_scenarios_all_tokens(ctx, golden):
    gold = golden("random/results.json")
    n = 0
    for seed, entry in gold.items():
        w = W.random_scenario(int(seed), max_nodes=4)
        lw = loom.Lowered(w.dag, w.library, w.bounds)
        for token, ref in entry.get("search", {}).items():
            for algo in (0, 1):
                if ref.get("error"):
                    with pytest.raises(loom.NoFeasibleConfigError):
                        loom.search_argmin(ctx, lw.problem, loom.objective(token), 0, None, algo)
                else:
                    _check_ref(loom.search_argmin(ctx, lw.problem, loom.objective(token), 0, None, algo), ref, lw)
                    n += 1
        if "floor2" in entry:
            ref = entry["floor2"]
            obj = loom.objective({"constraint": w.objective["constraint"], "quality_floor": 2})
            if ref.get("error"):
                with pytest.raises(loom.NoFeasibleConfigError):
                    loom.search_argmin(ctx, lw.problem, obj)
            else:
                _check_ref(loom.search_argmin(ctx, lw.problem, obj), ref, lw)
    assert n > 400


def test_c2_full_space(ctx, golden):
    g = golden("c2/results.json")
    w = W.config2()
    lw, got = _search(ctx, w, w.objective)
    assert lw.total == g["total"] == 1_207_296
    _check_ref(got, g["config"], lw)
    _check_ref(loom.search_argmin(ctx, lw.problem, loom.objective("MIN_COST")), g["min_cost"], lw)
    _check_ref(loom.search_argmin(ctx, lw.problem, loom.objective({"constraint": "MIN_DOLLARS", "quality_floor": 3})),
               g["min_dollars_q3"], lw)


def test_c2_dropin_json(ctx, golden):
    g = golden("c2/results.json")["config"]
    w = W.config2()
    got = loom.exhaustive_search(w.dag, w.library, w.objective, w.bounds, ctx=ctx)
    assert got["identifier"] == g["identifier"]
    assert got["gpu_wh"] == g["gpu_wh"] and got["latency_us"] == g["latency_us"]


def test_c2_random_subranges_vs_oracle(ctx):
    """Unaligned ranges exercise the edge (full re-evaluation) path and the
    subrow path together."""
    w = W.config2()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    rng = random.Random(2)
    for token in TOKENS:
        for _ in range(3):
            b = rng.randrange(lw.total - 1)
            e = min(lw.total, b + rng.randrange(1, 300_000))
            obj = {"constraint": token, "quality_floor": rng.choice([None, 2, 3])}
            ora = O.argmin(p, obj, b, e, threads=cpu_threads())
            if ora is None:
                with pytest.raises(loom.NoFeasibleConfigError):
                    loom.search_argmin(ctx, lw.problem, loom.objective(obj), b, e)
                continue
            for algo in (0, 1):
                _check_oracle(loom.search_argmin(ctx, lw.problem, loom.objective(obj), b, e, algo), ora)


def test_c3_slices(ctx, golden):
    g = golden("c3/slices.json")
    w = W.config3()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    for s in g["slices"]:
        ref = s["result"]
        if not ref["found"]:
            with pytest.raises(loom.NoFeasibleConfigError):
                loom.search_argmin(ctx, lw.problem, loom.objective(g["objective"]), s["begin"], s["end"])
            continue
        got = loom.search_argmin(ctx, lw.problem, loom.objective(g["objective"]), s["begin"], s["end"])
        assert got["plan_index"] == ref["winner"]["plan_index"]
        _check_ref(got, ref["winner"], lw)
    s = g["slice_no_slo"]
    got = loom.search_argmin(ctx, lw.problem, loom.objective("MIN_COST"), s["begin"], s["end"])
    _check_ref(got, s["result"]["winner"], lw)


def test_c3_hierarchical_equals_full_eval_on_large_slices(ctx):
    """Two independent GPU algorithms (max-plus hierarchical vs one plan per
    thread from scratch) agree on 64M-plan slices, plus the oracle on 4M."""
    w = W.config3()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    obj = loom.objective(w.objective)
    rng = random.Random(9)
    def outcome(b, e, algo):
        try:
            return loom.search_argmin(ctx, lw.problem, obj, b, e, algo)
        except loom.NoFeasibleConfigError:
            return None

    feasible = 0
    for _ in range(6):
        b = rng.randrange(lw.total - (1 << 26))
        a0, a1 = outcome(b, b + (1 << 26), 0), outcome(b, b + (1 << 26), 1)
        assert a0 == a1
        feasible += a0 is not None
    # a slice that holds feasible plans (around the golden slice's winner)
    c = 123_457_159_103
    a0, a1 = outcome(c - (1 << 25), c + (1 << 25), 0), outcome(c - (1 << 25), c + (1 << 25), 1)
    assert a0 is not None and a0 == a1
    for b in (c - 2_000_000, 777_777_777):  # one slice with feasible plans, one without
        ora = O.argmin(p, w.objective, b, b + 4_000_000, threads=cpu_threads())
        got = outcome(b, b + 4_000_000, 0)
        if ora is None:
            assert got is None
        else:
            _check_oracle(got, ora)


def test_c4_batch(ctx, golden):
    gold = golden("c4/jobs.json")["jobs"]
    jobs = W.config4(96)
    lws = [loom.Lowered(j.dag, j.library, j.bounds) for j in jobs]
    out = loom.search_argmin_batch(ctx, [lw.problem for lw in lws], [loom.objective(j.objective) for j in jobs])
    for k, ((st, got), lw) in enumerate(zip(out, lws)):
        assert st == 0
        if str(k) in gold:
            _check_ref(got, gold[str(k)]["result"], lw)
        elif k < 40:
            p = O.problem(jobs[k].dag, jobs[k].library, jobs[k].bounds)
            _check_oracle(got, O.argmin(p, jobs[k].objective, threads=cpu_threads()))


def test_c4_batch_json_and_lowered(ctx, golden):
    """The multi-tenant entry points (one JSON call; lowered handles + one
    objective) return exactly the per-job batch results, which are pinned to
    the reference goldens above.  Includes an invalid DAG (per-job status)."""
    gold = golden("c4/jobs.json")["jobs"]
    jobs = W.config4(64)
    dags = [j.dag for j in jobs] + [{"nodes": [{"id": "x"}], "edges": []}, {"nodes": [], "edges": []}]
    lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
    res = loom.exhaustive_search_batch(dags, lib_t, jobs[0].objective, bounds_t, ctx=ctx)
    assert len(res) == 66 and res.feasible() == 64
    assert res.status[64] == loom.LOOM_INVALID and res.status[65] == loom.LOOM_INFEASIBLE
    batch = loom.LoweredBatch(dags[:64], lib_t, bounds_t)
    res2 = loom.search_lowered_batch(ctx, batch, loom.objective(jobs[0].objective))
    per_job = loom.search_argmin_batch(ctx, [batch[k].problem for k in range(64)],
                                       [loom.objective(j.objective) for j in jobs])
    for k in range(64):
        assert res[k] == res2[k] == per_job[k]
        if str(k) in gold:
            _check_ref(res[k][1], gold[str(k)]["result"], batch[k])
    batch.close()


def test_resident_problem_async(ctx):
    w = W.config3()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    obj = loom.objective(w.objective)
    dp = loom.DeviceProblem(ctx, lw.problem, obj)
    b, e = 10_000_000_019, 10_000_000_019 + (1 << 27)
    dp.search_async(b, e)
    got = dp.result()
    assert got == loom.search_argmin(ctx, lw.problem, obj, b, e, 1)
    dp.close()


def test_infeasible_and_empty(ctx):
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    with pytest.raises(loom.NoFeasibleConfigError):
        loom.search_argmin(ctx, lw.problem, loom.objective({"constraint": "MIN_COST", "quality_floor": 9}))
    with pytest.raises(loom.NoFeasibleConfigError):
        loom.search_argmin(ctx, lw.problem, loom.objective("MIN_COST"), 100, 100)
    with pytest.raises(loom.NoFeasibleConfigError):
        loom.exhaustive_search({"nodes": [], "edges": []}, w.library, "MIN_COST", w.bounds, ctx=ctx)
    assert ctx.launches > 0


@pytest.mark.parametrize("cfg,ranks", [("c1", 3), ("c2", 8), ("c3", 8), ("c5", 4)])
def test_shard_search_with_incumbent_combines_to_argmin(ctx, cfg, ranks):
    """loom_search_argmin_shard: every rank searches its index range plus the
    greedy seed as a common incumbent; the reduce over ranks equals the
    whole-space search, and each rank's result is in its range or is the
    incumbent."""
    from paper_2501_16634_b200 import dist as D
    w = {"c1": W.config1, "c2": W.config2, "c3": W.config3, "c5": W.config5}[cfg]()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    obj = loom.objective(w.objective if cfg != "c5" else {"constraint": "MIN_COST"})
    total = lw.total if cfg != "c3" else 1 << 36  # C3: a 2^36-plan prefix keeps the test short
    full = loom.search_argmin(ctx, lw.problem, obj, 0, total)
    import ctypes as C
    sd = (C.c_int32 * lw.problem.n_nodes)()
    assert loom.lib().loom_greedy_seed(C.byref(lw.problem), C.byref(obj), sd) == 0
    seed = 0
    for i in range(lw.problem.n_nodes):
        seed = seed * lw.problem.radix[i] + sd[i]
    winners = []
    for r in range(ranks):
        b, e = D.shard_range(total, r, ranks)
        try:
            got = loom.search_argmin_shard(ctx, lw.problem, obj, b, e)
        except loom.NoFeasibleConfigError:
            got = D.empty_winner()
        if got["found"]:
            assert b <= got["plan_index"] < e or got["plan_index"] == seed
        winners.append(got)
    if seed < total:
        best = D.combine(winners, obj)
        assert best["plan_index"] == full["plan_index"]
        for k in METRICS:
            assert best[k] == full[k]
    else:  # the incumbent lies outside the searched prefix: the reduce is over prefix u {seed}
        ref = D.combine([full, lw.evaluate(seed) | {"found": 1}] if _feasible(lw.evaluate(seed), w) else [full], obj)
        assert D.combine(winners, obj)["plan_index"] == ref["plan_index"]


def _feasible(est: dict, w) -> bool:
    slo = w.objective.get("latency_slo_us") if isinstance(w.objective, dict) else None
    return slo is None or est["latency_us"] <= slo


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_energy_first_under_binding_slos_vs_oracle(ctx, seed):
    """The energy-first sweep flags every context whose best option beats the
    running bound; with a tight latency SLO the low-energy plans are mostly
    infeasible, so the flagged path (two-criteria re-test, lazy latency
    coefficients, exact scan) carries the search.  C3-shaped problems with
    SLOs at the 1st / 10th / 50th latency percentile of a sample, MIN_COST and
    MIN_DOLLARS, 2^22-plan slices, against the CPU oracle."""
    w0 = W.config3(seed=seed, slo_us=None)
    lw = loom.Lowered(w0.dag, w0.library, w0.bounds)
    p = O.problem(w0.dag, w0.library, w0.bounds)
    rng = random.Random(seed)
    sample = sorted(lw.evaluate(rng.randrange(lw.total))["latency_us"] for _ in range(400))
    for pct in (0.01, 0.10, 0.50):
        slo = sample[int(pct * (len(sample) - 1))]
        for token in ("MIN_COST", "MIN_DOLLARS"):
            obj = {"constraint": token, "latency_slo_us": slo}
            b = rng.randrange(lw.total - (1 << 22))
            e = b + (1 << 22)
            ref = O.argmin(p, obj, b, e, threads=cpu_threads())  # None: nothing feasible
            if ref is None:
                with pytest.raises(loom.NoFeasibleConfigError):
                    loom.search_argmin(ctx, lw.problem, loom.objective(obj), b, e)
                continue
            got = loom.search_argmin(ctx, lw.problem, loom.objective(obj), b, e)
            _check_oracle(got, ref)


def _subset_problem(lw, keep: dict):
    """A copy of a lowered problem keeping only the listed options of some
    nodes ({node: [option, ...]}); other nodes keep all theirs."""
    import ctypes as C
    pr = lw.problem
    n = pr.n_nodes
    keep_all = []
    off = 0
    radix = []
    for i in range(n):
        opts = keep.get(i, list(range(pr.radix[i])))
        keep_all += [off + o for o in opts]
        radix.append(len(opts))
        off += pr.radix[i]
    held = []

    def arr(ct, vals):
        a = (ct * max(1, len(vals)))(*vals)
        held.append(a)
        return C.cast(a, C.POINTER(ct))

    q = loom.Problem()
    q.n_nodes, q.n_edges = n, pr.n_edges
    q.radix = arr(C.c_int32, radix)
    for f, ct in (("wall_us", C.c_int64), ("gpu_wh", C.c_double), ("cpu_wh", C.c_double),
                  ("dollars", C.c_double), ("quality", C.c_int32)):
        setattr(q, f, arr(ct, [getattr(pr, f)[k] for k in keep_all]))
    # identifier ranks re-ranked within each node (order preserved)
    lex = []
    off = 0
    for i in range(n):
        opts = keep.get(i, list(range(pr.radix[i])))
        ranks = [pr.lexrank[off + o] for o in opts]
        order = sorted(range(len(opts)), key=lambda k: ranks[k])
        rr = [0] * len(opts)
        for r, k in enumerate(order):
            rr[k] = r
        lex += rr
        off += pr.radix[i]
    q.lexrank = arr(C.c_int32, lex)
    # mixed-radix identifier weights in sorted node-id order, recomputed for the new radices
    w = [0] * n
    order = sorted(range(n), key=lambda i: pr.lex_weight[i])  # ascending weight = least significant first
    acc = 1
    for i in order:
        w[i] = acc
        acc *= radix[i]
    q.lex_weight = arr(C.c_uint64, w)
    q.edge_from = arr(C.c_int32, [pr.edge_from[e] for e in range(pr.n_edges)])
    q.edge_to = arr(C.c_int32, [pr.edge_to[e] for e in range(pr.n_edges)])
    q._held = held
    return q


@pytest.mark.parametrize("keep", [{7: list(range(15))}, {8: list(range(12))}, {7: [0, 3, 5], 9: list(range(11))}])
def test_sweep_shapes_hierarchical_equals_full_eval(ctx, keep):
    """C3 with some suffix nodes cut to odd / narrower radices, so the sweep
    takes its unpaired and non-unrolled forms: the hierarchical search equals
    the one-plan-per-thread re-evaluation on 2^24-plan slices."""
    w = W.config3()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    q = _subset_problem(lw, keep)
    obj = loom.objective(w.objective)
    total = C_total(q)
    rng = random.Random(11)
    for _ in range(4):
        b = rng.randrange(total - (1 << 24))
        res = []
        for algo in (0, 1):
            try:
                res.append(loom.search_argmin(ctx, q, obj, b, b + (1 << 24), algo))
            except loom.NoFeasibleConfigError:
                res.append(None)
        assert res[0] == res[1]
    full = [loom.search_argmin(ctx, q, loom.objective("MIN_COST"), 0, 1 << 24, a) for a in (0, 1)]
    assert full[0] == full[1]


def C_total(q) -> int:
    import ctypes as C
    t = C.c_uint64()
    assert loom.lib().loom_problem_total(C.byref(q), C.byref(t)) == 0
    return t.value
