"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED reference
compiled into oracle/_ref/ (oracle/Makefile).  Needs /root/reference, i.e.
runs only in the build container; the outputs are committed so the GPU box
(which has no /root/reference) can check against them.

    make -C oracle ref && python tests/golden/make_golden.py [--only c1,c2,...]

Every number written here comes from a call into the reference's own
functions (see oracle/ref_harness.cpp): LexiconPlanner::plan,
exhaustive_search, greedy_search, node_options + plan_node_execution,
estimate, pareto_filter, and the multi-threaded range driver over
estimate / meets_quality_floor / objective_less.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2501_16634_b200 import workloads as W  # noqa: E402

GOLD = ROOT / "tests" / "golden"
FIX = Path("/root/reference/proj/fixtures/video_understanding")
TOKENS = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]


def digest(w: W.Workload) -> str:
    return hashlib.sha256(json.dumps([w.dag, w.library, w.bounds], sort_keys=True).encode()).hexdigest()[:16]


def dump(path: Path, obj) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(obj, indent=1, sort_keys=True) + "\n")


def search(w: W.Workload, obj: dict, mode: str = "exhaustive") -> dict:
    rc, out = O.ref_search(w.dag, w.library, obj, w.bounds, mode)
    out["status"] = rc
    return out


def cluster_bounds(cluster: dict, max_fanout=4, max_paths=2) -> dict:
    # loom_main.cpp:67-78 bounds_for: per-sku largest pool and total capacity;
    # every (node, sku) entry of the cluster file is one pool (cluster.hpp:145-171).
    pool, total = {}, {}
    for node in cluster["nodes"]:
        for s in node["skus"]:
            pool[s["sku_id"]] = max(pool.get(s["sku_id"], 0), s["units"])
            total[s["sku_id"]] = total.get(s["sku_id"], 0) + s["units"]
    return {"max_fanout": max_fanout, "max_paths": max_paths, "sku_pool_cap": pool, "sku_total_cap": total}


def make_c1() -> None:
    spec = json.loads((FIX / "job_declarative.json").read_text())
    lib = json.loads((FIX / "profiles.json").read_text())
    lex = json.loads((FIX / "lexicon.json").read_text())
    rc, planned = O.ref_plan(spec, lib, lex)
    assert rc == 0, planned
    d = GOLD / "c1"
    dump(d / "dag.json", {"nodes": planned["nodes"], "edges": planned["edges"]})
    dump(d / "library.json", planned["library"])
    dump(d / "bounds.json", cluster_bounds(json.loads((FIX / "cluster.json").read_text())))
    w = W.config1()
    res = {"digest": digest(w), "tokens": {}, "floors": {}, "pins": {}}
    for t in TOKENS:
        res["tokens"][t] = {"exhaustive": search(w, {"constraint": t}), "greedy": search(w, {"constraint": t}, "greedy")}
    for f in range(0, 6):
        res["floors"][str(f)] = search(w, {"constraint": "MIN_COST", "quality_floor": f})
    rc, fr = O.ref_pareto(w.dag, w.library, w.bounds)
    res["pareto"] = fr
    rc, low = O.ref_lower(w.dag, w.library, w.bounds)
    res["lowered"] = low
    rc, ests = O.ref_enumerate(w.dag, w.library, w.bounds, 0, 168)
    res["estimates"] = ests
    # the published pins (Table 2) as plan estimates
    for pin in ["pin_stt_cpu.json", "pin_stt_gpu.json", "pin_stt_gpu_cpu.json"]:
        res["pins"][pin] = json.loads((FIX / pin).read_text())
    res["min_latency_job"] = json.loads((FIX / "job_min_latency.json").read_text())["constraint"]
    dump(d / "results.json", res)


def make_c2() -> None:
    w = W.config2()
    rc, planned = O.ref_plan(W.C2_SPEC, w.library, W.C2_LEXICON)
    keys = ("id", "capability", "work_units", "splittable", "min_chunk", "multi_path", "path_quality_ceiling")
    same = [{k: n.get(k) for k in keys} for n in planned["nodes"]] == [{k: n.get(k) for k in keys}
                                                                        for n in w.dag["nodes"]]
    assert same and planned["edges"] == w.dag["edges"], "C2 generator drifted from the reference planner"
    res = {"digest": digest(w), "planner_agrees": True}
    rc, low = O.ref_lower(w.dag, w.library, w.bounds)
    res["radix"] = [len(n["options"]) for n in low["nodes"]]
    res["total"] = low["total_count"]
    t0 = time.time()
    res["config"] = search(w, w.objective)
    res["config_seconds_single_thread"] = time.time() - t0
    res["min_cost"] = search(w, {"constraint": "MIN_COST"})
    res["min_dollars_q3"] = search(w, {"constraint": "MIN_DOLLARS", "quality_floor": 3})
    dump(GOLD / "c2" / "results.json", res)


def make_random(n: int = 80) -> None:
    out = {}
    for seed in range(n):
        w = W.random_scenario(seed, max_nodes=4)
        rc, low = O.ref_lower(w.dag, w.library, w.bounds)
        total = low["total_count"]
        entry = {"digest": digest(w), "total": total, "radix": [len(x["options"]) for x in low["nodes"]]}
        if total <= 200_000:
            entry["search"] = {t: search(w, {"constraint": t}) for t in TOKENS}
            entry["floor2"] = search(w, {"constraint": w.objective["constraint"], "quality_floor": 2})
        if total <= 3000:
            rc, fr = O.ref_pareto(w.dag, w.library, w.bounds)
            entry["pareto"] = [r["plan_index"] for r in fr["frontier"]]
        out[str(seed)] = entry
    dump(GOLD / "random" / "results.json", out)


def make_greedy(n: int = 80) -> None:
    """Reference greedy_search on the random scenarios (all tokens, plus a
    quality floor), C2, C3 (no SLO: the reference has none) and C4 jobs."""
    out = {"random": {}, "c2": {}, "c3": {}, "c4": {}}
    for seed in range(n):
        w = W.random_scenario(seed, max_nodes=5)
        entry = {"digest": digest(w)}
        for t in TOKENS:
            entry[t] = search(w, {"constraint": t}, "greedy")
        entry["floor2"] = search(w, {"constraint": w.objective["constraint"], "quality_floor": 2}, "greedy")
        out["random"][str(seed)] = entry
    w = W.config2()
    for t in TOKENS:
        out["c2"][t] = search(w, {"constraint": t}, "greedy")
    out["c2"]["config"] = search(w, w.objective, "greedy")
    w = W.config3(slo_us=None)
    for t in TOKENS:
        out["c3"][t] = search(w, {"constraint": t}, "greedy")
    for j, w in enumerate(W.config4(16)):
        out["c4"][str(j)] = search(w, w.objective, "greedy")
    dump(GOLD / "greedy" / "results.json", out)


def make_c3() -> None:
    w = W.config3()
    threads = os.cpu_count() or 8
    slices = [(0, 400_000), (123_456_789_012, 123_457_189_012), ((1 << 40) - 400_000, 1 << 40)]
    res = {"digest": digest(w), "objective": w.objective, "slices": []}
    for b, e in slices:
        rc, r = O.ref_range_argmin(w.dag, w.library, w.objective, w.bounds, b, e, threads)
        res["slices"].append({"begin": b, "end": e, "result": r})
    # a slice without the SLO: plain MIN_COST
    rc, r = O.ref_range_argmin(w.dag, w.library, {"constraint": "MIN_COST"}, w.bounds, 0, 400_000, threads)
    res["slice_no_slo"] = {"begin": 0, "end": 400_000, "result": r}
    dump(GOLD / "c3" / "slices.json", res)


def make_c4(n_jobs: int = 12) -> None:
    res = {"jobs": {}}
    for j, w in enumerate(W.config4(n_jobs)):
        res["jobs"][str(j)] = {"digest": digest(w), "result": search(w, w.objective)}
    dump(GOLD / "c4" / "jobs.json", res)


def make_c5() -> None:
    res = {}
    for n in (3, 4, 5):
        w = W.config5(n_nodes=n)
        t0 = time.time()
        rc, fr = O.ref_pareto(w.dag, w.library, w.bounds)
        res[str(n)] = {"digest": digest(w), "total": fr["total_count"],
                       "frontier": [r["plan_index"] for r in fr["frontier"]], "seconds": time.time() - t0}
    dump(GOLD / "c5" / "reduced_pareto.json", res)


if __name__ == "__main__":
    only = None
    for a in sys.argv[1:]:
        if a.startswith("--only"):
            only = set(a.split("=", 1)[1].split(","))
    for name, fn in [("c1", make_c1), ("c2", make_c2), ("random", make_random), ("c3", make_c3),
                     ("c4", make_c4), ("c5", make_c5), ("greedy", make_greedy)]:
        if only is None or name in only:
            t = time.time()
            fn()
            print(f"{name}: {time.time() - t:.1f}s", flush=True)
