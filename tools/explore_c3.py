"""Exploration: time the resident C3 search under several objectives
(binding latency SLOs, MIN_LATENCY, MIN_DOLLARS) and report the winner and the
greedy seed.  python tools/explore_c3.py [--reps 3] [--objectives JSON...]"""
import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--plans", type=float, default=0)
ap.add_argument("objectives", nargs="*")
a = ap.parse_args()
objs = [json.loads(o) for o in a.objectives] or [
    {"constraint": "MIN_COST", "latency_slo_us": s} for s in (46_000_000, 44_000_000, 42_000_000, 40_000_000,
                                                               38_000_000, 36_000_000)] + [
    {"constraint": "MIN_LATENCY"}, {"constraint": "MIN_DOLLARS", "latency_slo_us": 40_000_000}]
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
ctx = loom.Context(0)
stats = bool(os.environ.get("LOOM_STATS_READ"))
for o in objs:
    obj = loom.objective(o)
    seed = (C.c_int32 * 10)()
    rc = loom.lib().loom_greedy_seed(C.byref(lw.problem), C.byref(obj), seed)
    sidx = 0
    for d in seed:
        sidx = sidx * 16 + d
    dp = loom.DeviceProblem(ctx, lw.problem, obj)
    end = lw.total if not a.plans else int(a.plans)
    if stats:
        buf = (C.c_uint64 * 8)()
        loom.lib().loom_debug_counters(buf, 1)
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        dp.search_async(0, end)
        try:
            r = dp.result()
        except loom.NoFeasibleConfigError:
            r = {"plan_index": None}
        ts.append(time.perf_counter() - t0)
    line = {"objective": o, "best_ms": 1e3 * min(ts), "plans_per_s": end / min(ts), "winner": r,
            "seed": sidx, "seed_is_winner": sidx == r.get("plan_index")}
    if stats:
        loom.lib().loom_debug_counters(buf, 1)
        line["stats_per_run"] = [buf[i] / a.reps for i in range(8)]
    print(json.dumps(line), flush=True)
    dp.close()
