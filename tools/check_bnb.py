"""GPU check + timing of the branch-and-bound search against the sweep and
the CPU oracle.  python tools/check_bnb.py"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ctx = loom.Context(0)
bad = 0


def run(dp, algo, reps=1, begin=0, end=None):
    ts = []
    r = None
    for _ in range(reps):
        t0 = time.perf_counter()
        dp.search_algo_async(begin, end, algo)
        try:
            r = dp.result()
        except loom.NoFeasibleConfigError:
            r = None
        ts.append(time.perf_counter() - t0)
    return r, min(ts)


# random scenarios: auto vs oracle
for seed in range(80):
    w = W.random_scenario(seed)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for extra in ({}, {"quality_floor": 2}, {"latency_slo_us": 30_000_000}):
        o = dict(w.objective, **extra)
        dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
        r, _ = run(dp, loom.ALGO_AUTO)
        ref = O.argmin(p, o)
        if (r is None) != (ref is None) or (r and r["plan_index"] != ref["index"]):
            bad += 1
            print("MISMATCH random", seed, o, r, ref)
        dp.close()
print("random done, bad", bad, flush=True)

cases = [("c1", W.config1(), [{"constraint": t} for t in ("MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY")]),
         ("c2", W.config2(), [W.config2().objective, {"constraint": "MIN_COST"}]),
         ("c3", W.config3(slo_us=None),
          [{"constraint": "MIN_COST", "latency_slo_us": s} for s in (72043534, 46000000, 40000000, 36000000)]
          + [{"constraint": "MIN_LATENCY"}, {"constraint": "MIN_DOLLARS", "latency_slo_us": 40000000},
             {"constraint": "MAX_QUALITY"}, {"constraint": "MIN_COST"}])]
for name, w, objs in cases:
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for o in objs:
        dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
        ra, ta = run(dp, loom.ALGO_AUTO, reps=5)
        st = loom.bnb_last_stats()
        rs, ts = run(dp, loom.ALGO_SWEEP, reps=2)
        ref, _ = O.argmin_bnb(p, o)
        ok = (ra and ref and ra["plan_index"] == ref["index"] and rs["plan_index"] == ref["index"]) or (
            ra is None and ref is None and rs is None)
        if not ok:
            bad += 1
        print(json.dumps({"case": name, "objective": o, "ok": bool(ok), "bnb_ms": 1e3 * ta, "sweep_ms": 1e3 * ts,
                          "bnb": st, "index": ra and ra["plan_index"]}), flush=True)
        dp.close()
print("ALL BAD", bad)
