"""Timing of the default (branch-and-bound) search on C3 objectives, with its
launch statistics.  LOOM_B200_LIB selects an experiment build."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

reps = int(os.environ.get("REPS", "5"))
ctx = loom.Context(0)
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
objs = [{"constraint": "MIN_COST", "latency_slo_us": s} for s in (46000000, 44000000, 42000000, 40000000, 38000000,
                                                                   36000000)] + [
    {"constraint": "MIN_LATENCY"}, {"constraint": "MIN_DOLLARS", "latency_slo_us": 40000000},
    {"constraint": "MAX_QUALITY"}, {"constraint": "MIN_COST"}]
tot = 0
for o in objs:
    dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        dp.search_async(0, None)
        r = dp.result()
        ts.append(time.perf_counter() - t0)
    st = loom.bnb_last_stats()
    tot += min(ts)
    print(json.dumps({"objective": o, "ms": round(1e3 * min(ts), 3), "index": r["plan_index"], **st}), flush=True)
    tr = loom.bfs_trace()
    print("   trace", round(tr["total_us"] or 0, 1), [(round(l["us"], 1), l["parents"], "R" if l["redundant"] else "D")
                                               for l in tr["levels"]], flush=True)
    dp.close()
print(os.environ.get("LOOM_B200_LIB", "default"), "total ms", round(1e3 * tot, 3))
