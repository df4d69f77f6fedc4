"""C4 time-to-plan, 15 calls per objective (min / median)."""
import json, sys, time, os
sys.path.insert(0, os.getcwd())
from paper_2501_16634_b200 import loom, workloads as W
jobs = W.config4(10_000)
dags = [json.dumps(j.dag).encode() for j in jobs]
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
ctx = loom.Context(0)
for token in ("MIN_LATENCY", "MIN_COST"):
    obj_t = json.dumps({"constraint": token})
    loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx); ts.append(1e3*(time.perf_counter()-t0))
    ts.sort(); print(token, "min %.2f median %.2f" % (ts[0], ts[7]))
