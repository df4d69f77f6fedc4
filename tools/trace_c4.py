import json, sys, time, os
sys.path.insert(0, '.')
from paper_2501_16634_b200 import loom, workloads as W
jobs = W.config4(10_000)
dags = [json.dumps(j.dag) for j in jobs]
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
obj_t = json.dumps(jobs[0].objective)
ctx = loom.Context(0)
loom.exhaustive_search_batch(dags[:64], lib_t, obj_t, bounds_t, ctx=ctx)
for _ in range(3):
    t0 = time.perf_counter()
    res = loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
    print('batch ms', 1e3*(time.perf_counter()-t0), file=sys.stderr)
batch = loom.LoweredBatch(dags, lib_t, bounds_t)
for _ in range(3):
    t0 = time.perf_counter()
    res2 = loom.search_lowered_batch(ctx, batch, loom.objective(jobs[0].objective))
    print('lowered search ms', 1e3*(time.perf_counter()-t0), file=sys.stderr)
print(os.cpu_count(), file=sys.stderr)
