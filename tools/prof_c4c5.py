"""Profiling driver for the secondary rooflines: the C4 multi-tenant batch
search (10,000 jobs, one launch of the depth-first kernel, one CTA per job)
and the C5 Pareto frontier (1e9 plans: guard, pareto_eval_kernel, refine,
pareto_filter_kernel), once each after a warm-up, for
    ncu --set full -k regex:"bnb_kernel|pareto_eval_kernel|pareto_filter_kernel" ..."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ctx = loom.Context(0)
jobs = W.config4(10_000)
dags = [json.dumps(j.dag) for j in jobs]
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
obj_t = json.dumps({"constraint": "MIN_LATENCY"})
for _ in range(2):
    res = loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
print("c4 feasible", res.feasible(), flush=True)
w5 = W.config5()
lw5 = loom.Lowered(w5.dag, w5.library, w5.bounds)
for k in range(2):
    front = loom.search_pareto_points(ctx, lw5.problem, 0, lw5.total - k)
print("c5 frontier", len(front), flush=True)
