"""Profiling driver: the default (branch-and-bound) search of the bench's
headline instance (C3, MIN_COST under the binding SLO) on cuda:0, a few
times, for `ncu -k bnb_kernel`."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--objective", default=None)
a = ap.parse_args()
w = W.config3(slo_us=W.C3_BINDING_SLO_US)
lw = loom.Lowered(w.dag, w.library, w.bounds)
obj = loom.objective(json.loads(a.objective) if a.objective else w.objective)
ctx = loom.Context(0)
dp = loom.DeviceProblem(ctx, lw.problem, obj)
for _ in range(a.repeat):
    dp.search_async(0, None)
    r = dp.result()
    print(r["plan_index"], r["latency_us"], r["gpu_wh"], loom.bnb_last_stats())
