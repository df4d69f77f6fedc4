"""Profiling driver: one search over a slice of a config's plan space on
cuda:0 (short enough for `ncu --set full` replays)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--plans", type=float, default=2 ** 36)
ap.add_argument("--begin", type=int, default=0)
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--objective", default=None)
a = ap.parse_args()
w = {"c1": W.config1, "c2": W.config2, "c3": W.config3, "c5": W.config5}[a.config]()
lw = loom.Lowered(w.dag, w.library, w.bounds)
obj = loom.objective(a.objective or w.objective)
ctx = loom.Context(0)
for _ in range(a.repeat):
    try:
        r = loom.search_argmin(ctx, lw.problem, obj, a.begin, a.begin + int(a.plans))
        print(r["plan_index"], r["latency_us"], r["gpu_wh"])
    except loom.NoFeasibleConfigError as e:
        print("infeasible", e)
