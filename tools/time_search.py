"""Quick A/B timing of one config's resident search (no bench contract, no
L2 flush): python tools/time_search.py [--config c3] [--reps 5].  Set
LOOM_B200_LIB to time an experiment build (build.py --variant)."""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--objective", default=None)
a = ap.parse_args()
w = {"c1": W.config1, "c2": W.config2, "c3": W.config3, "c5": W.config5}[a.config]()
lw = loom.Lowered(w.dag, w.library, w.bounds)
obj = loom.objective(a.objective or w.objective)
ctx = loom.Context(0)
dp = loom.DeviceProblem(ctx, lw.problem, obj)
dp.search_async(0, lw.total)
r = dp.result()
ts = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    dp.search_async(0, lw.total)
    r = dp.result()
    ts.append(time.perf_counter() - t0)
best = min(ts)
print(f"{os.environ.get('LOOM_B200_LIB', 'default')}: {a.config} best {1e3 * best:.2f} ms "
      f"median {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms  {lw.total / best:.4g} plans/s  index {r['plan_index']}")
