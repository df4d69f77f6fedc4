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
ap.add_argument("--begin", type=int, default=0)
ap.add_argument("--plans", type=float, default=0, help="plans to search from --begin (0: the whole space)")
a = ap.parse_args()
w = {"c1": W.config1, "c2": W.config2, "c3": W.config3, "c5": W.config5}[a.config]()
lw = loom.Lowered(w.dag, w.library, w.bounds)
obj = loom.objective(a.objective or w.objective)
ctx = loom.Context(0)
dp = loom.DeviceProblem(ctx, lw.problem, obj)
end = lw.total if not a.plans else min(lw.total, a.begin + int(a.plans))
dp.search_async(a.begin, end)
r = dp.result()
ts = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    dp.search_async(a.begin, end)
    r = dp.result()
    ts.append(time.perf_counter() - t0)
best = min(ts)
print(f"{os.environ.get('LOOM_B200_LIB', 'default')}: {a.config} best {1e3 * best:.2f} ms "
      f"median {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms  {(end - a.begin) / best:.4g} plans/s  index {r['plan_index']}")

if os.environ.get("LOOM_STATS_READ"):
    import ctypes as C
    buf = (C.c_uint64 * 8)()
    loom.lib().loom_debug_counters(buf, 1)
    runs = 1 + a.reps
    print("  stats per run: flagged steps %.4g  bound-pass ctx %.4g  exact-pass ctx %.4g  steps %.4g" %
          tuple(buf[i] / runs for i in (0, 1, 2, 3)))
