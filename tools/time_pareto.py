"""Phase timing of the C5 Pareto frontier (9 tasks x 10 options = 1e9
plans).  Run with LOOM_DEBUG=1 for the eval / refine split."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = W.config5()
lw = loom.Lowered(w.dag, w.library, w.bounds)
ctx = loom.Context(0)
loom.search_pareto_points(ctx, lw.problem, 0, lw.total - 1)
for r in range(reps):
    t0 = time.perf_counter()
    f = loom.search_pareto_points(ctx, lw.problem, 0, lw.total - r)  # distinct ranges defeat the ctx cache
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.1f} ms, {len(f)} frontier points", flush=True)
