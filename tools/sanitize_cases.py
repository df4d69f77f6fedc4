"""Small invocations of every kernel family for compute-sanitizer
(tools/sanitize.sh): hierarchical argmin (K = 2..4, energy / latency /
quality primaries, register and shared-memory innermost tables), the
one-plan-per-thread path, the batch kernel, Pareto, greedy, shard searches
and the estimate-stream kernels."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ctx = loom.Context(0)
for w in (W.config1(), W.config2(), W.config3()):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    end = min(lw.total, 1 << 22)
    for tok in ("MIN_COST", "MIN_LATENCY", "MAX_QUALITY", "MIN_DOLLARS"):
        for algo in (0, 1):
            try:
                loom.search_argmin(ctx, lw.problem, loom.objective(tok), 0, end, algo)
            except loom.NoFeasibleConfigError:
                pass
for seed in range(6):
    w = W.random_scenario(seed, max_nodes=6)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    try:
        loom.search_argmin(ctx, lw.problem, loom.objective("MIN_COST"))
    except loom.NoFeasibleConfigError:
        pass
jobs = W.config4(16)
lws = [loom.Lowered(j.dag, j.library, j.bounds) for j in jobs]
loom.search_argmin_batch(ctx, [lw.problem for lw in lws], [loom.objective(j.objective) for j in jobs])
w5 = W.config5(n_nodes=6)
lw5 = loom.Lowered(w5.dag, w5.library, w5.bounds)
f = loom.search_pareto_points(ctx, lw5.problem)
loom.pareto_filter_points(ctx, f)
w3 = W.config3(slo_us=None)
loom.greedy_search(w3.dag, w3.library, {"constraint": "MIN_COST"}, w3.bounds, ctx=ctx)
# shard searches with a common incumbent, and a range search that seeds itself
w3s = W.config3()
lw3 = loom.Lowered(w3s.dag, w3s.library, w3s.bounds)
o3 = loom.objective(w3s.objective)
for b in (0, 1 << 22, 5 << 30):
    try:
        loom.search_argmin_shard(ctx, lw3.problem, o3, b, b + (1 << 22))
        loom.search_argmin(ctx, lw3.problem, o3, b, b + (1 << 22))
    except loom.NoFeasibleConfigError:
        pass
# estimate streams: range (aligned and ragged) and gather
import numpy as np  # noqa: E402
loom.estimate_range(ctx, lw3.problem, 12345, 12345 + 70_000)
loom.estimate_plans(ctx, lw3.problem, np.arange(0, 1 << 20, 997, dtype=np.uint64))
lw1 = loom.Lowered(W.config1().dag, W.config1().library, W.config1().bounds)
loom.estimate_range(ctx, lw1.problem, 0, lw1.total)
print("sanitize cases done", len(f))
