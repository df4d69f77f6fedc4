"""Strong-scaling estimate on one GPU: time each rank's shard of a config's
plan space (dist.shard_range, the bench's split) as its own resident search
(loom_search_argmin_shard_async with the greedy seed as common incumbent, as
bench.py does under torchrun).
On N GPUs every rank runs its shard concurrently, so max(shard time) is the
N-GPU search time (plus the winner all-gather).
    python tools/time_shards.py [--config c3] [--ranks 2 4 8] [--reps 3]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import dist as D, loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-incumbent", action="store_true", help="plain range searches (no common greedy incumbent)")
ap.add_argument("--binding", action="store_true", help="C3 under the bench's binding 40 s SLO")
a = ap.parse_args()
w = W.config3(slo_us=W.C3_BINDING_SLO_US) if a.binding else {"c3": W.config3, "c5": W.config5, "c2": W.config2}[a.config]()
lw = loom.Lowered(w.dag, w.library, w.bounds)
obj = loom.objective(w.objective)
ctx = loom.Context(0)
dp = loom.DeviceProblem(ctx, lw.problem, obj)
base = None
for n in a.ranks:
    ts, wins = [], []
    for r in range(n):
        b, e = D.shard_range(lw.total, r, n)
        best = 1e9
        for _ in range(a.reps):
            t0 = time.perf_counter()
            if a.no_incumbent or n == 1:
                dp.search_async(b, e)
            else:
                dp.search_shard_async(b, e)
            try:
                wins.append(dp.result())
            except loom.NoFeasibleConfigError:
                pass
            best = min(best, time.perf_counter() - t0)
        ts.append(best)
    t = max(ts)
    base = base or t * n if n == 1 else base
    print(f"N={n}: max shard {1e3 * t:.2f} ms (min {1e3 * min(ts):.2f})  -> {lw.total / t:.3g} plans/s  "
          f"scaling vs N=1 {(base or t) / t:.2f}x  shards ms {[round(1e3 * x, 1) for x in ts]}", flush=True)
