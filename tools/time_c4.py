"""Phase timing of the C4 multi-tenant batch (10,000 jobs x 6 tasks x 8
options): lowering, marshalling, the batched search call (run with
LOOM_TRACE=1 for its host/device split) and result decoding."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
jobs = W.config4(n)
dags = [json.dumps(j.dag) for j in jobs]
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
objs = [loom.objective(j.objective) for j in jobs]
ctx = loom.Context(0)
lws = loom.lower_batch(dags[:64], lib_t, bounds_t)
loom.search_argmin_batch(ctx, [lw.problem for lw in lws], objs[:64])
for rep in range(3):
    t0 = time.perf_counter()
    lws = loom.lower_batch(dags, lib_t, bounds_t)
    t1 = time.perf_counter()
    probs = [lw.problem for lw in lws]
    t2 = time.perf_counter()
    res = loom.search_argmin_batch(ctx, probs, objs)
    t3 = time.perf_counter()
    print(f"rep {rep}: lower {1e3 * (t1 - t0):.1f} ms  problems {1e3 * (t2 - t1):.1f} ms  "
          f"search+decode {1e3 * (t3 - t2):.1f} ms  total {1e3 * (t3 - t0):.1f} ms  "
          f"feasible {sum(1 for s, _ in res if s == 0)}", flush=True)
