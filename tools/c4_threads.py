"""C4 time-to-plan against the host thread count of the batch call
(loom_exhaustive_search_batch's `threads`; 0 = the library's default)."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

jobs = W.config4(10_000)
dags = [json.dumps(j.dag).encode() for j in jobs]
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
ctx = loom.Context(0)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for token in ("MIN_LATENCY", "MIN_COST"):
    obj_t = json.dumps({"constraint": token})
    loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
    for th in (0, 8, 12, 16, 20, 24, 32, 48):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx, threads=th)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{token} threads {th}: min {min(ts):.2f} ms  median {sorted(ts)[2]:.2f} ms", flush=True)
t0 = time.perf_counter()
for _ in range(20):
    arr, keep = loom._text_array(dags)
print(f"text array {1e3 * (time.perf_counter() - t0) / 20:.3f} ms")
