"""Host-thread scaling of the C4 batch lowering (loom_lower_batch) on this
machine: 10,000 6-task dag.json texts, 1 .. N threads."""
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
n = os.cpu_count() or 1
for th in sorted({1, 2, 4, 8, n}):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        b = loom.LoweredBatch(dags, lib_t, bounds_t, threads=th)
        t1 = time.perf_counter()
        b.close()
        ts.append(t1 - t0)
    print(f"threads {th:3d}: lower {1e3 * min(ts):7.2f} ms", flush=True)
