"""Host-side phase trace (LOOM_TRACE) of the C4 multi-tenant call: 10,000
6-task jobs through loom_exhaustive_search_batch, a few times."""
import json
import os
import sys
import time
from pathlib import Path

os.environ["LOOM_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

jobs = W.config4(10_000)
dags = [json.dumps(j.dag).encode() for j in jobs]  # bytes, as the bench passes them
lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
ctx = loom.Context(0)
for token in sys.argv[1:] or ["MIN_LATENCY"]:
    obj_t = json.dumps({"constraint": token})
    for i in range(3):
        t0 = time.perf_counter()
        res = loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
        print(f"--- {token} call {i}: {1e3 * (time.perf_counter() - t0):.3f} ms (python wall)", file=sys.stderr,
              flush=True)
