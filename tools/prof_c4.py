"""Profiling driver for the C4 batch kernel: one batched search of the
10,000 lowered jobs (python tools/prof_c4.py [n_jobs])."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
jobs = W.config4(n)
dags = [json.dumps(j.dag) for j in jobs]
batch = loom.LoweredBatch(dags, json.dumps(jobs[0].library), json.dumps(jobs[0].bounds))
ctx = loom.Context(0)
res = loom.search_lowered_batch(ctx, batch, loom.objective(jobs[0].objective))
print("feasible", res.feasible())
