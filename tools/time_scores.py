"""Timing of the per-plan estimate streams (loom_estimate_range_device /
loom_estimate_range / loom_estimate_plans): plans/s and achieved HBM GB/s of
the score streams, device-timed with CUDA events on the ctx stream.

    python tools/time_scores.py [--config c3] [--log2 28] [--reps 5] [--fields all|gpu_wh,latency_us]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--log2", type=int, default=28)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--fields", default="all")
ap.add_argument("--begin", type=int, default=123_456_789)
ap.add_argument("--host-log2", type=int, default=24)
a = ap.parse_args()

w = {"c2": W.config2, "c3": W.config3, "c5": W.config5}[a.config]()
lw = loom.Lowered(w.dag, w.library, w.bounds)
fields = list(loom.STREAM_FIELDS) if a.fields == "all" else a.fields.split(",")
dt = {"int64": torch.int64, "float64": torch.float64, "int32": torch.int32}
n = min(1 << a.log2, lw.total - a.begin)
bytes_per_plan = sum(torch.empty(0, dtype=dt[loom.STREAM_FIELDS[f]]).element_size() for f in fields)
stream = torch.cuda.Stream()
ctx = loom.Context(0, stream.cuda_stream)
dev = {f: torch.empty(n, dtype=dt[loom.STREAM_FIELDS[f]], device="cuda") for f in fields}
loom.estimate_range_device(ctx, lw.problem, a.begin, a.begin + n, dev)
torch.cuda.synchronize()
ms = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    loom.estimate_range_device(ctx, lw.problem, a.begin, a.begin + n, dev)
    e1.record(stream)
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
best = min(ms)
res = {"config": a.config, "plans": n, "fields": fields, "bytes_per_plan": bytes_per_plan,
       "device_ms_best": best, "device_ms_median": sorted(ms)[len(ms) // 2],
       "plans_per_s": n / (best / 1e3), "gbs": n * bytes_per_plan / (best / 1e3) / 1e9}
# host path into pinned buffers (e2e: kernel + D2H of every stream)
nh = min(1 << a.host_log2, n)
host = {f: torch.empty(nh, dtype=dt[loom.STREAM_FIELDS[f]], pin_memory=True) for f in fields}
loom.estimate_range_host(ctx, lw.problem, a.begin, a.begin + nh, host)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    loom.estimate_range_host(ctx, lw.problem, a.begin, a.begin + nh, host)
    ts.append(time.perf_counter() - t0)
res["host_plans"] = nh
res["host_ms_best"] = 1e3 * min(ts)
res["host_plans_per_s"] = nh / min(ts)
res["host_gbs"] = nh * bytes_per_plan / min(ts) / 1e9
# gather path
idx = torch.randint(0, lw.total, (1 << 22,), dtype=torch.int64).numpy().astype("uint64")
loom.estimate_plans(ctx, lw.problem, idx[:1024])
t0 = time.perf_counter()
loom.estimate_plans(ctx, lw.problem, idx)
res["gather_plans_per_s"] = len(idx) / (time.perf_counter() - t0)
print(json.dumps(res))
