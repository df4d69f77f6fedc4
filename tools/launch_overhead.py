"""Device time of one default search (CUDA events around the search graph)
against the frontier kernel's own %globaltimer span, for C1 (4 tasks: the
kernel does almost nothing) and C3 under the binding SLO: the difference is
the launch / teardown cost of the graph."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

stream = torch.cuda.Stream()
ctx = loom.Context(0, stream.cuda_stream)
for name, w in (("c1", W.config1()), ("c3", W.config3(slo_us=W.C3_BINDING_SLO_US))):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(w.objective))
    ev, tr = [], []
    for i in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dp.search_async(0, None)
        e1.record(stream)
        dp.result()
        e1.synchronize()
        if i >= 5:
            ev.append(1e3 * e0.elapsed_time(e1))
            tr.append(loom.bfs_trace()["total_us"])
    print(name, "event us", round(statistics.median(ev), 1), "kernel trace us", round(statistics.median(tr), 1))
