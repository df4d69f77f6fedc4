"""Host-side phase trace (LOOM_TRACE) of the bench's e2e call: the JSON drop-in
search of C3 under the binding SLO, a few times."""
import os
import sys
import time
from pathlib import Path

os.environ["LOOM_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

w = W.config3(slo_us=W.C3_BINDING_SLO_US)
texts = w.texts()
ctx = loom.Context(0)
for i in range(4):
    t0 = time.perf_counter()
    loom.exhaustive_search(*texts, ctx=ctx)
    print(f"--- call {i}: {1e3 * (time.perf_counter() - t0):.3f} ms (python wall)", file=sys.stderr, flush=True)
