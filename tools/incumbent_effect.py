"""How much a better starting incumbent shrinks the frontier search: each C3
golden objective searched from its default incumbent, then from the golden
optimum itself (an oracle incumbent -- an upper bound on what any incumbent
heuristic could buy)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

gold = json.loads((Path(__file__).resolve().parents[1] / "tests/golden/c3/full_space.json").read_text())
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
ctx = loom.Context(0)
for case in gold["cases"]:
    if case["winner"] is None:
        continue
    dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(case["objective"]))
    row = [case["objective"]]
    for inc in (None, case["winner"]["index"]):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            if inc is None:
                dp.search_async(0, None)
            else:
                dp.search_algo_async(0, None, loom.ALGO_AUTO, inc)
            r = dp.result()
            ts.append(time.perf_counter() - t0)
        st = loom.bnb_last_stats()
        assert r["plan_index"] == case["winner"]["index"]
        row.append((round(1e3 * min(ts), 3), st["child_evaluations"], st["max_frontier"]))
    print(row, flush=True)
    dp.close()
