"""Driver for compute-sanitizer runs of the frontier search (tools/sanitize_fr.sh):
C1 under all four tokens, C2 MIN_LATENCY with a quality floor, C3 under the
binding SLO and MAX_QUALITY with an SLO, through the one-shot path and the
device-problem graph; each answer checked against the CPU oracle or the C3
golden."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

ctx = loom.Context(0)
n = 0
for w, objs in ((W.config1(), [{"constraint": t} for t in ("MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY")]),
                (W.config2(), [{"constraint": "MIN_LATENCY", "quality_floor": 3}])):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for o in objs:
        ref = O.argmin(p, o)
        got = loom.search_argmin(ctx, lw.problem, loom.objective(o))
        dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
        dp.search_async(0, None)
        g2 = dp.result()
        dp.close()
        assert got["plan_index"] == ref["index"] == g2["plan_index"], (w.name, o)
        n += 1
gold = json.loads((ROOT / "tests/golden/c3/full_space.json").read_text())
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
for o in ({"constraint": "MIN_COST", "latency_slo_us": 40000000},
          {"constraint": "MAX_QUALITY", "latency_slo_us": 60000000}):
    win = next(c for c in gold["cases"] if c["objective"] == o)["winner"]
    got = loom.search_argmin(ctx, lw.problem, loom.objective(o))
    dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
    dp.search_async(0, None)
    g2 = dp.result()
    dp.close()
    assert got["plan_index"] == win["index"] == g2["plan_index"], o
    n += 1
print("sanitize driver ok:", n, "searches x 2 paths")
