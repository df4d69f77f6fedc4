"""Phase marks of the frontier kernel (experiment build with -DLOOM_FR_PROF=1):
cycles per phase per level for one C3 objective.
    LOOM_B200_LIB=.../libloom_b200.so python tools/fr_prof.py '{"constraint": "MIN_LATENCY"}'"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_16634_b200 import loom, workloads as W  # noqa: E402

o = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {"constraint": "MIN_COST", "latency_slo_us": 40000000}
w = W.config3(slo_us=None)
lw = loom.Lowered(w.dag, w.library, w.bounds)
ctx = loom.Context(0)
dp = loom.DeviceProblem(ctx, lw.problem, loom.objective(o))
for _ in range(3):
    dp.search_async(0, None)
    dp.result()
buf = (C.c_uint64 * (8 * 33))()
assert loom.lib().loom_debug_fr_prof(buf, 8 * 33) == 0
names = ["startA", "A->warpbest", "->phaseB end", "->batches", "->blockbest", "->sync/barrier", "->end"]
print(o)
for d in range(lw.problem.n_nodes):
    m = [buf[8 * d + i] for i in range(8)]
    if m[7] and m[1] > m[7] > m[0]:  # LOOM_FR_PROF=2: mark 7 = end of the first (cold) expansion
        print(d, "expand cold", m[7] - m[0], "warm", m[1] - m[7])
    if not m[0]:
        continue
    segs = []
    prev = m[0]
    for i in range(1, 8):
        if m[i] and m[i] >= prev:
            segs.append(f"{names[i - 1]} {m[i] - prev}")
            prev = m[i]
    nxt = buf[8 * (d + 1)] if d + 1 < 33 else 0
    print(d, " | ".join(segs), "| to next level", (nxt - prev) if nxt > prev else "")

b2 = (C.c_uint64 * 16)()
lib_ok = loom.lib().loom_debug_fr_prof2(b2) == 0
if lib_ok and b2[14] and b2[12]:
    m = list(b2)
    d = lambda a, b: (m[b] - m[a]) if m[a] and m[b] and m[b] >= m[a] else None  # noqa: E731
    print("LOOM_FR_PROF=4 (cycles): blob load", d(14, 15), "| prologue", d(15, 12), "| heuristic", d(12, 13),
          "| H1 choose", d(0, 1), "| H1 eval", d(1, 2), "| reduce0", d(2, 3), "| H2 eval1", d(3, 4),
          "| reduce1", d(4, 5), "| H2 eval2", d(5, 6), "| reduce2", d(6, 7))
