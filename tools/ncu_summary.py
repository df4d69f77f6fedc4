"""Fold one ncu --set full capture of the frontier kernel (tools/ncu_fr.sh ->
gpurun_out/fr_<S>_raw.csv) into profiles/ncu_summary.json["bfs_kernel"]:
the per-launch numbers bench.py's roofline reads (warp instructions, DRAM
bytes) plus the issue/occupancy context.

    python tools/ncu_summary.py gpurun_out/fr_<S>_raw.csv [workload note]"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
raw = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else "C3, MIN_COST under the binding 40 s SLO (tools/prof_bnb.py)"
rows = list(csv.reader(open(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def get(name):
    i = hdr.index(name)
    v = vals[i].replace(",", "")
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e3, "ms": 1e6, "ns": 1, "s": 1e9}.get(units[i], 1)
    return float(v) * scale


out = {
    "workload": note,
    "capture": str(Path(raw).name),
    "duration_ns_under_ncu": get("gpu__time_duration.sum"),
    "warp_inst_per_launch": get("smsp__inst_executed.sum"),
    "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "threads_per_warp_inst": get("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "registers_per_thread": get("launch__registers_per_thread"),
}
p = ROOT / "profiles" / "ncu_summary.json"
cur = json.loads(p.read_text()) if p.exists() else {}
if "bfs_kernel" not in cur and "c3_launch_ns" in cur:  # keep round 1's sweep numbers under their own key
    cur = {"round1_search_kernel": cur}
cur["round"] = "round2"
cur["bfs_kernel"] = out
p.write_text(json.dumps(cur, indent=1) + "\n")
print(json.dumps(out, indent=1))
