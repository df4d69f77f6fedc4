"""Summarise the ncu outputs of tools/profile_round.sh into profiles/:
profiles/<round>/launches.csv (copied), profiles/<round>/search_kernel_full.txt
(key metrics of the full-set capture), profiles/ncu_summary.json (numbers
bench.py quotes: DRAM bytes per C3 launch, instructions per plan, issue %)."""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
out = ROOT / "profiles" / rnd
out.mkdir(parents=True, exist_ok=True)
src = ROOT / "gpurun_out"

# launch list
rows = []
if (src / "launches.csv").exists():
    shutil.copy(src / "launches.csv", out / "launches.csv")
    lines = (src / "launches.csv").read_text().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
launch = {}
for r in rows:
    launch.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = r["Metric Value"]
PLANS_C3 = 1_099_511_627_776
c3 = [(k, m) for k, m in launch.items() if "search_kernel" in k[1]]
# the C3 launches are the long ones
c3_long = [m for k, m in c3 if float(m.get("gpu__time_duration.sum", 0)) > 5e7]
summary = {"round": rnd}
if c3_long:
    m = c3_long[-1]
    f = lambda k: float(m[k].replace(",", ""))
    summary.update({
        "c3_launch_ns": f("gpu__time_duration.sum"),
        "dram_bytes_per_launch": f("dram__bytes_read.sum") + f("dram__bytes_write.sum"),
        "thread_inst_per_plan": f("smsp__inst_executed.sum") * 32 / PLANS_C3,
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "sm_clock_hz": f("sm__cycles_elapsed.avg.per_second"),
        "c3_plans_per_s_under_ncu": PLANS_C3 / (f("gpu__time_duration.sum") * 1e-9),
    })
total_ns = sum(float(m.get("gpu__time_duration.sum", 0)) for m in launch.values())
kern_ns = {}
for (i, name), m in launch.items():
    short = name.split("(")[0].replace("void ", "")
    kern_ns[short] = kern_ns.get(short, 0.0) + float(m.get("gpu__time_duration.sum", 0))
summary["launch_time_share"] = {k: round(v / total_ns, 4) for k, v in sorted(kern_ns.items(), key=lambda x: -x[1])}
summary["launches"] = len(launch)

# full captures
KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Achieved Active Warps Per SM", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Branch Efficiency",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "L1/TEX Hit Rate", "L2 Hit Rate"]


def full_summary(rep: Path, name: str) -> dict:
    det = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"], capture_output=True, text=True).stdout
    lines = []
    for r in csv.DictReader(det.splitlines()):
        if r.get("Metric Name") in KEEP:
            lines.append(f'{r["Section Name"][:34]:34s} {r["Metric Name"][:40]:40s} {r["Metric Value"]:>16s} {r["Metric Unit"]}')
    src_csv = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
    try:
        hdr_i = next(i for i, l in enumerate(src_csv) if l.startswith('"Address"'))
        srows = list(csv.DictReader(src_csv[hdr_i:]))
        stall = {}
        for r in srows:
            for k, v in r.items():
                if k and k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
                    stall[k] = stall.get(k, 0.0) + float(v)
        tot = sum(stall.values()) or 1.0
        lines.append("")
        lines.append("warp stall samples (share of all samples):")
        for k, v in sorted(stall.items(), key=lambda x: -x[1])[:10]:
            lines.append(f"  {k:32s} {100 * v / tot:5.1f}%")
    except StopIteration:
        pass
    (out / name).write_text("\n".join(lines) + "\n")
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    vals = {}
    if len(rr) >= 3:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "": 1}
        for k, u, v in zip(rr[0], rr[1], rr[2]):
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum"):
                vals[k] = float(v.replace(",", "")) * scale.get(u, 1)
    return vals


if (src / "prof_full.ncu-rep").exists():
    full_summary(src / "prof_full.ncu-rep", "search_kernel_full.txt")
if (src / "prof_scores.ncu-rep").exists():
    # tools/time_scores.py --log2 26: 2^26 C3 plans, six streams, 44 B per plan
    v = full_summary(src / "prof_scores.ncu-rep", "score_kernel_full.txt")
    plans = 1 << 26
    if v:
        summary["score_stream"] = {
            "plans_per_launch": plans, "algorithmic_bytes_per_launch": plans * 44,
            "dram_bytes_per_launch": v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0),
            "launch_ns_cold": v.get("gpu__time_duration.sum"),
            "thread_inst_per_plan": v.get("smsp__inst_executed.sum", 0) * 32 / plans}
if (src / "bench.json").exists():
    shutil.copy(src / "bench.json", out / "bench.json")
(ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary, indent=1))
