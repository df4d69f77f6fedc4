"""Summarise an ncu capture exported as raw + SASS-source CSVs: headline
metrics, warp-stall reasons, and the hottest SASS instructions by stall
samples.  python tools/ncu_hot.py PREFIX  (reads PREFIX_raw.csv, PREFIX_sass.csv)"""
import csv
import sys

pre = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(pre + "_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
for w in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
          "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]:>16s} {units[i]}")
st = [(hdr[i], float(vals[i] or 0)) for i in range(len(hdr))
      if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled") and not hdr[i].endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                           for h, v in sorted(st, key=lambda x: -x[1])[:10]))
rows = list(csv.reader(open(pre + "_sass.csv")))
h2 = rows[1]
ai, si, wi, ei = (h2.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                         "Instructions Executed"))
data = [(r[si].strip(), int(r[wi] or 0), int(r[ei] or 0)) for r in rows[2:] if len(r) > ei]
tot = sum(d[1] for d in data) or 1
print("instructions:", len(data), "samples:", tot)
for i in sorted(sorted(range(len(data)), key=lambda i: -data[i][1])[:top_n]):
    print(f"{i:6d} {data[i][0][:70]:70s} {100 * data[i][1] / tot:5.1f}% {data[i][2]}")
