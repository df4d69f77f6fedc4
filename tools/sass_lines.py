"""Attribute an ncu SASS-page capture to CUDA source lines.

    python tools/sass_lines.py OBJ.o KERNEL_SUBSTR CAPTURE_sass.csv[.gz] [TOP]

OBJ.o is the object the captured library was linked from (build.py keeps
them under paper_2501_16634_b200/_build[/variants/NAME]); its cubin is
disassembled with line info (nvdisasm -g) and instruction i of the kernel is
matched with row i of ncu's SASS page (both are in address order).  Prints
per source line: warp-stall samples (all, and the top reasons), instructions
executed and static SASS instruction count, sorted by samples."""
import collections
import csv
import gzip
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

obj, kname, cap = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, check=True,
                   capture_output=True)
    cub = next(Path(td).glob("*.cubin"))
    dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout

lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l)
loc = None
inst_loc = []
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m:
        loc = f"{Path(m.group(1)).name}:{m.group(2)}"
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        inst_loc.append(loc)

opener = gzip.open if cap.endswith(".gz") else open
with opener(cap, "rt") as f:
    rows = list(csv.reader(f))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
if len(data) != len(inst_loc):
    print(f"warning: {len(data)} captured rows vs {len(inst_loc)} disassembled instructions")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: {"samples": 0, "exec": 0, "n": 0, "st": collections.Counter()})
tot = 0
for r, lc in zip(data, inst_loc):
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    a = agg[lc]
    a["samples"] += s
    a["exec"] += int(r[ix["Instructions Executed"]] or 0)
    a["n"] += 1
    for c in stall_cols:
        v = int(r[ix[c]] or 0)
        if v:
            a["st"][c[6:]] += v
    tot += s
print(f"total samples {tot}, instructions {len(inst_loc)}")
for lc, a in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
    reasons = ", ".join(f"{k} {100 * v / max(1, a['samples']):.0f}%" for k, v in a["st"].most_common(3))
    print(f"{lc:28s} {100 * a['samples'] / max(1, tot):5.1f}%  exec {a['exec']:>10d}  sass {a['n']:>5d}  {reasons}")
