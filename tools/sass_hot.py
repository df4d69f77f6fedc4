"""Print the hot innermost-context loop of a search_kernel instantiation from
the built object (the block holding >= 16 DSETP within 120 instructions) and
count its instructions by class.  Usage: python tools/sass_hot.py 4 0 16"""
import re
import subprocess
import sys
import tempfile
from pathlib import Path

K, P, NV = sys.argv[1:4]
PT = sys.argv[4] if len(sys.argv) > 4 else "1"
import os
obj = Path(os.path.abspath(os.environ.get("SASS_OBJ")) if os.environ.get("SASS_OBJ") else Path(__file__).resolve().parents[1] / "paper_2501_16634_b200" / "_build" / "loom_search.cu.o")
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(obj)], cwd=td, capture_output=True)
    cubin = next(Path(td).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-c", str(cubin)], capture_output=True, text=True).stdout
for sec in re.split(r"\n\s*\.section\s+\.text\.", sass)[1:]:
    name = sec.split(",")[0]
    if f"search_kernelILi{K}ELi{P}ELi{NV}ELb{PT}E" not in name or "slow" in name:
        continue
    lines = [l for l in sec.split("\n") if re.search(r"/\*[0-9a-f]{4,5}\*/", l) or l.strip().startswith(".L_x")]
    idx = [i for i, l in enumerate(lines) if "DSETP" in l or ("ISETP.LE.AND" in l)]
    start = None
    for k in range(len(idx) - 15):
        if idx[k + 15] - idx[k] < 120:
            start = idx[k]
            break
    if start is None:
        print("no hot block found")
        break
    # extend to the enclosing label .. backward branch
    a = start
    while a > 0 and not lines[a].strip().startswith(".L_x"):
        a -= 1
    b = start
    while b < len(lines) and "BRA" not in lines[b] or (b < start + 40):
        b += 1
    body = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in lines[a:b + 1]]
    for l in body:
        print(l)
    ops = [l.split()[1] if l.startswith("@") else (l.split()[1] if l.startswith("/*") else l.split()[0])
           for l in body if not l.startswith(".L_x")]
    from collections import Counter
    cnt = Counter(o.split(".")[0] for o in ops)
    print(len(ops), cnt.most_common())
    # pipes at 16 lanes/clk/SMSP (2 issue cycles per warp instruction)
    fp64 = sum(cnt[o] for o in ("DADD", "DSETP", "DMUL", "DFMA", "DMNMX"))
    alu = sum(cnt[o] for o in ("ISETP", "PLOP3", "SEL", "LOP3", "IADD3", "VIADDMNMX", "VIADD", "SHF", "LEA", "IMNMX"))
    print(f"issue {len(ops)}  alu {alu} ({2 * alu} cycles)  fp64 {fp64} ({2 * fp64} cycles)")
    break
