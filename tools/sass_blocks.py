"""List the basic blocks of a search_kernel instantiation that hold many
compare instructions (the innermost sweeps), with per-class counts.
Usage: python tools/sass_blocks.py [K P NV PT] [min_setp]   (default 4 0 16 1 12)"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter
from pathlib import Path

K, P, NV, PT = (sys.argv[1:5] + ["4", "0", "16", "1"][len(sys.argv[1:5]):])[:4]
MIN = int(sys.argv[5]) if len(sys.argv) > 5 else 12
obj = os.environ.get("SASS_OBJ") or str(Path(__file__).resolve().parents[1] / "paper_2501_16634_b200" / "_build" /
                                         "loom_search.cu.o")
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=td, capture_output=True)
    cubin = next(Path(td).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-c", str(cubin)], capture_output=True, text=True).stdout
for sec in re.split(r"\n\s*\.section\s+\.text\.", sass)[1:]:
    if f"search_kernelILi{K}ELi{P}ELi{NV}ELb{PT}E" not in sec.split(",")[0]:
        continue
    blocks, cur = [], ["(entry)"]
    for l in sec.split("\n"):
        if l.strip().startswith(".L_x"):
            blocks.append(cur)
            cur = [l.strip().rstrip(":")]
        elif re.search(r"/\*[0-9a-f]{4,5}\*/", l):
            cur.append(re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", re.sub(r"^\s*/\*[0-9a-f]+\*/\s*", "", l)).strip())
    blocks.append(cur)
    for b in blocks:
        ops = [o.split()[1] if o.startswith("@") else o.split()[0] for o in b[1:] if o]
        c = Counter(o.split(".")[0] for o in ops)
        if c["DSETP"] + c["ISETP"] >= MIN:
            fp64 = sum(c[o] for o in ("DADD", "DSETP", "DMUL", "DFMA"))
            alu = sum(c[o] for o in ("ISETP", "PLOP3", "SEL", "FSEL", "LOP3", "IADD3", "VIADDMNMX", "VIADD", "SHF",
                                     "LEA", "VIMNMX", "FMNMX"))
            print(f"{b[0]:12s} issue {len(ops):4d}  alu {alu:3d}  fp64 {fp64:3d}  {c.most_common(9)}")
            if "-v" in sys.argv:
                print("\n".join("    " + x for x in b[1:]))
    break
