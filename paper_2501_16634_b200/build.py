"""Build recipe for libloom_b200.so (sm_100a).  Built in-tree so the .so
travels with the gpurun snapshot; no JIT cache is involved.

    python -m paper_2501_16634_b200.build [--force]
    python -m paper_2501_16634_b200.build --variant NAME -DMACRO=V ...
        (experiment builds: _build/variants/NAME/libloom_b200.so, loaded by
        loom.py when LOOM_B200_LIB points at it)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libloom_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
# -fmad=false / -ffp-contract=off: no FMA contraction anywhere, so every
# product and sum rounds like the reference's default x86-64 build.
CU_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xptxas", "-v",
            "-Xcompiler", "-fPIC,-ffp-contract=off", *ARCH, *INCLUDES]
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
             "-Wno-unused-parameter", *INCLUDES, "-I", "/usr/local/cuda/include"]

CU_SOURCES = ["loom_search.cu", "loom_scores.cu"]
CXX_SOURCES = ["loom_capi.cpp", "loom_host.cpp", "json.cpp", "loom_group.cpp"]


def _run(cmd: list[str], log: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd))
    log.append(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write("\n".join(log[-2:]))
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def _stale(out: Path, deps: list[Path]) -> bool:
    return not out.exists() or any(d.stat().st_mtime > out.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: list[str] | None = None) -> Path:
    OBJ.mkdir(exist_ok=True)
    defines = defines or []
    cu_obj = OBJ if variant is None else OBJ / "variants" / variant
    lib = LIB if variant is None else cu_obj / "libloom_b200.so"
    cu_obj.mkdir(parents=True, exist_ok=True)
    headers = (list(CSRC.glob("*.h")) + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh"))
               + list((ROOT / "include").rglob("*.h*")))
    log: list[str] = []
    objs = []
    for src in CU_SOURCES:
        o = cu_obj / (src + ".o")
        if force or variant is not None or _stale(o, [CSRC / src, *headers]):
            _run([NVCC, *CU_FLAGS, *defines, "-c", str(CSRC / src), "-o", str(o)], log)
        objs.append(o)
    for src in CXX_SOURCES:
        o = OBJ / (src + ".o")
        if force or _stale(o, [CSRC / src, *headers]):
            _run(["g++", *CXX_FLAGS, "-c", str(CSRC / src), "-o", str(o)], log)
        objs.append(o)
    if force or _stale(lib, objs):
        _run([NVCC, "-shared", *ARCH, "-o", str(lib), *map(str, objs), "-lpthread", "-ldl"], log)
    if verbose:
        print("\n".join(log))
    (cu_obj / "build.log").write_text("\n".join(log))
    return lib


if __name__ == "__main__":
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else None
    build(force="--force" in argv, verbose=var is None, variant=var,
          defines=[a for a in argv if a.startswith("-D")])
