"""loom-b200: B200-native exhaustive plan evaluation for the Murakkab / loom
scheduler (arXiv 2501.16634).  See DESIGN.md.

The compute lives in libloom_b200.so (C ABI: include/loom_b200.h, C++ drop-in:
include/loom_b200/loom.hpp); this package is the Python binding and the
synthetic workload generators used by tests and bench.py.
"""
from . import loom, workloads  # noqa: F401

__all__ = ["loom", "workloads"]
