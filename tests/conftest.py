import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def loomlib():
    from paper_2501_16634_b200 import build, loom
    build.build()
    return loom.lib()


@pytest.fixture(scope="session")
def ctx(loomlib):
    from paper_2501_16634_b200 import loom
    c = loom.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def golden():
    def load(rel):
        return json.loads((GOLDEN / rel).read_text())
    return load


def cpu_threads() -> int:
    return max(1, min(16, os.cpu_count() or 1))
