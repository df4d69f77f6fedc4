"""The reference-side binding (integration/loom_b200_adapter.hpp) compiled
against the UNMODIFIED reference headers (oracle/_ref/adapter_check): the
reference's own exhaustive_search and the drop-in GPU search must select the
same ConfigPoint with bit-identical metrics, and raise the same error."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_2501_16634_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "adapter_check"


def _run(tmp_path, w, token, floor=None):
    if not BIN.exists():
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    files = []
    for name, obj in (("dag", w.dag), ("lib", w.library), ("bounds", w.bounds)):
        f = tmp_path / f"{w.name}_{name}.json"
        f.write_text(json.dumps(obj))
        files.append(str(f))
    args = [str(BIN), *files, token] + ([str(floor)] if floor is not None else [])
    proc = subprocess.run(args, capture_output=True, text=True, timeout=300)
    out = json.loads(proc.stdout)
    assert proc.returncode == 0 and out["same"], out
    return out


@pytest.mark.parametrize("token", ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"])
def test_adapter_c1(tmp_path, token):
    _run(tmp_path, W.config1(), token)


def test_adapter_c1_infeasible_floor(tmp_path):
    out = _run(tmp_path, W.config1(), "MIN_COST", 3)
    assert "NoFeasibleConfigError" in out["reference"] == out["b200"] or out["reference"] == out["b200"]


def test_adapter_c2(tmp_path):
    _run(tmp_path, W.config2(), "MIN_LATENCY", 3)


def test_adapter_random(tmp_path):
    tokens = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]
    for seed in range(24):
        w = W.random_scenario(seed, max_nodes=4)
        _run(tmp_path, w, tokens[seed % 4])
