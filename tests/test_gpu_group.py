"""Multi-GPU inside the library: a loom_group owns the member
contexts and the NCCL communicator, shards the plan space by contiguous
index ranges with a common greedy incumbent, and all-gathers the per-rank
records with ncclAllGather.  On the one-GPU box the group has one device
(device mask 1), which runs the real NCCL path (ncclCommInitAll + the
all-gathers) end to end and must be bit-identical to the single-context
calls; the N > 1 shard logic is covered on CPU (tests/test_distributed.py).
Also the C++ drop-in (include/loom_b200/loom.hpp) compiled and run:
loom::pareto_filter on the reference's own test shapes, and
loom::exhaustive_search through a group."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def group(loomlib):
    g = loom.Group(device_mask=1)
    yield g
    g.close()


def test_group_shape(group):
    assert group.world == 1 and group.local == 1 and group.rank == 0


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_group_argmin_equals_single_context(ctx, group, cfg):
    w = {"c1": W.config1(), "c2": W.config2(), "c3": W.config3(slo_us=W.C3_BINDING_SLO_US)}[cfg]
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    for o in (w.objective, {"constraint": "MIN_LATENCY"}, {"constraint": "MAX_QUALITY"}):
        ob = loom.objective(o)
        assert group.search_argmin(lw.problem, ob) == loom.search_argmin(ctx, lw.problem, ob)
    lw.close()


def test_group_json_dropin(ctx, group, golden):
    w = W.config3(slo_us=W.C3_BINDING_SLO_US)
    case = next(c for c in golden("c3/full_space.json")["cases"] if c["objective"] == w.objective)
    est = group.exhaustive_search(*w.texts())
    assert est["plan_index"] == case["winner"]["index"] and est["identifier"] == case["identifier"]
    assert est == loom.exhaustive_search(*w.texts(), ctx=ctx)
    with pytest.raises(loom.NoFeasibleConfigError):
        group.exhaustive_search(w.dag, w.library, {"constraint": "MIN_COST", "latency_slo_us": 1}, w.bounds)


def test_group_pareto_equals_single_context(ctx, group, golden):
    w = W.config5(n_nodes=7)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    assert group.search_pareto_points(lw.problem) == loom.search_pareto_points(ctx, lw.problem)
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    assert [p["plan_index"] for p in group.search_pareto_points(lw.problem)] == [42, 162]


def test_group_batch_equals_single_context(ctx, group):
    jobs = W.config4(300)
    lws = [loom.Lowered(j.dag, j.library, j.bounds) for j in jobs]
    objs = [loom.objective(W.c4_slo_objective(loom.latency_floor(lw.problem))) for lw in lws]
    a = group.search_argmin_batch([lw.problem for lw in lws], objs)
    b = loom.search_argmin_batch(ctx, [lw.problem for lw in lws], objs)
    assert a == b


def _dropin_binary(tmp_path_factory) -> Path:
    exe = tmp_path_factory.mktemp("dropin") / "dropin_check"
    pkg = ROOT / "paper_2501_16634_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/dropin_check.cpp"),
                    "-o", str(exe), f"-L{pkg}", "-lloom_b200", f"-Wl,-rpath,{pkg}"], check=True)
    return exe


def test_cpp_dropin_pareto_filter(loomlib, tmp_path_factory):
    """loom::pareto_filter (optimizer.hpp:153-171) through the C++ drop-in, on
    the device: test_optimizer.cpp:259-327 and acceptance.cpp:202-234 shapes
    against the quadratic oracle (stable order, duplicates kept)."""
    exe = _dropin_binary(tmp_path_factory)
    r = subprocess.run([str(exe), "pareto"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok pareto" in r.stdout, r.stdout + r.stderr


def test_cpp_dropin_group_search(loomlib, tmp_path_factory):
    exe = _dropin_binary(tmp_path_factory)
    g = ROOT / "tests" / "golden" / "c1"
    r = subprocess.run([str(exe), "group", str(g / "dag.json"), str(g / "library.json"), str(g / "bounds.json")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok group" in r.stdout, r.stdout + r.stderr
