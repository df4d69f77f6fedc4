"""The batch search's host staging (loomi::argmin_batch): jobs lowered, built
and packed block by block into the pinned arena, with the copy of each block
queued as soon as it is packed.  Blocks that do not fit the arena sized from
the previous batch ("late" blocks) are staged after the others; the
LOOM_BATCH_HINT test knob shrinks the arena so that every path runs: all
blocks late, some late, none late.  Every answer is checked against the
full-space goldens of C4 (tests/golden/c4/all_jobs.json)."""
import json
import os

import pytest

from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu


def _check(res, gold, ks):
    mism = []
    for i, k in enumerate(ks):
        st, got = res[i]
        g = gold[k]
        if g is None:
            assert st == loom.LOOM_INFEASIBLE
            continue
        assert st == 0
        if [got["plan_index"], got["latency_us"], got["gpu_wh"], got["dollars"]] != g:
            mism.append(k)
    assert not mism, mism[:10]


@pytest.mark.parametrize("hint", ["1", "6000", None])
def test_batch_staging_late_blocks(golden, hint):
    gold = golden("c4/all_jobs.json")["objectives"]["MIN_LATENCY"]
    jobs = W.config4(10_000)
    ks = list(range(0, 10_000, 7))  # 1,429 jobs: 23 blocks, the last one partial
    dags = [json.dumps(jobs[k].dag).encode() for k in ks]
    lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
    obj_t = json.dumps({"constraint": "MIN_LATENCY"})
    old = os.environ.pop("LOOM_BATCH_HINT", None)
    try:
        if hint is not None:
            os.environ["LOOM_BATCH_HINT"] = hint
        with loom.Context(0) as ctx:  # fresh: no image-size history
            for _ in range(2):  # the second call sizes the arena from the first
                res = loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
                _check(res, gold, ks)
    finally:
        os.environ.pop("LOOM_BATCH_HINT", None)
        if old is not None:
            os.environ["LOOM_BATCH_HINT"] = old


def test_batch_staging_failed_jobs(golden):
    """Jobs that fail to lower (malformed dag.json, a cycle) sit between good
    ones in the same blocks: their status is set, the others are unaffected."""
    gold = golden("c4/all_jobs.json")["objectives"]["MIN_LATENCY"]
    jobs = W.config4(400)
    dags = [json.dumps(j.dag).encode() for j in jobs]
    bad = {5: b"{not json", 77: None, 130: None}
    for k in (77, 130):  # a cycle: the last edge reversed onto the first node
        d = json.loads(dags[k])
        d["edges"].append({"from": d["nodes"][-1]["id"], "to": d["nodes"][0]["id"]})
        bad[k] = json.dumps(d).encode()
    for k, v in bad.items():
        dags[k] = v
    with loom.Context(0) as ctx:
        res = loom.exhaustive_search_batch(dags, json.dumps(jobs[0].library), json.dumps({"constraint": "MIN_LATENCY"}),
                                           json.dumps(jobs[0].bounds), ctx=ctx)
    for k in range(400):
        st, got = res[k]
        if k in bad:
            assert st == loom.LOOM_INVALID
            assert got["found"] == 0
            continue
        g = gold[k]
        assert st == 0 and [got["plan_index"], got["latency_us"], got["gpu_wh"], got["dollars"]] == g
