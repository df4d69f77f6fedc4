"""Config points / --pin files (§8f rank 1): parse_config_point
(config.hpp:66-117) and the host estimate of a pinned config
(loom_estimate_config_json; the reference's --pin path, loom_main.cpp:125-146)
against the compiled reference's estimates of every C1 plan
(tests/golden/c1/results.json "estimates", from oracle/_ref)."""
import json

import pytest

from paper_2501_16634_b200 import loom, workloads as W

FIELDS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")


@pytest.fixture(scope="module")
def c1(golden):
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    yield w, lw, golden("c1/results.json")
    lw.close()


def _check(est, row):
    idx, lat, gpu, cpu, tot, dol, q = row
    assert [est[k] for k in FIELDS] == [lat, gpu, cpu, tot, dol, q], idx


def test_every_c1_plan_round_trips_through_its_config_point(c1):
    w, lw, g = c1
    for row in g["estimates"]:
        cfg = lw.config(row[0])
        ident = cfg.pop("identifier")
        est = loom.estimate_config(w.dag, w.library, json.dumps(cfg))
        _check(est, row)
        assert est["identifier"] == ident
        assert "plan_index" not in est


def test_published_pins(c1):
    """The paper's pinned plans (fixture pin_*.json): each is a plan of the C1
    space; its estimate equals the reference's estimate of that plan."""
    w, lw, g = c1
    by_id = {lw.config(r[0])["identifier"]: r for r in g["estimates"]}
    for name, pin in g["pins"].items():
        est = loom.estimate_config(w.dag, w.library, json.dumps(pin))
        _check(est, by_id[est["identifier"]])
        assert est["config"]["label"] == pin["label"], name


def test_defaults(c1):
    """workers and path_count default to 1, label to "" (config.hpp from_json)."""
    w, lw, g = c1
    pin = json.loads(json.dumps(next(iter(g["pins"].values()))))
    pin.pop("label")
    for a in pin["nodes"].values():
        a.pop("path_count")
        for p in a["placements"]:
            if p["workers"] == 1:
                p.pop("workers")
    est = loom.estimate_config(w.dag, w.library, json.dumps(pin))
    assert est["config"]["label"] == ""
    full = loom.estimate_config(w.dag, w.library, json.dumps(next(iter(g["pins"].values()))))
    assert [est[k] for k in FIELDS] == [full[k] for k in FIELDS]


@pytest.mark.parametrize("mutate, cls, msg", [
    (lambda p: p.pop("nodes"), loom.SchemaError, "malformed config point"),
    (lambda p: next(iter(p["nodes"].values())).update(implementation=""), loom.SchemaError, "empty implementation"),
    (lambda p: next(iter(p["nodes"].values())).update(placements=[]), loom.SchemaError, "no placements"),
    (lambda p: next(iter(p["nodes"].values()))["placements"][0].update(units=0), loom.SchemaError,
     "units and workers must be >= 1"),
    (lambda p: next(iter(p["nodes"].values()))["placements"][0].update(workers=0), loom.SchemaError,
     "units and workers must be >= 1"),
    (lambda p: next(iter(p["nodes"].values())).update(path_count=0), loom.SchemaError, "path_count must be >= 1"),
    (lambda p: p["nodes"].pop(sorted(p["nodes"])[-1]), loom.ValidationError, "pinned_plan: missing assignment"),
])
def test_rejections(c1, mutate, cls, msg):
    w, lw, g = c1
    pin = json.loads(json.dumps(next(iter(g["pins"].values()))))
    mutate(pin)
    with pytest.raises(cls, match=msg):
        loom.estimate_config(w.dag, w.library, json.dumps(pin))


def test_malformed_text(c1):
    w, _, _ = c1
    with pytest.raises(loom.SchemaError, match="malformed config point"):
        loom.estimate_config(w.dag, w.library, "{not json")
