"""Host side of the product, no GPU needed: the C ABI library loads and
exports every entry point include/loom_b200.h declares; the C++ lowering
(node_options + plan_node_execution + identifier ranks) is bit-identical to
the oracle's restatement; host estimate / total order / objective parsing and
error behaviour mirror the reference."""
import ctypes as C
import random
import subprocess
from pathlib import Path

import pytest

from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

TOKENS = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]


def test_library_exports_every_declared_symbol(loomlib):
    declared = loom.exported_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(loom.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(loomlib, s)
    assert loomlib.loom_abi_version() == 1


def _workloads():
    yield W.config1()
    yield W.config2()
    yield W.config3()
    yield W.config5()
    yield from W.config4(3)
    for seed in range(0, 40):
        yield W.random_scenario(seed)


@pytest.mark.parametrize("w", list(_workloads()), ids=lambda w: w.name)
def test_lowering_bit_identical_to_oracle(loomlib, w):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    assert lw.radix == p.lowered.radix
    assert lw.total == p.total
    flat = [(pl, op, q, t) for pls, ops, qs, ts in zip(p.lowered.plans, p.lowered.options, p.lowered.quality,
                                                        p.lowered.tokens) for pl, op, q, t in zip(pls, ops, qs, ts)]
    wall, gpu, cpu, dol = (lw.table(n) for n in ("wall_us", "gpu_wh", "cpu_wh", "dollars"))
    qual, rank = lw.table("quality"), lw.table("lexrank")
    for k, (pl, op, q, tok) in enumerate(flat):
        k_paths = op["path_count"]
        assert wall[k] == pl["wall_us"]
        assert gpu[k] == pl["gpu_wh"] * k_paths
        assert cpu[k] == pl["cpu_wh"] * k_paths
        assert dol[k] == pl["dollars"] * k_paths
        assert qual[k] == q
    # identifier ranks per node and the sorted-id weights
    off = 0
    for i, toks in enumerate(p.lowered.tokens):
        order = sorted(range(len(toks)), key=lambda j: toks[j].encode())
        for r, j in enumerate(order):
            assert rank[off + j] == r
        off += len(toks)
    ids = p.lowered.node_ids
    by_id = sorted(range(len(ids)), key=lambda i: ids[i].encode())
    weight, expect = lw.table("lex_weight"), 1
    for i in reversed(by_id):
        assert weight[i] == expect
        expect *= p.lowered.radix[i]


@pytest.mark.parametrize("w", [W.config1(), W.config2(), W.config3(), W.random_scenario(7)], ids=lambda w: w.name)
def test_lexkey_order_equals_identifier_order(loomlib, w):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    rng = random.Random(5)
    picks = [rng.randrange(p.total) for _ in range(300)]
    keyed = [(lw.evaluate(i)["lexkey"], O.identifier(p, i), i) for i in picks]
    assert sorted(keyed, key=lambda t: t[0]) == sorted(keyed, key=lambda t: t[1].encode())
    for i in picks[:40]:
        assert lw.config(i)["identifier"] == O.identifier(p, i)


@pytest.mark.parametrize("w", [W.config1(), W.config2(), W.config3(), W.config5()], ids=lambda w: w.name)
def test_host_evaluate_matches_oracle(loomlib, w):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    rng = random.Random(11)
    for i in [0, p.total - 1] + [rng.randrange(p.total) for _ in range(200)]:
        a, b = lw.evaluate(i), O.estimates(p, i, i + 1)[0]
        for k in ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality"):
            assert a[k] == b[k], k


def test_winner_order_and_reduce(loomlib):
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for token in TOKENS:
        obj = loom.objective(token)
        winners = [loom.winner_from_dict(lw.evaluate(i)) for i in range(lw.total)]
        best = loom.winner_reduce(winners, obj)
        assert best["plan_index"] == O.argmin(p, {"constraint": token})["index"]
        # order independence
        rng = random.Random(3)
        rng.shuffle(winners)
        assert loom.winner_reduce(winners, obj)["plan_index"] == best["plan_index"]
    with pytest.raises(loom.NoFeasibleConfigError):
        loom.winner_reduce([loom.Winner(), loom.Winner()], loom.objective("MIN_COST"))


def test_objective_parse():
    o = loom.objective({"constraint": "MAX_QUALITY", "quality_floor": 3, "latency_slo_us": 99})
    assert o.n_criteria == 3 and list(o.criteria)[:3] == [3, 1, 2]
    assert o.has_quality_floor == 1 and o.quality_floor == 3 and o.has_latency_slo == 1 and o.latency_slo_us == 99
    o = loom.objective({"criteria": ["min_cost_dollars", "min_energy"]})
    assert o.n_criteria == 2 and list(o.criteria)[:2] == [0, 1]
    with pytest.raises(loom.SchemaError, match="unknown constraint token 'FASTEST'"):
        loom.objective("FASTEST")


def test_lowering_errors_mirror_reference(loomlib):
    w = W.config1()
    dag = {"nodes": w.dag["nodes"] + [dict(w.dag["nodes"][0], id="t9_x", capability="nope")], "edges": w.dag["edges"]}
    with pytest.raises(loom.UnknownCapabilityError, match="capability 'nope' is not registered"):
        loom.Lowered(dag, w.library, w.bounds)
    cyc = {"nodes": w.dag["nodes"], "edges": w.dag["edges"] + [
        {"from": "t3_summarization", "to": "t0_frame_extraction", "kind": "text"}]}
    with pytest.raises(loom.CycleError):
        loom.Lowered(cyc, w.library, w.bounds)
    with pytest.raises(loom.SchemaError):
        loom.Lowered("{not json", w.library, w.bounds)
    bad = dict(w.library, profiles=w.library["profiles"] + [dict(w.library["profiles"][0], units=99, throughput=0)])
    with pytest.raises(loom.ValidationError, match="throughput must be > 0"):
        loom.Lowered(w.dag, bad, w.bounds)


def test_empty_dag_has_no_plans(loomlib):
    w = W.config1()
    lw = loom.Lowered({"nodes": [], "edges": []}, w.library, w.bounds)
    assert lw.total == 0


def test_device_entry_points_fail_loudly_without_gpu(loomlib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(loom.DeviceError, match="no CUDA device"):
        loom.Context(0)


def _tables(lw):
    return [lw.table(t) for t in ("wall_us", "gpu_wh", "cpu_wh", "dollars", "quality", "lexrank", "lex_weight")]


def test_dag_fast_reader_equals_dom_reader(loomlib):
    """WorkflowDag::from_json_text reads dag.json with a DOM-free cursor and
    falls back to the DOM reader on anything unusual; both must give the same
    lowering (escaped strings, reordered / extra / duplicate keys, a null or
    integral-real path_quality_ceiling, whitespace) and the same errors."""
    import json
    for w in (W.config1(), W.config3(), W.config5(n_nodes=5)) + tuple(W.config4(3)):
        ref = loom.Lowered(json.dumps(w.dag), w.library, w.bounds)
        variants = [
            json.dumps(w.dag, indent=3),
            json.dumps(w.dag, ensure_ascii=True).replace('"t0', '"\\u0074' + "0"),  # escape -> DOM path
            json.dumps({"edges": w.dag["edges"], "extra": [1, {"a": None}], "nodes": [
                dict(reversed(list(n.items())), note="x\\ny", path_quality_ceiling=None) for n in w.dag["nodes"]]}),
        ]
        for text in variants:
            got = loom.Lowered(text, w.library, w.bounds)
            assert got.radix == ref.radix and _tables(got) == _tables(ref)
            assert got.config(0)["identifier"] == ref.config(0)["identifier"]
    w = W.config1()
    nodes = [dict(n) for n in w.dag["nodes"]]
    nodes[1]["path_quality_ceiling"] = 2.0  # integral real: DOM reader accepts it
    a = loom.Lowered(json.dumps({"nodes": nodes, "edges": w.dag["edges"]}), w.library, w.bounds)
    nodes[1]["path_quality_ceiling"] = 2
    b = loom.Lowered(json.dumps({"nodes": nodes, "edges": w.dag["edges"]}), w.library, w.bounds)
    assert _tables(a) == _tables(b)
    dup = json.dumps({"nodes": w.dag["nodes"], "edges": w.dag["edges"]})[:-1] + ', "nodes": []}'
    with pytest.raises(loom.CycleError):  # duplicate key: the DOM reader's semantics (the later "nodes" wins)
        loom.Lowered(dup, w.library, w.bounds)
    for bad in ('{"nodes": [{"id": "a"}], "edges": []}', '{"nodes": []}', '{"nodes": [], "edges": [{"from": "a"}]}',
                '[1, 2]', '{"nodes": [], "edges": []} trailing'):
        with pytest.raises(loom.LoomError):
            loom.Lowered(bad, w.library, w.bounds)


def test_bench_fast_path_matches_compiled_sass(loomlib):
    """bench.py's roofline divides by the compiled fast path's instruction
    counts; they must be the ones in the object file that was built (the
    fully unrolled energy-first sweep of search_kernel<4, kPrimFp, 16, true>)."""
    import shutil
    import subprocess
    import sys
    if not (shutil.which("cuobjdump") or Path("/usr/local/cuda/bin/cuobjdump").exists()):
        pytest.skip("no cuobjdump")
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "tools" / "sass_blocks.py"), "4", "0", "16", "1", "200"],
                         capture_output=True, text=True, check=True).stdout
    import re
    rows = [tuple(int(x) for x in re.search(r"issue\s+(\d+)\s+alu\s+(\d+)\s+fp64\s+(\d+)", l).groups())
            for l in out.splitlines() if "issue" in l]
    assert rows, out
    sys.path.insert(0, str(root))
    import bench
    fp = bench.FAST_PATH
    assert (fp["issue"], fp["alu"], fp["fp64"]) in rows, (fp, rows)


@pytest.mark.parametrize("w", list(_workloads())[:12], ids=lambda w: w.name)
def test_latency_floor_is_min_latency(loomlib, w):
    """loom_latency_floor (every node at its fastest option meeting the
    floor) equals the latency of the oracle's MIN_LATENCY argmin."""
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    p = O.problem(w.dag, w.library, w.bounds)
    for extra in ({}, {"quality_floor": 2}):
        o = {"constraint": "MIN_LATENCY", **extra}
        ref = O.argmin(p, o, 0, min(p.total, 2_000_000)) if p.total <= 2_000_000 else None
        try:
            got = loom.latency_floor(lw.problem, loom.objective(o))
        except loom.NoFeasibleConfigError:
            assert ref is None or p.total > 2_000_000
            continue
        if ref is not None:
            assert got == ref["latency_us"]
    lw.close()


def test_batch_objective_array_is_validated(loomlib):
    """The multi-tenant JSON call takes one objective or one per job; a
    mismatched array is a schema error (status 2), before any device work."""
    jobs = W.config4(3)
    import json

    class _Unused:  # the objectives are parsed before the context is touched
        handle = C.c_void_p(16)

    with pytest.raises(loom.LoomError, match="objective array has 2 entries for 3 jobs"):
        loom.exhaustive_search_batch([j.dag for j in jobs], json.dumps(jobs[0].library),
                                     [{"constraint": "MIN_COST"}] * 2, json.dumps(jobs[0].bounds), ctx=_Unused())


def test_batch_lowering_cache_equals_plain_lowering(loomlib):
    """loom_lower_batch memoises option sets across the DAGs of a batch
    (LowerCache); every table, option config and identifier must equal the
    plain per-DAG lowering: 300 C4 jobs (one library), and per random
    scenario a batch of the scenario's DAG with work units and chunks
    perturbed (same capabilities, other fan-out caps / split validity)."""
    import json as _json
    jobs = W.config4(300)
    cases = [([j.dag for j in jobs], jobs[0].library, jobs[0].bounds)]
    rng = random.Random(11)
    for seed in range(0, 40, 2):
        w = W.random_scenario(seed)
        dags = []
        for _ in range(6):
            d = _json.loads(_json.dumps(w.dag))
            for node in d["nodes"]:
                node["work_units"] = node["work_units"] * rng.choice([0.25, 0.5, 1.0, 2.0, 5.0])
                if node.get("min_chunk"):
                    node["min_chunk"] = node["min_chunk"] * rng.choice([0.5, 1.0, 3.0])
            dags.append(d)
        cases.append((dags, w.library, w.bounds))
    for dags, lib_, bounds in cases:
        batch = loom.LoweredBatch(dags, lib_, bounds, threads=2)
        for k, d in enumerate(dags):
            plain = loom.Lowered(d, lib_, bounds)
            got = batch[k]
            assert _tables(got) == _tables(plain), k
            for idx in {0, plain.total // 3, plain.total - 1}:
                assert got.config(idx) == plain.config(idx)
            for node in range(plain.problem.n_nodes):
                for opt in range(plain.problem.radix[node]):
                    assert got.option(node, opt) == plain.option(node, opt)
            plain.close()
        batch.close()


def test_library_fast_reader_equals_dom_reader(loomlib):
    """AgentLibrary::from_json_text reads the library bundle with a DOM-free
    cursor and falls back to the DOM reader on anything unusual; both must
    give the same lowering (reordered / extra keys, escapes, whitespace) and
    the same errors (duplicates, dangling references, bad classes)."""
    import json
    for w in (W.config1(), W.config2(), W.config3(), W.config5(n_nodes=5)) + tuple(W.config4(2)):
        ref = loom.Lowered(w.dag, json.dumps(w.library), w.bounds)
        lib = w.library
        variants = [
            json.dumps(lib, indent=2),
            json.dumps({k: lib[k] for k in reversed(list(lib))}),  # section order: registration order is fixed
            json.dumps(dict(lib, note="\\u0041 escaped", extra=[{"x": None}])).replace("escaped", "\\u0065"),
            json.dumps({k: [dict(reversed(list(e.items())), comment="c") if isinstance(e, dict) else e for e in v]
                        if isinstance(v, list) else v for k, v in lib.items()}),
        ]
        for text in variants:
            got = loom.Lowered(w.dag, text, w.bounds)
            assert got.radix == ref.radix and _tables(got) == _tables(ref)
            assert got.config(got.total - 1)["identifier"] == ref.config(ref.total - 1)["identifier"]
    w = W.config1()
    lib = json.loads(json.dumps(w.library))
    bad = []
    d = json.loads(json.dumps(lib)); d["skus"].append(dict(d["skus"][0])); bad.append((d, loom.LoomError))
    d = json.loads(json.dumps(lib)); d["profiles"][0]["sku"] = "nope"; bad.append((d, loom.LoomError))
    d = json.loads(json.dumps(lib)); d["skus"][0]["class"] = "tpu"; bad.append((d, loom.SchemaError))
    d = json.loads(json.dumps(lib)); del d["profiles"][0]["units"]; bad.append((d, loom.SchemaError))
    d = json.loads(json.dumps(lib)); d["implementations"][0]["quality"] = 1.5; bad.append((d, loom.SchemaError))
    for d, cls in bad:
        with pytest.raises(cls):
            loom.Lowered(w.dag, json.dumps(d), w.bounds)
