"""GPU parity of the per-plan estimate streams (loom_estimate_range /
_device / loom_estimate_plans): estimate() (estimator.hpp:43-78) for every
plan of a range, in ConfigEnumerator order, against the reference's golden
estimates (tests/golden/c1, made by the compiled reference) and the CPU
oracle on the same inputs.  The bar is bit-exact: identical integers and
bit-identical doubles."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2501_16634_b200 import loom, workloads as W

pytestmark = pytest.mark.gpu
FIELDS = ("latency_us", "gpu_wh", "cpu_wh", "total_wh", "dollars", "quality")
TILE = 32 * 17  # plans per warp tile of the range kernel


def _oracle_arrays(p, begin, end):
    est = O.estimates(p, begin, end)
    return {k: np.array([e[k] for e in est], dtype=loom.STREAM_FIELDS[k]) for k in FIELDS}


def _same(got: dict, ref: dict, fields=FIELDS):
    for k in fields:
        a, b = got[k], ref[k]
        assert a.shape == b.shape, k
        # bit-exact: compare the raw bits (doubles included)
        bad = np.flatnonzero(a.view(f"u{a.itemsize}") != b.view(f"u{b.itemsize}"))
        assert bad.size == 0, (k, bad[:5], a[bad[:5]], b[bad[:5]])


def _setup(w):
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    return lw, O.problem(w.dag, w.library, w.bounds)


def test_c1_all_plans_vs_reference_goldens(ctx, golden):
    """Every one of the 168 plans against the compiled reference's estimate()."""
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    got = loom.estimate_range(ctx, lw.problem, 0, lw.total)
    ref = golden("c1/results.json")["estimates"]
    assert len(ref) == lw.total == 168
    for row in ref:
        i, lat, g, c, t, d, q = row
        assert got["latency_us"][i] == lat
        assert got["gpu_wh"][i] == g and got["cpu_wh"][i] == c and got["total_wh"][i] == t
        assert got["dollars"][i] == d and got["quality"][i] == q


def test_c1_plans_gather(ctx, golden):
    w = W.config1()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    ref = {r[0]: r for r in golden("c1/results.json")["estimates"]}
    idx = [167, 0, 42, 162, 42, 5, 100]
    got = loom.estimate_plans(ctx, lw.problem, idx)
    for k, i in enumerate(idx):
        assert [got[f][k] for f in FIELDS] == ref[i][1:]


@pytest.mark.parametrize("cfg", ["c2", "c3", "c5"])
def test_ragged_ranges_vs_oracle(ctx, cfg):
    """Ranges that start and end inside tiles, inside rows, cross prefix
    carries, single plans, and whole multi-tile spans."""
    w = {"c2": W.config2, "c3": W.config3, "c5": W.config5}[cfg]()
    lw, p = _setup(w)
    total = lw.total
    rng = random.Random(7)
    ranges = [(0, 1), (0, TILE), (0, TILE + 1), (1, 2 * TILE + 3), (total - 5, total), (total - TILE - 7, total),
              (12345, 12345 + 3 * TILE)]
    for _ in range(6):
        b = rng.randrange(0, total - 50_000)
        ranges.append((b, b + rng.randrange(1, 50_000)))
    for b, e in ranges:
        got = loom.estimate_range(ctx, lw.problem, b, e)
        _same(got, _oracle_arrays(p, b, e))


def test_field_subsets_and_clamping(ctx):
    w = W.config3()
    lw, p = _setup(w)
    b = 987_654_321
    got = loom.estimate_range(ctx, lw.problem, b, b + 5000, fields=("gpu_wh", "quality"))
    assert set(got) == {"gpu_wh", "quality"}
    _same(got, _oracle_arrays(p, b, b + 5000), fields=("gpu_wh", "quality"))
    # end past the plan space is clamped; an empty range writes nothing
    tail = loom.estimate_range(ctx, lw.problem, lw.total - 3, lw.total - 3 + 3)
    _same(tail, _oracle_arrays(p, lw.total - 3, lw.total))
    empty = loom.estimate_range(ctx, lw.problem, 10, 10)
    assert all(v.size == 0 for v in empty.values())


def test_device_streams_aligned_and_unaligned(ctx):
    """Device arrays, 16-byte aligned and offset by one element; ranges that
    start and end inside groups."""
    import torch
    w = W.config3()
    lw, p = _setup(w)
    b, n = 55_555_555, 40 * TILE + 77
    ref = _oracle_arrays(p, b, b + n)
    for off in (0, 1):
        dt = {"int64": torch.int64, "float64": torch.float64, "int32": torch.int32}
        bufs = {k: torch.full((n + 4,), -1, dtype=dt[loom.STREAM_FIELDS[k]], device="cuda") for k in FIELDS}
        views = {k: (t[off:off + n] if loom.STREAM_FIELDS[k] != "int32" else t[2 * off:2 * off + n])
                 for k, t in bufs.items()}
        torch.cuda.synchronize()
        loom.estimate_range_device(ctx, lw.problem, b, b + n, views)
        torch.cuda.synchronize()
        _same({k: v.cpu().numpy() for k, v in views.items()}, ref)


def test_random_scenarios_vs_oracle(ctx, golden):
    """The 80 random scenarios of the argmin goldens: every plan, every field."""
    for seed in range(0, 80, 4):
        w = W.random_scenario(seed)
        lw, p = _setup(w)
        if lw.total == 0:
            continue
        end = min(lw.total, 200_000)
        _same(loom.estimate_range(ctx, lw.problem, 0, end), _oracle_arrays(p, 0, end))


def test_gather_random_indices_vs_oracle(ctx):
    w = W.config3()
    lw, p = _setup(w)
    rng = random.Random(3)
    idx = [rng.randrange(lw.total) for _ in range(3000)] + [0, lw.total - 1]
    got = loom.estimate_plans(ctx, lw.problem, idx)
    for k, i in enumerate(idx[:400]):
        e = O.estimates(p, i, i + 1)[0]
        for f in FIELDS:
            assert got[f][k] == e[f], (i, f)
    with pytest.raises(loom.InvalidConfigError, match="plan index out of range"):
        loom.estimate_plans(ctx, lw.problem, [lw.total])


def test_full_size_stream_argmin_matches_search(ctx):
    """Size-independent property at scale: the MIN_COST-under-SLO argmin taken
    over a 2^27-plan C3 score stream (quantize, then latency, then identifier
    rank) equals the search kernel's winner on the same range."""
    import torch
    w = W.config3()
    lw, _ = _setup(w)
    b, n = 3 * 10**11 + 17, 1 << 27
    dev = {k: torch.empty(n, dtype=torch.float64 if k == "gpu_wh" else torch.int64, device="cuda")
           for k in ("gpu_wh", "latency_us")}
    loom.estimate_range_device(ctx, lw.problem, b, b + n, dev)
    torch.cuda.synchronize()
    obj = loom.objective({"constraint": "MIN_COST", "latency_slo_us": W.C3_SLO_US})
    win = loom.search_argmin(ctx, lw.problem, obj, b, b + n)
    feas = dev["latency_us"] <= W.C3_SLO_US
    x = dev["gpu_wh"] * 1e9  # quantize = llround(v * 1e9), half away from zero (estimator.hpp:85-87)
    t = torch.trunc(x)
    q = t + (x - t >= 0.5).double() - (x - t <= -0.5).double()
    q = torch.where(feas, q, torch.full_like(q, float("inf")))
    qmin = q.min()
    cand = torch.nonzero(q == qmin).flatten()
    lat = dev["latency_us"][cand]
    cand = cand[lat == lat.min()]
    i = int(cand[0]) if cand.numel() == 1 else None
    if i is not None:
        assert b + i == win["plan_index"]
    else:  # residual tie: the search picked one of them
        assert (win["plan_index"] - b) in set(cand.tolist())
    assert dev["latency_us"][win["plan_index"] - b].item() == win["latency_us"]
    assert dev["gpu_wh"][win["plan_index"] - b].item() == win["gpu_wh"]


def _scaled_problem(lw, wall_scale: int):
    """A copy of a lowered problem with every wall multiplied (exercises the
    64-bit latency fold: walls beyond 2^30 us)."""
    import ctypes as C
    pr = lw.problem
    n, m = pr.n_nodes, lw.n_options
    keep = []

    def arr(ct, vals):
        a = (ct * max(1, len(vals)))(*vals)
        keep.append(a)
        return C.cast(a, C.POINTER(ct))

    q = loom.Problem()
    q.n_nodes, q.n_edges = n, pr.n_edges
    q.radix = arr(C.c_int32, [pr.radix[i] for i in range(n)])
    q.wall_us = arr(C.c_int64, [pr.wall_us[i] * wall_scale for i in range(m)])
    for f, ct in (("gpu_wh", C.c_double), ("cpu_wh", C.c_double), ("dollars", C.c_double),
                  ("quality", C.c_int32), ("lexrank", C.c_int32)):
        setattr(q, f, arr(ct, [getattr(pr, f)[i] for i in range(m)]))
    q.lex_weight = arr(C.c_uint64, [pr.lex_weight[i] for i in range(n)])
    q.edge_from = arr(C.c_int32, [pr.edge_from[i] for i in range(pr.n_edges)])
    q.edge_to = arr(C.c_int32, [pr.edge_to[i] for i in range(pr.n_edges)])
    q._keep = keep
    return q


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_wide_walls_int64_latency_path(ctx, cfg):
    """Walls scaled x1000 (latencies beyond 2^30 us): the range kernel's
    64-bit max-plus fold against the host's exact per-plan estimate."""
    w = {"c3": W.config3, "c5": W.config5}[cfg]()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    q = _scaled_problem(lw, 1000)
    b = 777_777_777 % lw.total
    got = loom.estimate_range(ctx, q, b, b + 3 * 4096 + 5)
    import ctypes as C
    for k in list(range(0, 3 * 4096 + 5, 97)) + [3 * 4096 + 4]:
        ref = loom.Winner()
        assert loom.lib().loom_evaluate_plan(C.byref(q), b + k, C.byref(ref)) == 0
        assert got["latency_us"][k] == ref.latency_us and ref.latency_us >= (1 << 30)
        for f in ("gpu_wh", "cpu_wh", "total_wh", "dollars", "quality"):
            assert got[f][k] == getattr(ref, f)


def test_single_node_and_tiny_spaces(ctx):
    """One-node DAGs and plan spaces smaller than a warp (groups of < 32 plans)."""
    for seed in range(200, 260):
        w = W.random_scenario(seed, max_nodes=2)
        lw, p = _setup(w)
        if lw.total == 0:
            continue
        _same(loom.estimate_range(ctx, lw.problem, 0, lw.total), _oracle_arrays(p, 0, lw.total))
