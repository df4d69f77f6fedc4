"""ORACLE TEST INFRASTRUCTURE -- NOT PRODUCT CODE.

Python driver of the CPU oracle: lowering restated in oracle/lower.py, the
per-plan work restated in plain C (oracle/flat_oracle.c, built by
oracle/Makefile into oracle/_build/).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference legs may import this, as the checker.

Also wraps the compiled UNMODIFIED reference (oracle/_ref/libloomref.so, built
from /root/reference by oracle/Makefile) when it is present.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

from . import lower as L

HERE = Path(__file__).resolve().parent
FLAT_SO = HERE / "_build" / "libflat_oracle.so"
REF_SO = HERE / "_ref" / "libloomref.so"


class OrProblem(C.Structure):
    _fields_ = [("n_nodes", C.c_int), ("n_edges", C.c_int), ("radix", C.POINTER(C.c_int)),
                ("wall", C.POINTER(C.c_int64)), ("gpu", C.POINTER(C.c_double)), ("cpu", C.POINTER(C.c_double)),
                ("dol", C.POINTER(C.c_double)), ("path_count", C.POINTER(C.c_int)),
                ("quality", C.POINTER(C.c_int)), ("token", C.POINTER(C.c_char_p)),
                ("id_order", C.POINTER(C.c_int)), ("topo", C.POINTER(C.c_int)),
                ("edge_from", C.POINTER(C.c_int)), ("edge_to", C.POINTER(C.c_int))]


class OrObjective(C.Structure):
    _fields_ = [("n_criteria", C.c_int), ("criteria", C.c_int * 4), ("has_floor", C.c_int), ("floor", C.c_int),
                ("has_slo", C.c_int), ("slo", C.c_int64)]


class OrEstimate(C.Structure):
    _fields_ = [("index", C.c_uint64), ("latency_us", C.c_int64), ("gpu_wh", C.c_double), ("cpu_wh", C.c_double),
                ("total_wh", C.c_double), ("dollars", C.c_double), ("quality", C.c_int), ("found", C.c_int)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def build_flat() -> Path:
    if not FLAT_SO.exists() or FLAT_SO.stat().st_mtime < (HERE / "flat_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "flat"], check=True)
    return FLAT_SO


_flat = None


def _lib():
    global _flat
    if _flat is None:
        _flat = C.CDLL(str(build_flat()))
        _flat.oracle_argmin.argtypes = [C.POINTER(OrProblem), C.POINTER(OrObjective), C.c_uint64, C.c_uint64,
                                        C.c_int, C.POINTER(OrEstimate)]
        _flat.oracle_estimates.argtypes = [C.POINTER(OrProblem), C.c_uint64, C.c_uint64, C.POINTER(OrEstimate)]
        _flat.oracle_argmin_bnb.argtypes = [C.POINTER(OrProblem), C.POINTER(OrObjective), C.c_int,
                                            C.POINTER(OrEstimate), C.POINTER(C.c_uint64)]
        _flat.oracle_pareto.argtypes = [C.POINTER(OrProblem), C.c_uint64, C.c_uint64, C.c_int,
                                        C.POINTER(OrEstimate), C.c_uint64, C.POINTER(C.c_uint64)]
    return _flat


def _arr(ctype, values):
    return (ctype * max(1, len(values)))(*values)


@dataclass
class OracleProblem:
    lowered: L.Lowered
    keep: list
    struct: OrProblem

    @property
    def total(self) -> int:
        return self.lowered.total


def problem(dag: dict, bundle: dict, bounds: dict) -> OracleProblem:
    return _from_lowered(L.lower(dag, bundle, bounds))


def subproblem(p: OracleProblem, keep: list[list[int]]) -> OracleProblem:
    """The plan space restricted to options keep[i] (ascending) of each node:
    the same DAG and option values, fewer options, so the flat per-plan loop
    can check the branch and bound on spaces the full loop cannot finish."""
    low = p.lowered
    pick = lambda per_node: [[lst[k] for k in ks] for lst, ks in zip(per_node, keep)]  # noqa: E731
    return _from_lowered(dataclasses.replace(low, options=pick(low.options), plans=pick(low.plans),
                                             quality=pick(low.quality), tokens=pick(low.tokens)))


def _from_lowered(low) -> OracleProblem:
    flat = [(p, o, q, t) for pl, op, ql, tl in zip(low.plans, low.options, low.quality, low.tokens)
            for p, o, q, t in zip(pl, op, ql, tl)]
    keep = []
    radix = _arr(C.c_int, low.radix)
    wall = _arr(C.c_int64, [f[0]["wall_us"] for f in flat])
    gpu = _arr(C.c_double, [f[0]["gpu_wh"] for f in flat])
    cpu = _arr(C.c_double, [f[0]["cpu_wh"] for f in flat])
    dol = _arr(C.c_double, [f[0]["dollars"] for f in flat])
    paths = _arr(C.c_int, [f[1]["path_count"] for f in flat])
    qual = _arr(C.c_int, [f[2] for f in flat])
    tok_bytes = [f[3].encode() for f in flat]
    toks = _arr(C.c_char_p, tok_bytes)
    id_order = _arr(C.c_int, sorted(range(len(low.node_ids)), key=lambda i: low.node_ids[i].encode()))
    topo = _arr(C.c_int, low.topo)
    efrom = _arr(C.c_int, [e[0] for e in low.edges])
    eto = _arr(C.c_int, [e[1] for e in low.edges])
    keep += [radix, wall, gpu, cpu, dol, paths, qual, tok_bytes, toks, id_order, topo, efrom, eto]
    s = OrProblem(len(low.node_ids), len(low.edges), radix, wall, gpu, cpu, dol, paths, qual, toks, id_order, topo,
                  efrom, eto)
    return OracleProblem(low, keep, s)


def objective_struct(objective: dict) -> OrObjective:
    crit = [L.CRITERIA[c] for c in L.objective_criteria(objective)]
    o = OrObjective()
    o.n_criteria = len(crit)
    for i, c in enumerate(crit):
        o.criteria[i] = c
    if objective.get("quality_floor") is not None:
        o.has_floor, o.floor = 1, int(objective["quality_floor"])
    if objective.get("latency_slo_us") is not None:
        o.has_slo, o.slo = 1, int(objective["latency_slo_us"])
    return o


def argmin(p: OracleProblem, objective: dict, begin: int = 0, end: int | None = None,
           threads: int | None = None) -> dict | None:
    end = p.total if end is None else min(end, p.total)
    threads = threads or os.cpu_count() or 1
    out = OrEstimate()
    o = objective_struct(objective)
    rc = _lib().oracle_argmin(C.byref(p.struct), C.byref(o), begin, end, threads, C.byref(out))
    if rc != 0:
        raise RuntimeError("oracle_argmin failed")
    return out.as_dict() if out.found else None


def argmin_bnb(p: OracleProblem, objective: dict, threads: int | None = None) -> tuple[dict | None, int]:
    """Exact argmin over the WHOLE space by branch and bound (flat_oracle.c:
    oracle_argmin_bnb); returns (winner or None, subtrees + leaves visited)."""
    threads = threads or os.cpu_count() or 1
    out = OrEstimate()
    vis = C.c_uint64(0)
    o = objective_struct(objective)
    rc = _lib().oracle_argmin_bnb(C.byref(p.struct), C.byref(o), threads, C.byref(out), C.byref(vis))
    if rc != 0:
        raise RuntimeError("oracle_argmin_bnb failed")
    return (out.as_dict() if out.found else None), vis.value


def estimates(p: OracleProblem, begin: int, end: int) -> list[dict]:
    n = max(0, end - begin)
    buf = (OrEstimate * max(1, n))()
    _lib().oracle_estimates(C.byref(p.struct), begin, end, buf)
    return [buf[i].as_dict() for i in range(n)]


def pareto(p: OracleProblem, begin: int = 0, end: int | None = None, threads: int | None = None) -> list[dict]:
    end = p.total if end is None else min(end, p.total)
    threads = threads or os.cpu_count() or 1
    cnt = C.c_uint64(0)
    cap = 1 << 20
    buf = (OrEstimate * cap)()
    _lib().oracle_pareto(C.byref(p.struct), begin, end, threads, buf, cap, C.byref(cnt))
    if cnt.value > cap:
        raise RuntimeError("frontier larger than oracle buffer")
    return [buf[i].as_dict() for i in range(cnt.value)]


def identifier(p: OracleProblem, index: int) -> str:
    low = p.lowered
    digits = []
    for r in reversed(low.radix):
        digits.append(index % r)
        index //= r
    digits.reverse()
    order = sorted(range(len(low.node_ids)), key=lambda i: low.node_ids[i].encode())
    return "".join(low.tokens[i][digits[i]] for i in order)


# ---------------------------------------------------------------------------
# the compiled reference (oracle/_ref), when present
# ---------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return REF_SO.exists()


def _reflib():
    global _ref
    if _ref is None:
        _ref = C.CDLL(str(REF_SO))
        _ref.loomref_free.argtypes = [C.c_void_p]
        for name, extra in [("loomref_plan", 3), ("loomref_lower", 3), ("loomref_pareto", 3)]:
            getattr(_ref, name).argtypes = [C.c_char_p] * extra + [C.POINTER(C.c_void_p)]
        _ref.loomref_search.argtypes = [C.c_char_p] * 5 + [C.POINTER(C.c_void_p)]
        _ref.loomref_enumerate.argtypes = [C.c_char_p] * 3 + [C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]
        _ref.loomref_range_argmin.argtypes = [C.c_char_p] * 4 + [C.c_uint64, C.c_uint64, C.c_int,
                                                                 C.POINTER(C.c_void_p)]
    return _ref


def _call(fn, *args) -> tuple[int, dict]:
    out = C.c_void_p()
    rc = fn(*args, C.byref(out))
    text = C.string_at(out.value).decode()
    _reflib().loomref_free(out)
    return rc, json.loads(text)


def _b(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def ref_search(dag, bundle, objective, bounds, mode="exhaustive") -> tuple[int, dict]:
    return _call(_reflib().loomref_search, _b(dag), _b(bundle), _b(objective), _b(bounds), mode.encode())


def ref_lower(dag, bundle, bounds) -> tuple[int, dict]:
    return _call(_reflib().loomref_lower, _b(dag), _b(bundle), _b(bounds))


def ref_pareto(dag, bundle, bounds) -> tuple[int, dict]:
    return _call(_reflib().loomref_pareto, _b(dag), _b(bundle), _b(bounds))


def ref_enumerate(dag, bundle, bounds, begin, end) -> tuple[int, list]:
    return _call(_reflib().loomref_enumerate, _b(dag), _b(bundle), _b(bounds), begin, end)


def ref_range_argmin(dag, bundle, objective, bounds, begin, end, threads) -> tuple[int, dict]:
    return _call(_reflib().loomref_range_argmin, _b(dag), _b(bundle), _b(objective), _b(bounds), begin, end,
                 threads)


def ref_plan(spec, bundle, lexicon) -> tuple[int, dict]:
    return _call(_reflib().loomref_plan, _b(spec), _b(bundle), _b(lexicon))
