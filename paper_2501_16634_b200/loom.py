"""Python binding of libloom_b200.so (include/loom_b200.h) for tests and the
bench.  It mirrors the reference's public search API (namespace loom,
optimizer.hpp / estimator.hpp): exhaustive_search(dag, library, objective,
bounds) returns the ConfigEstimate, errors surface as the reference's error
classes (errors.hpp:53-54) with the same messages.

There is no CPU fallback: loading fails loudly if the library is missing, and
device calls raise DeviceError without an sm_100 GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Any, Sequence

PKG = Path(__file__).resolve().parent
# LOOM_B200_LIB: an experiment build of the same library (build.py --variant)
LIB_PATH = Path(os.environ["LOOM_B200_LIB"]) if os.environ.get("LOOM_B200_LIB") else PKG / "libloom_b200.so"

LOOM_OK, LOOM_INFEASIBLE, LOOM_INVALID, LOOM_DEVICE_ERROR = 0, 1, 2, 3
CRITERIA = {"min_cost_dollars": 0, "min_energy": 1, "min_latency": 2, "max_quality": 3}


# ---- errors (errors.hpp) --------------------------------------------------
class LoomError(RuntimeError):
    code = "Error"
    category = 0

    def __init__(self, message: str, status: int = LOOM_INVALID):
        super().__init__(message)
        self.status = status


class SchemaError(LoomError):
    code, category = "SchemaError", 2


class ValidationError(LoomError):
    code, category = "ValidationError", 2


class CycleError(LoomError):
    code, category = "CycleError", 2


class DuplicateKeyError(LoomError):
    code, category = "DuplicateKeyError", 2


class DanglingReferenceError(LoomError):
    code, category = "DanglingReferenceError", 2


class UnknownCapabilityError(LoomError):
    code, category = "UnknownCapabilityError", 2


class InvalidConfigError(LoomError):
    code, category = "InvalidConfigError", 4


class NoFeasibleConfigError(LoomError):
    code, category = "NoFeasibleConfigError", 4


class DeviceError(LoomError):
    code, category = "DeviceError", 5


_ERRORS = {cls.code: cls for cls in (SchemaError, ValidationError, CycleError, DuplicateKeyError,
                                     DanglingReferenceError, UnknownCapabilityError, InvalidConfigError,
                                     NoFeasibleConfigError, DeviceError)}


def _raise(status: int, message: str):
    code = message.split(":", 1)[0].strip()
    cls = _ERRORS.get(code)
    if cls is None:
        cls = {LOOM_INFEASIBLE: NoFeasibleConfigError, LOOM_DEVICE_ERROR: DeviceError}.get(status,
                                                                                            InvalidConfigError)
    raise cls(message, status)


# ---- ABI structs ------------------------------------------------------------
class Problem(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_edges", C.c_int32), ("radix", C.POINTER(C.c_int32)),
                ("wall_us", C.POINTER(C.c_int64)), ("gpu_wh", C.POINTER(C.c_double)),
                ("cpu_wh", C.POINTER(C.c_double)), ("dollars", C.POINTER(C.c_double)),
                ("quality", C.POINTER(C.c_int32)), ("lexrank", C.POINTER(C.c_int32)),
                ("lex_weight", C.POINTER(C.c_uint64)), ("edge_from", C.POINTER(C.c_int32)),
                ("edge_to", C.POINTER(C.c_int32))]


class Objective(C.Structure):
    _fields_ = [("n_criteria", C.c_int32), ("criteria", C.c_int32 * 4), ("has_quality_floor", C.c_int32),
                ("quality_floor", C.c_int32), ("has_latency_slo", C.c_int32), ("reserved", C.c_int32),
                ("latency_slo_us", C.c_int64)]


class Winner(C.Structure):
    _fields_ = [("plan_index", C.c_uint64), ("lexkey", C.c_uint64), ("latency_us", C.c_int64),
                ("gpu_wh", C.c_double), ("cpu_wh", C.c_double), ("total_wh", C.c_double),
                ("dollars", C.c_double), ("quality", C.c_int32), ("found", C.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


assert C.sizeof(Winner) == 64


class Point(C.Structure):
    _fields_ = [("plan_index", C.c_uint64), ("dollars", C.c_double), ("gpu_wh", C.c_double),
                ("latency_us", C.c_int64), ("quality", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


assert C.sizeof(Point) == 40


class EstimateStreams(C.Structure):
    _fields_ = [("latency_us", C.c_void_p), ("gpu_wh", C.c_void_p), ("cpu_wh", C.c_void_p),
                ("total_wh", C.c_void_p), ("dollars", C.c_void_p), ("quality", C.c_void_p)]


# ConfigEstimate fields of a score stream and their element types
STREAM_FIELDS = {"latency_us": "int64", "gpu_wh": "float64", "cpu_wh": "float64", "total_wh": "float64",
                 "dollars": "float64", "quality": "int32"}


_lib = None


def lib() -> C.CDLL:
    """Load libloom_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2501_16634_b200.build`")
    L = C.CDLL(str(LIB_PATH))
    P, O, W = C.POINTER(Problem), C.POINTER(Objective), C.POINTER(Winner)
    vp = C.c_void_p
    sig = {
        "loom_abi_version": ([], C.c_int),
        "loom_last_error": ([], C.c_char_p),
        "loom_problem_total": ([P, C.POINTER(C.c_uint64)], C.c_int),
        "loom_evaluate_plan": ([P, C.c_uint64, W], C.c_int),
        "loom_winner_less": ([W, W, O], C.c_int),
        "loom_winner_reduce": ([W, C.c_int32, O, W], C.c_int),
        "loom_objective_parse": ([C.c_char_p, O], C.c_int),
        "loom_lower": ([C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(vp)], C.c_int),
        "loom_lowered_problem": ([vp], P),
        "loom_lower_batch": ([C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int32, C.c_int32, C.POINTER(vp),
                              C.POINTER(C.c_int32)], C.c_int),
        "loom_lowered_config_json": ([vp, C.c_uint64, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "loom_lowered_option_json": ([vp, C.c_int32, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
                                     C.c_int),
        "loom_lowered_destroy": ([vp], None),
        "loom_ctx_create": ([C.c_int32, vp, C.POINTER(vp)], C.c_int),
        "loom_ctx_destroy": ([vp], C.c_int),
        "loom_ctx_launch_count": ([vp], C.c_uint64),
        "loom_search_argmin": ([vp, P, O, C.c_uint64, C.c_uint64, W], C.c_int),
        "loom_search_argmin_algo": ([vp, P, O, C.c_uint64, C.c_uint64, C.c_int32, W], C.c_int),
        "loom_search_argmin_batch": ([vp, P, O, C.c_int32, W, C.POINTER(C.c_int32)], C.c_int),
        "loom_search_argmin_lowered": ([vp, C.POINTER(vp), C.c_int32, O, W, C.POINTER(C.c_int32)], C.c_int),
        "loom_exhaustive_search_batch": ([vp, C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int32, C.c_char_p,
                                          C.c_int32, W, C.POINTER(C.c_int32)], C.c_int),
        "loom_problem_upload": ([vp, P, O, C.POINTER(vp)], C.c_int),
        "loom_problem_release": ([vp], C.c_int),
        "loom_search_argmin_async": ([vp, vp, C.c_uint64, C.c_uint64], C.c_int),
        "loom_search_argmin_shard": ([vp, P, O, C.c_uint64, C.c_uint64, C.c_uint64, W], C.c_int),
        "loom_search_argmin_shard_async": ([vp, vp, C.c_uint64, C.c_uint64, C.c_uint64], C.c_int),
        "loom_search_argmin_algo_async": ([vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32], C.c_int),
        "loom_bnb_last_stats": ([C.POINTER(C.c_uint64)], C.c_int),
        "loom_bfs_trace": ([C.POINTER(C.c_uint64), C.c_int32], C.c_int),
        "loom_device_problem_bytes": ([vp], C.c_uint64),
        "loom_search_argmin_result": ([vp, vp, W], C.c_int),
        "loom_search_pareto": ([vp, P, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.c_uint64,
                                C.POINTER(C.c_uint64)], C.c_int),
        "loom_search_pareto_points": ([vp, P, C.c_uint64, C.c_uint64, C.POINTER(Point), C.c_uint64,
                                       C.POINTER(C.c_uint64)], C.c_int),
        "loom_pareto_filter_points": ([vp, C.POINTER(Point), C.c_uint64, C.POINTER(C.c_uint8)], C.c_int),
        "loom_estimate_range": ([vp, P, C.c_uint64, C.c_uint64, C.POINTER(EstimateStreams)], C.c_int),
        "loom_estimate_range_device": ([vp, P, C.c_uint64, C.c_uint64, C.POINTER(EstimateStreams)], C.c_int),
        "loom_estimate_plans": ([vp, P, C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(EstimateStreams)], C.c_int),
        "loom_greedy_seed": ([P, O, C.POINTER(C.c_int32)], C.c_int),
        "loom_latency_floor": ([P, vp, C.POINTER(C.c_int64)], C.c_int),
        "loom_search_greedy": ([vp, P, O, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, W], C.c_int),
        "loom_lowered_sweep_order": ([vp, C.POINTER(C.c_int32)], C.c_int),
        "loom_greedy_search_json": ([vp, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32, C.c_char_p,
                                     C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "loom_estimate_config_json": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                                       C.POINTER(C.c_size_t)], C.c_int),
        "loom_exhaustive_search_json": ([vp, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                         C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "loom_search_argmin_lowered_each": ([vp, C.POINTER(vp), C.c_int32, O, W, C.POINTER(C.c_int32)], C.c_int),
        "loom_ctx_stream": ([vp], vp),
        "loom_nccl_unique_id": ([C.POINTER(C.c_uint8)], C.c_int),
        "loom_group_create": ([C.c_uint64, C.POINTER(vp)], C.c_int),
        "loom_group_create_rank": ([C.c_int32, vp, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.POINTER(vp)],
                                   C.c_int),
        "loom_group_destroy": ([vp], C.c_int),
        "loom_group_world": ([vp], C.c_int32),
        "loom_group_local": ([vp], C.c_int32),
        "loom_group_rank": ([vp], C.c_int32),
        "loom_group_ctx": ([vp, C.c_int32], vp),
        "loom_shard_range": ([C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)], C.c_int),
        "loom_group_search_argmin": ([vp, P, O, C.c_uint64, C.c_uint64, W], C.c_int),
        "loom_group_search_pareto_points": ([vp, P, C.c_uint64, C.c_uint64, C.POINTER(Point), C.c_uint64,
                                             C.POINTER(C.c_uint64)], C.c_int),
        "loom_group_search_argmin_batch": ([vp, P, O, C.c_int32, W, C.POINTER(C.c_int32)], C.c_int),
        "loom_group_exhaustive_search_json": ([vp, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                               C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Function names declared in include/loom_b200.h."""
    import re
    text = (PKG.parent / "include" / "loom_b200.h").read_text()
    return sorted(set(re.findall(r"\b(loom_[a-z0-9_]+)\s*\(", text)))


def last_error() -> str:
    return (lib().loom_last_error() or b"").decode()


def _check(rc: int) -> None:
    if rc != LOOM_OK:
        _raise(rc, last_error())


def _text(x: Any) -> bytes:
    """JSON text for the C ABI: bytes pass through, str is encoded, anything
    else is serialised."""
    if isinstance(x, (bytes, bytearray)):
        return bytes(x)
    return (x if isinstance(x, str) else json.dumps(x)).encode()


_BYTES_DATA_OFFSET: int | None = None


def _text_array(items: Sequence[Any]):
    """A char*[] over the JSON texts of `items` -> (pointer, keep-alive).
    Large batches of bytes build it from the objects' addresses in one numpy
    pass (10,000 ctypes conversions cost milliseconds): the text of a bytes
    object sits at a fixed offset from its address, measured once here."""
    global _BYTES_DATA_OFFSET
    texts = items if all(type(d) is bytes for d in items) else [_text(d) for d in items]
    n = len(texts)
    if n < 256:
        arr = (C.c_char_p * max(1, n))(*texts)
        return arr, (texts, arr)
    import numpy as np
    if _BYTES_DATA_OFFSET is None:
        probe = b"loom"
        _BYTES_DATA_OFFSET = C.cast(C.c_char_p(probe), C.c_void_p).value - id(probe)
    ptrs = np.fromiter(map(id, texts), dtype=np.uint64, count=n)
    ptrs += np.uint64(_BYTES_DATA_OFFSET)
    return ptrs.ctypes.data_as(C.POINTER(C.c_char_p)), (texts, ptrs)


def objective(obj: dict | str) -> Objective:
    """Objective JSON / token -> loom_objective (workflow.hpp:91-106)."""
    if isinstance(obj, str) and not obj.lstrip().startswith("{"):
        obj = {"constraint": obj}
    o = Objective()
    _check(lib().loom_objective_parse(_text(obj), C.byref(o)))
    return o


# ---- lowering -----------------------------------------------------------
class Lowered:
    """Reference-format JSON lowered to the flat plan space (host-side C++)."""

    def __init__(self, dag: Any, library: Any, bounds: Any, _handle: C.c_void_p | None = None):
        if _handle is None:
            h = C.c_void_p()
            _check(lib().loom_lower(_text(dag), _text(library), _text(bounds), C.byref(h)))
        else:
            h = _handle
        self._h = h
        self._owned = True
        self.problem: Problem = lib().loom_lowered_problem(h).contents

    def close(self) -> None:
        if self._h and self._owned:
            lib().loom_lowered_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def radix(self) -> list[int]:
        return [self.problem.radix[i] for i in range(self.problem.n_nodes)]

    @property
    def n_options(self) -> int:
        return sum(self.radix)

    @property
    def total(self) -> int:
        t = C.c_uint64(0)
        _check(lib().loom_problem_total(C.byref(self.problem), C.byref(t)))
        return t.value

    def table(self, name: str) -> list:
        arr = getattr(self.problem, name)
        n = self.problem.n_nodes if name == "lex_weight" else self.n_options
        return [arr[i] for i in range(n)]

    def _json(self, fn, *args) -> dict:
        need = C.c_size_t(0)
        fn(self._h, *args, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        _check(fn(self._h, *args, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())

    def config(self, plan_index: int) -> dict:
        return self._json(lib().loom_lowered_config_json, C.c_uint64(plan_index))

    def option(self, node: int, option: int) -> dict:
        return self._json(lib().loom_lowered_option_json, node, option)

    def sweep_order(self) -> list[int]:
        out = (C.c_int32 * max(1, self.problem.n_nodes))()
        _check(lib().loom_lowered_sweep_order(self._h, out))
        return list(out)[: self.problem.n_nodes]

    def evaluate(self, plan_index: int) -> dict:
        w = Winner()
        _check(lib().loom_evaluate_plan(C.byref(self.problem), plan_index, C.byref(w)))
        return w.as_dict()


def lower_batch(dags: Sequence[Any], library: Any, bounds: Any, threads: int = 0) -> list[Lowered]:
    """Lower many DAGs against one library bundle (parsed once, multi-threaded)."""
    n = len(dags)
    arr, keep = _text_array(dags)
    out = (C.c_void_p * max(1, n))()
    st = (C.c_int32 * max(1, n))()
    _check(lib().loom_lower_batch(_text(library), _text(bounds), arr, n, threads, out, st))
    del keep
    res = []
    for i in range(n):
        if st[i] != LOOM_OK:
            _raise(st[i], f"job {i}: " + last_error())
        res.append(Lowered(None, None, None, _handle=C.c_void_p(out[i])))
    return res


class LoweredBatch:
    """Many lowered DAGs as one array of C handles (config 4): no per-job
    Python objects on the batch path.  batch[i] is a non-owning view."""

    def __init__(self, dags: Sequence[Any], library: Any, bounds: Any, threads: int = 0):
        n = len(dags)
        self.n = n
        arr, keep = _text_array(dags)
        self.handles = (C.c_void_p * max(1, n))()
        self.status = (C.c_int32 * max(1, n))()
        _check(lib().loom_lower_batch(_text(library), _text(bounds), arr, n, threads, self.handles, self.status))
        del keep

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int) -> "Lowered":
        if self.status[i] != LOOM_OK:
            _raise(self.status[i], f"job {i} was not lowered")
        v = Lowered.__new__(Lowered)
        v._h = C.c_void_p(self.handles[i])
        v._owned = False  # the batch destroys its handles
        v.problem = lib().loom_lowered_problem(v._h).contents
        return v

    def close(self) -> None:
        if self.handles is not None:
            for i in range(self.n):
                if self.handles[i]:
                    lib().loom_lowered_destroy(self.handles[i])
            self.handles = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BatchResult:
    """Per-job winners of a multi-tenant batch, kept in the C arrays the
    library filled (decoded to dicts only on request)."""

    def __init__(self, n: int):
        self.n = n
        self.winners = (Winner * max(1, n))()
        self.status = (C.c_int32 * max(1, n))()

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int) -> tuple[int, dict]:
        return self.status[i], self.winners[i].as_dict()

    def feasible(self) -> int:
        return sum(1 for i in range(self.n) if self.status[i] == LOOM_OK)


def search_lowered_batch(ctx: "Context", batch: LoweredBatch, obj: Objective) -> BatchResult:
    """Per-job argmin of every lowered DAG of the batch under one objective."""
    res = BatchResult(batch.n)
    _check(lib().loom_search_argmin_lowered(ctx.handle, batch.handles, batch.n, C.byref(obj), res.winners,
                                            res.status))
    return res


def exhaustive_search_batch(dags: Sequence[Any], library: Any, objective: Any, bounds: Any, *,
                            ctx: "Context", threads: int = 0) -> BatchResult:
    """The multi-tenant call on reference-format JSON: exhaustive_search
    (optimizer.hpp:173-188) for every DAG against one library, objective and
    bounds, lowered on host threads and searched in one batched launch.
    `objective` may also be a list with one objective per DAG."""
    n = len(dags)
    arr, keep = _text_array(dags)
    res = BatchResult(n)
    _check(lib().loom_exhaustive_search_batch(ctx.handle, _text(library), _text(bounds), arr, n, _text(objective),
                                              threads, res.winners, res.status))
    del keep
    return res


# ---- device context --------------------------------------------------------
class Context:
    def __init__(self, device: int = 0, stream: int | None = None):
        """stream: a cudaStream_t handle to launch on; None -> the ctx owns a
        stream; 0 (torch's legacy default stream) -> cudaStreamLegacy."""
        h = C.c_void_p()
        handle = None if stream is None else C.c_void_p(stream if stream else 1)
        _check(lib().loom_ctx_create(device, handle, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def launches(self) -> int:
        return lib().loom_ctx_launch_count(self._h)

    def close(self) -> None:
        if self._h:
            lib().loom_ctx_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def search_argmin(ctx: Context, problem: Problem, obj: Objective, begin: int = 0, end: int | None = None,
                  algo: int = 0) -> dict:
    w = Winner()
    end = (1 << 64) - 1 if end is None else end
    _check(lib().loom_search_argmin_algo(ctx.handle, C.byref(problem), C.byref(obj), begin, end, algo, C.byref(w)))
    return w.as_dict()


INCUMBENT_GREEDY = (1 << 64) - 1
NO_INCUMBENT = (1 << 64) - 2
ALGO_AUTO, ALGO_FULL, ALGO_SWEEP = 0, 1, 2


def bfs_trace() -> dict:
    """Per-level timeline of the last frontier search: microseconds per level,
    parents expanded, and whether the level ran redundantly in every CTA."""
    buf = (C.c_uint64 * 68)()
    _check(lib().loom_bfs_trace(buf, 68))
    t0, levels, prev = buf[0], [], buf[0]
    for d in range(33):
        end, par = buf[2 * d + 2], buf[2 * d + 3]
        if not end:
            break
        levels.append({"us": (end - prev) / 1e3, "parents": par & ((1 << 63) - 1), "redundant": bool(par >> 63)})
        prev = end
    return {"total_us": (buf[1] - t0) / 1e3 if buf[1] else None, "levels": levels}


def latency_floor(problem: Problem, obj: Objective | None = None) -> int:
    """Smallest latency of any plan (loom_latency_floor): the critical path
    with every node at its fastest option meeting the quality floor."""
    out = C.c_int64()
    _check(lib().loom_latency_floor(C.byref(problem), C.byref(obj) if obj is not None else None, C.byref(out)))
    return out.value


def bnb_last_stats() -> dict:
    """Evidence of the last default (branch-and-bound) search: subtree bounds +
    leaves evaluated, whether the depth-first search had to take over from the
    frontier search and whether the every-plan sweep finished it ("aborted"),
    the largest frontier, and the leaves (plans evaluated exactly)."""
    buf = (C.c_uint64 * 6)()
    _check(lib().loom_bnb_last_stats(buf))
    return {"child_evaluations": buf[0], "depth_first": bool(buf[1] & 1), "aborted": bool(buf[1] & 2),
            "max_frontier": buf[2], "ctas": buf[3], "leaves": buf[4], "depth_first_evaluations": buf[5]}


def search_argmin_shard(ctx: Context, problem: Problem, obj: Objective, begin: int, end: int,
                        incumbent: int = INCUMBENT_GREEDY) -> dict:
    """argmin of [begin, end) u {incumbent} (a multi-GPU shard search); the
    incumbent defaults to the greedy seed.  The result may be the incumbent."""
    w = Winner()
    _check(lib().loom_search_argmin_shard(ctx.handle, C.byref(problem), C.byref(obj), begin, end, incumbent,
                                          C.byref(w)))
    return w.as_dict()


def search_argmin_batch(ctx: Context, problems: Sequence[Problem], objectives: Sequence[Objective]
                        ) -> list[tuple[int, dict]]:
    n = len(problems)
    P = (Problem * n)(*problems)
    O = (Objective * n)(*objectives)
    W = (Winner * n)()
    S = (C.c_int32 * n)()
    _check(lib().loom_search_argmin_batch(ctx.handle, P, O, n, W, S))
    return [(S[i], W[i].as_dict()) for i in range(n)]


def winner_reduce(winners: Sequence[Winner], obj: Objective) -> dict:
    n = len(winners)
    arr = (Winner * max(1, n))(*winners)
    out = Winner()
    _check(lib().loom_winner_reduce(arr, n, C.byref(obj), C.byref(out)))
    return out.as_dict()


def winner_from_dict(d: dict) -> Winner:
    w = Winner()
    for k, _ in Winner._fields_:
        setattr(w, k, d[k])
    return w


class DeviceProblem:
    """A problem resident in HBM for repeated searches (bench 'value' path)."""

    def __init__(self, ctx: Context, problem: Problem, obj: Objective):
        h = C.c_void_p()
        _check(lib().loom_problem_upload(ctx.handle, C.byref(problem), C.byref(obj), C.byref(h)))
        self._h, self.ctx = h, ctx

    def search_async(self, begin: int = 0, end: int | None = None) -> None:
        end = (1 << 64) - 1 if end is None else end
        _check(lib().loom_search_argmin_async(self.ctx.handle, self._h, begin, end))

    def search_algo_async(self, begin: int = 0, end: int | None = None, algo: int = ALGO_AUTO,
                          incumbent: int = NO_INCUMBENT) -> None:
        """Enqueue a search with a chosen algorithm (ALGO_AUTO: branch and bound
        with the sweep as fallback; ALGO_FULL; ALGO_SWEEP: every plan tested)."""
        end = (1 << 64) - 1 if end is None else end
        _check(lib().loom_search_argmin_algo_async(self.ctx.handle, self._h, begin, end, incumbent, algo))

    def search_shard_async(self, begin: int, end: int, incumbent: int = INCUMBENT_GREEDY) -> None:
        """Enqueue loom_search_argmin_shard_async (argmin of [begin, end) u {incumbent})."""
        _check(lib().loom_search_argmin_shard_async(self.ctx.handle, self._h, begin, end, incumbent))

    @property
    def image_bytes(self) -> int:
        return lib().loom_device_problem_bytes(self._h)

    def result(self) -> dict:
        w = Winner()
        _check(lib().loom_search_argmin_result(self.ctx.handle, self._h, C.byref(w)))
        return w.as_dict()

    def close(self) -> None:
        if self._h:
            lib().loom_problem_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def search_pareto(ctx: Context, problem: Problem, begin: int = 0, end: int | None = None) -> list[int]:
    end = (1 << 64) - 1 if end is None else end
    cnt = C.c_uint64(0)
    _check(lib().loom_search_pareto(ctx.handle, C.byref(problem), begin, end, None, 0, C.byref(cnt)))
    buf = (C.c_uint64 * max(1, cnt.value))()
    _check(lib().loom_search_pareto(ctx.handle, C.byref(problem), begin, end, buf, cnt.value, C.byref(cnt)))
    return [buf[i] for i in range(cnt.value)]


def search_pareto_points(ctx: Context, problem: Problem, begin: int = 0, end: int | None = None) -> list[dict]:
    """Frontier of plans [begin, end) under pareto_filter's dominance, ascending index."""
    end = (1 << 64) - 1 if end is None else end
    cnt = C.c_uint64(0)
    _check(lib().loom_search_pareto_points(ctx.handle, C.byref(problem), begin, end, None, 0, C.byref(cnt)))
    buf = (Point * max(1, cnt.value))()
    _check(lib().loom_search_pareto_points(ctx.handle, C.byref(problem), begin, end, buf, cnt.value, C.byref(cnt)))
    return [buf[i].as_dict() for i in range(cnt.value)]


def pareto_filter_points(ctx: Context, points: Sequence[dict]) -> list[bool]:
    """pareto_filter (optimizer.hpp:153-171) on arbitrary points, on the device."""
    n = len(points)
    arr = (Point * max(1, n))()
    for i, p in enumerate(points):
        for k in ("plan_index", "dollars", "gpu_wh", "latency_us", "quality"):
            setattr(arr[i], k, p[k])
    keep = (C.c_uint8 * max(1, n))()
    _check(lib().loom_pareto_filter_points(ctx.handle, arr, n, keep))
    return [bool(keep[i]) for i in range(n)]


# ---- the drop-in call ----------------------------------------------------
_default_ctx: Context | None = None


# ---- per-plan estimate streams (estimator.hpp:43-78) --------------------------
def _streams_struct(arrays: dict, ptr) -> EstimateStreams:
    st = EstimateStreams()
    for k, a in arrays.items():
        if k not in STREAM_FIELDS:
            raise ValueError(f"unknown estimate stream {k!r}")
        setattr(st, k, ptr(a))
    return st


def estimate_range(ctx: Context, problem: Problem, begin: int, end: int,
                   fields: Sequence[str] = tuple(STREAM_FIELDS)) -> dict:
    """estimate(p) for every plan p in [begin, end) (ConfigEnumerator order),
    as numpy arrays keyed by ConfigEstimate field.  Host arrays."""
    import numpy as np
    n = max(0, end - begin)
    out = {k: np.empty(n, dtype=STREAM_FIELDS[k]) for k in fields}
    st = _streams_struct(out, lambda a: a.ctypes.data)
    _check(lib().loom_estimate_range(ctx.handle, C.byref(problem), begin, end, C.byref(st)))
    return out


def estimate_range_device(ctx: Context, problem: Problem, begin: int, end: int, tensors: dict) -> None:
    """Same into device tensors (torch, on the ctx's device), enqueued on the
    ctx stream without synchronising."""
    st = _streams_struct(tensors, lambda t: t.data_ptr())
    _check(lib().loom_estimate_range_device(ctx.handle, C.byref(problem), begin, end, C.byref(st)))


def estimate_range_host(ctx: Context, problem: Problem, begin: int, end: int, tensors: dict) -> None:
    """Same into caller-owned host tensors (e.g. pinned torch CPU tensors);
    returns when they are filled."""
    st = _streams_struct(tensors, lambda t: t.data_ptr())
    _check(lib().loom_estimate_range(ctx.handle, C.byref(problem), begin, end, C.byref(st)))


def estimate_plans(ctx: Context, problem: Problem, indices: Sequence[int],
                   fields: Sequence[str] = tuple(STREAM_FIELDS)) -> dict:
    """Batched estimate of arbitrary plan indices (element i = plan indices[i])."""
    import numpy as np
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    out = {k: np.empty(len(idx), dtype=STREAM_FIELDS[k]) for k in fields}
    st = _streams_struct(out, lambda a: a.ctypes.data)
    _check(lib().loom_estimate_plans(ctx.handle, C.byref(problem), idx.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     len(idx), C.byref(st)))
    return out


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---- multi-GPU groups (loom_group_*; NCCL owned by the library) -------------
NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """A fresh NCCL id for loom_group_create_rank (made by rank 0, shared by the caller)."""
    buf = (C.c_uint8 * NCCL_ID_BYTES)()
    _check(lib().loom_nccl_unique_id(buf))
    return bytes(buf)


def shard_range(begin: int, end: int, rank: int, world: int) -> tuple[int, int]:
    """The library's contiguous shard of [begin, end) for rank of world (host)."""
    b, e = C.c_uint64(), C.c_uint64()
    _check(lib().loom_shard_range(begin, end, rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


class BorrowedContext:
    """A loom_ctx owned by someone else (a group member): usable wherever a
    Context is, never destroyed through this handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def launches(self) -> int:
        return lib().loom_ctx_launch_count(self._h)


class Group:
    """A set of GPUs searching one plan space together (loom_group_*): the
    plan space is sharded by contiguous index ranges inside the library and
    the per-rank results are exchanged with ncclAllGather; every rank gets the
    same answer.  Group(device_mask=m): this process drives every GPU in m;
    Group(device=d, rank=r, world=w, nccl_id=id): one process per GPU."""

    def __init__(self, device_mask: int | None = None, *, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, stream: int | None = None):
        h = C.c_void_p()
        if device_mask is not None:
            _check(lib().loom_group_create(device_mask, C.byref(h)))
        else:
            idb = (C.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(nccl_id)
            handle = None if stream is None else C.c_void_p(stream if stream else 1)
            _check(lib().loom_group_create_rank(device, handle, idb, rank, world, C.byref(h)))
        self._h = h

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    world = property(lambda self: lib().loom_group_world(self._h))
    local = property(lambda self: lib().loom_group_local(self._h))
    rank = property(lambda self: lib().loom_group_rank(self._h))

    def launches(self) -> int:
        return sum(lib().loom_ctx_launch_count(lib().loom_group_ctx(self._h, i)) for i in range(self.local))

    def context(self, i: int = 0) -> "BorrowedContext":
        """Member i's device context (owned by the group)."""
        return BorrowedContext(lib().loom_group_ctx(self._h, i))

    def close(self) -> None:
        if self._h:
            lib().loom_group_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search_argmin(self, problem: Problem, obj: Objective, begin: int = 0, end: int | None = None) -> dict:
        w = Winner()
        end = (1 << 64) - 1 if end is None else end
        _check(lib().loom_group_search_argmin(self._h, C.byref(problem), C.byref(obj), begin, end, C.byref(w)))
        return w.as_dict()

    def search_pareto_points(self, problem: Problem, begin: int = 0, end: int | None = None) -> list[dict]:
        end = (1 << 64) - 1 if end is None else end
        cnt = C.c_uint64(0)
        _check(lib().loom_group_search_pareto_points(self._h, C.byref(problem), begin, end, None, 0, C.byref(cnt)))
        buf = (Point * max(1, cnt.value))()
        _check(lib().loom_group_search_pareto_points(self._h, C.byref(problem), begin, end, buf, cnt.value,
                                                      C.byref(cnt)))
        return [buf[i].as_dict() for i in range(cnt.value)]

    def search_argmin_batch(self, problems: Sequence[Problem], objectives: Sequence[Objective]
                            ) -> list[tuple[int, dict]]:
        n = len(problems)
        P = (Problem * n)(*problems)
        O = (Objective * n)(*objectives)
        W = (Winner * n)()
        S = (C.c_int32 * n)()
        _check(lib().loom_group_search_argmin_batch(self._h, P, O, n, W, S))
        return [(S[i], W[i].as_dict()) for i in range(n)]

    def exhaustive_search(self, dag: Any, library: Any, objective_: Any, bounds: Any) -> dict:
        """loom_group_exhaustive_search_json: the drop-in call over the group."""
        return _json_call(lib().loom_group_exhaustive_search_json, self._h, dag, library, objective_, bounds)


def _json_call(fn, handle, dag: Any, library: Any, objective_: Any, bounds: Any) -> dict:
    if isinstance(objective_, str) and not objective_.lstrip().startswith("{"):
        objective_ = {"constraint": objective_}
    need = C.c_size_t(0)
    cap = 1 << 14  # grown on demand (the needed size comes back)
    buf = C.create_string_buffer(cap)
    rc = fn(handle, _text(dag), _text(library), _text(objective_), _text(bounds), buf, cap, C.byref(need))
    if rc != LOOM_OK and need.value > cap:
        buf = C.create_string_buffer(need.value)
        rc = fn(handle, _text(dag), _text(library), _text(objective_), _text(bounds), buf, need.value,
                C.byref(need))
    out = json.loads(buf.value.decode())
    if rc != LOOM_OK:
        _raise(rc, out.get("message", last_error()))
    return out


def exhaustive_search(dag: Any, library: Any, objective_: Any, bounds: Any, ctx: Context | None = None) -> dict:
    """loom::exhaustive_search (optimizer.hpp:173-188) on reference-format JSON;
    returns the ConfigEstimate as a dict (identifier, config, latency_us,
    gpu_wh, cpu_wh, total_wh, dollars, quality, plan_index, plans)."""
    ctx = ctx or default_context()
    if isinstance(objective_, str) and not objective_.lstrip().startswith("{"):
        objective_ = {"constraint": objective_}
    need = C.c_size_t(0)
    cap = 1 << 14  # grown on demand (the needed size comes back)
    buf = C.create_string_buffer(cap)
    rc = lib().loom_exhaustive_search_json(ctx.handle, _text(dag), _text(library), _text(objective_),
                                           _text(bounds), buf, cap, C.byref(need))
    if rc != LOOM_OK and need.value > cap:
        buf = C.create_string_buffer(need.value)
        rc = lib().loom_exhaustive_search_json(ctx.handle, _text(dag), _text(library), _text(objective_),
                                               _text(bounds), buf, need.value, C.byref(need))
    out = json.loads(buf.value.decode())
    if rc != LOOM_OK:
        _raise(rc, out.get("message", last_error()))
    return out


def estimate_config(dag: Any, library: Any, config: Any) -> dict:
    """The --pin path (loom_main.cpp:125-146): parse_config_point
    (config.hpp:66-117) + estimate (estimator.hpp:43-78) of one config point on
    the host; the ConfigEstimate as a dict (no plan_index)."""
    need = C.c_size_t(0)
    cap = 1 << 14  # grown on demand (the needed size comes back)
    buf = C.create_string_buffer(cap)
    rc = lib().loom_estimate_config_json(_text(dag), _text(library), _text(config), buf, cap, C.byref(need))
    if rc != LOOM_OK and need.value > cap:
        buf = C.create_string_buffer(need.value)
        rc = lib().loom_estimate_config_json(_text(dag), _text(library), _text(config), buf, need.value,
                                             C.byref(need))
    out = json.loads(buf.value.decode())
    if rc != LOOM_OK:
        _raise(rc, out.get("message", last_error()))
    return out


def greedy_search(dag: Any, library: Any, objective_: Any, bounds: Any, ctx: Context | None = None,
                  max_sweeps: int = 10) -> dict:
    """loom::greedy_search (optimizer.hpp:227-291) on reference-format JSON."""
    ctx = ctx or default_context()
    if isinstance(objective_, str) and not objective_.lstrip().startswith("{"):
        objective_ = {"constraint": objective_}
    need = C.c_size_t(0)
    cap = 1 << 14  # grown on demand (the needed size comes back)
    buf = C.create_string_buffer(cap)
    rc = lib().loom_greedy_search_json(ctx.handle, _text(dag), _text(library), _text(objective_), _text(bounds),
                                       max_sweeps, buf, cap, C.byref(need))
    out = json.loads(buf.value.decode())
    if rc != LOOM_OK:
        _raise(rc, out.get("message", last_error()))
    return out


def search_greedy(ctx: Context, problem: Problem, obj: Objective, sweep_order: Sequence[int] | None = None,
                  seed: Sequence[int] | None = None, max_sweeps: int = 10) -> dict:
    n = problem.n_nodes
    so = (C.c_int32 * n)(*sweep_order) if sweep_order is not None else None
    sd = (C.c_int32 * n)(*seed) if seed is not None else None
    w = Winner()
    _check(lib().loom_search_greedy(ctx.handle, C.byref(problem), C.byref(obj), so, sd, max_sweeps, C.byref(w)))
    return w.as_dict()


@dataclass
class SearchBounds:
    max_fanout: int = 4
    max_paths: int = 2
    sku_pool_cap: dict | None = None
    sku_total_cap: dict | None = None

    def to_json(self) -> dict:
        return {"max_fanout": self.max_fanout, "max_paths": self.max_paths,
                "sku_pool_cap": self.sku_pool_cap or {}, "sku_total_cap": self.sku_total_cap or {}}
