"""ORACLE TEST INFRASTRUCTURE -- NOT PRODUCT CODE.

Pure-Python restatement of the reference's per-node lowering, read from the
reference's own JSON formats (library bundle agent_library.hpp:327-344,
dag.json workflow.hpp:303-363).  Small loops only (once per node); the per-
plan work is in flat_oracle.c.  Only tests/, smoke() and bench.py's
cpu_baseline / reference legs may import this module, as the checker.

Function  <- reference (paths under /root/reference/proj/include/loom/)
  llround, to_micros      time.hpp:15-17 (std::llround: half away from zero)
  chunk_capacity          chunking.hpp:26-29
  split_task              chunking.hpp:17-24
  water_fill_split        chunking.hpp:35-58
  plan_node_execution     chunking.hpp:85-184
  placement_fits          optimizer.hpp:31-43
  node_options            optimizer.hpp:51-107
  implementations_for     agent_library.hpp:273-289
  profiles_for            agent_library.hpp:291-297
  node_quality            estimator.hpp:32-37
  identifier token        config.hpp:49-61
  topological_order       workflow.hpp:467-498
  objective_from_token    workflow.hpp:91-106
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field


def llround(x: float) -> int:
    t = math.trunc(x)
    f = x - t  # exact for binary64
    if f >= 0.5:
        t += 1
    elif f <= -0.5:
        t -= 1
    return int(t)


def to_micros(seconds: float) -> int:
    return llround(seconds * 1e6)


def to_seconds(us: int) -> float:
    return float(us) / 1e6


def chunk_capacity(work: float, min_chunk: float) -> int:
    if min_chunk <= 0:
        return 1
    return max(1, int(math.floor(work / min_chunk)))


def split_task(work: float, fan_out: int, min_chunk: float) -> list[float]:
    count = 1
    if fan_out > 1 and min_chunk > 0:
        capacity = int(math.floor(work / min_chunk))
        count = max(1, min(fan_out, capacity))
    return [work / count] * count


def water_fill_split(work: float, min_chunk: float, speeds: list[float]) -> list[float]:
    quanta = chunk_capacity(work, min_chunk)
    quantum = work / quanta
    completion = [0.0] * len(speeds)
    counts = [0] * len(speeds)
    for _ in range(quanta):
        best = 0
        best_time = completion[0] + quantum / speeds[0]
        for w in range(1, len(speeds)):
            t = completion[w] + quantum / speeds[w]
            if t < best_time:
                best, best_time = w, t
        completion[best] = best_time
        counts[best] += 1
    return [counts[w] * quantum for w in range(len(speeds))]


@dataclass
class Library:
    skus: dict            # id -> dict(class, busy, rate)
    capabilities: set
    impls: dict           # name -> dict(capability, quality, classes:set)
    profiles: dict        # (impl, sku, units) -> dict(throughput, setup)

    @staticmethod
    def from_bundle(b: dict) -> "Library":
        skus = {s["id"]: {"class": s["class"], "busy": float(s["busy_watts_per_unit"]),
                          "rate": float(s["dollars_per_unit_hour"])} for s in b.get("skus", [])}
        caps = {a["capability"] for a in b.get("agents", [])}
        impls = {i["name"]: {"capability": i["capability"], "quality": int(i["quality"]),
                             "classes": set(i["supported_classes"])} for i in b.get("implementations", [])}
        profs = {}
        for p in b.get("profiles", []):
            profs[(p["implementation"], p["sku"], int(p["units"]))] = {
                "throughput": float(p["throughput"]), "setup": float(p.get("setup_seconds", 0.0))}
        return Library(skus, caps, impls, profs)

    def implementations_for(self, capability: str) -> list[str]:
        if capability not in self.capabilities:
            raise KeyError(f"UnknownCapabilityError: capability '{capability}' is not registered")
        names = [n for n in sorted(self.impls) if self.impls[n]["capability"] == capability]
        return sorted(names, key=lambda n: (-self.impls[n]["quality"], n))

    def profiles_for(self, impl: str) -> list[tuple]:
        # std::map order over (implementation, sku, units); strings compare bytewise
        return sorted((k for k in self.profiles if k[0] == impl),
                      key=lambda k: (k[0].encode(), k[1].encode(), k[2]))


@dataclass
class Bounds:
    max_fanout: int = 4
    max_paths: int = 2
    sku_pool_cap: dict = field(default_factory=dict)
    sku_total_cap: dict = field(default_factory=dict)

    @staticmethod
    def from_json(j: dict) -> "Bounds":
        return Bounds(int(j.get("max_fanout", 4)), int(j.get("max_paths", 2)),
                      dict(j.get("sku_pool_cap", {})), dict(j.get("sku_total_cap", {})))


def placement_fits(b: Bounds, sku: str, units: int, total_units: int) -> bool:
    if b.sku_pool_cap:
        if sku not in b.sku_pool_cap or units > b.sku_pool_cap[sku]:
            return False
    if b.sku_total_cap:
        if sku not in b.sku_total_cap or total_units > b.sku_total_cap[sku]:
            return False
    return True


def node_options(node: dict, lib: Library, b: Bounds) -> list[dict]:
    opts = []
    max_paths = max(1, b.max_paths) if node.get("multi_path", False) else 1
    work, min_chunk = float(node["work_units"]), float(node.get("min_chunk", 0.0))
    fan_cap = min(b.max_fanout, chunk_capacity(work, min_chunk)) if node["splittable"] else 1
    for impl in lib.implementations_for(node["capability"]):
        classes = lib.impls[impl]["classes"]
        profiles = [k for k in lib.profiles_for(impl) if lib.skus[k[1]]["class"] in classes]
        for (_, sku, units) in profiles:
            for workers in range(1, max(1, fan_cap) + 1):
                if not placement_fits(b, sku, units, units * workers):
                    continue
                for paths in range(1, max_paths + 1):
                    opts.append({"implementation": impl, "placements": [(sku, units, workers)], "path_count": paths})
        if node["splittable"] and b.max_fanout >= 2:
            for gk in profiles:
                if lib.skus[gk[1]]["class"] != "gpu":
                    continue
                for ck in profiles:
                    if lib.skus[ck[1]]["class"] != "cpu":
                        continue
                    if not placement_fits(b, gk[1], gk[2], gk[2]) or not placement_fits(b, ck[1], ck[2], ck[2]):
                        continue
                    split = water_fill_split(work, min_chunk, [lib.profiles[gk]["throughput"],
                                                               lib.profiles[ck]["throughput"]])
                    if work > 0 and (split[0] <= 0 or split[1] <= 0):
                        continue
                    for paths in range(1, max_paths + 1):
                        opts.append({"implementation": impl,
                                     "placements": [(gk[1], gk[2], 1), (ck[1], ck[2], 1)],
                                     "path_count": paths})
    return opts


def plan_node_execution(node: dict, opt: dict, lib: Library) -> dict:
    impl = opt["implementation"]
    resolved = []
    for (sku, units, workers) in opt["placements"]:
        prof = lib.profiles[(impl, sku, units)]
        resolved += [(sku, units, prof)] * workers
    work, min_chunk = float(node["work_units"]), float(node.get("min_chunk", 0.0))
    total_workers = sum(p[2] for p in opt["placements"])
    if len(resolved) == 1:
        chunks = [work]
    elif len(opt["placements"]) <= 1:
        chunks = split_task(work, total_workers, min_chunk)
    else:
        chunks = water_fill_split(work, min_chunk, [r[2]["throughput"] for r in resolved])
    wall, gpu, cpu, dol = 0, 0.0, 0.0, 0.0
    for (sku, units, prof), chunk in zip(resolved, chunks):
        setup = to_micros(prof["setup"])
        run = to_micros(chunk / prof["throughput"])
        dur = setup + run
        wall = max(wall, dur)
        hours = to_seconds(dur) / 3600.0
        s = lib.skus[sku]
        wh = units * s["busy"] * hours
        if s["class"] == "gpu":
            gpu += wh
        else:
            cpu += wh
        dol += units * s["rate"] * hours
    return {"wall_us": wall, "gpu_wh": gpu, "cpu_wh": cpu, "dollars": dol}


def node_quality(node: dict, impl_quality: int, path_count: int) -> int:
    q = impl_quality + (path_count - 1)
    if node.get("path_quality_ceiling") is not None:
        q = min(q, int(node["path_quality_ceiling"]))
    return q


def token(node_id: str, opt: dict) -> str:
    placements = "+".join(f"{s}:{u}x{w}" for (s, u, w) in opt["placements"])
    return f"{node_id}={opt['implementation']}[{placements}]p{opt['path_count']};"


def topological_order(dag: dict) -> list[str]:
    ids = [n["id"] for n in dag["nodes"]]
    indeg = {i: 0 for i in ids}
    adj: dict[str, list[str]] = {}
    for e in dag["edges"]:
        adj.setdefault(e["from"], []).append(e["to"])
        indeg[e["to"]] += 1
    ready = [i for i in sorted(indeg) if indeg[i] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        i = heapq.heappop(ready)
        order.append(i)
        for nxt in adj.get(i, []):
            indeg[nxt] -= 1
            if indeg[nxt] == 0:
                heapq.heappush(ready, nxt)
    if len(order) != len(ids):
        raise ValueError("CycleError: dag has a cycle")
    return order


CRITERIA = {"min_cost_dollars": 0, "min_energy": 1, "min_latency": 2, "max_quality": 3}
TOKENS = {"MIN_COST": ["min_energy", "min_latency"],
          "MIN_DOLLARS": ["min_cost_dollars", "min_latency"],
          "MIN_LATENCY": ["min_latency", "min_energy"],
          "MAX_QUALITY": ["max_quality", "min_energy", "min_latency"]}


def objective_criteria(objective: dict) -> list[str]:
    if "criteria" in objective:
        return list(objective["criteria"])
    return TOKENS[objective["constraint"]]


@dataclass
class Lowered:
    node_ids: list
    options: list          # per node: list of option dicts
    plans: list            # per node: list of plan_node_execution dicts
    quality: list          # per node: list of node_quality
    tokens: list           # per node: list of identifier substrings
    topo: list             # node indices, reference topological_order
    edges: list            # (from_idx, to_idx)

    @property
    def radix(self) -> list[int]:
        return [len(o) for o in self.options]

    @property
    def total(self) -> int:
        t = 1 if self.options else 0
        for r in self.radix:
            t *= r
        return t


def lower(dag: dict, bundle: dict, bounds: dict) -> Lowered:
    lib = Library.from_bundle(bundle)
    b = Bounds.from_json(bounds)
    ids = [n["id"] for n in dag["nodes"]]
    index = {i: k for k, i in enumerate(ids)}
    options, plans, quality, tokens = [], [], [], []
    for n in dag["nodes"]:
        opts = node_options(n, lib, b)
        options.append(opts)
        plans.append([plan_node_execution(n, o, lib) for o in opts])
        quality.append([node_quality(n, lib.impls[o["implementation"]]["quality"], o["path_count"]) for o in opts])
        tokens.append([token(n["id"], o) for o in opts])
    topo = [index[i] for i in topological_order(dag)]
    edges = [(index[e["from"]], index[e["to"]]) for e in dag["edges"]]
    return Lowered(ids, options, plans, quality, tokens, topo, edges)
