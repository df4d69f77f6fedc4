"""Synthetic plan spaces for the five BASELINE.json configs, emitted in the
reference's own JSON formats (library bundle agent_library.hpp:327-344,
dag.json workflow.hpp:303-363, objective = the spec's constraint token +
optional quality_floor, workflow.hpp:91-106,182-183) so the compiled
reference and the oracle read them unchanged.  Seeds are fixed; generation
uses only random.Random.random() so it is identical on every Python 3.

  C1  video-understanding fixture (tests/golden/c1, produced by the reference
      planner from the bundled fixture), MIN_COST, 168 plans
  C2  the same 4-task video DAG over a sweep library (model variant x CPU/GPU
      x GPU generation x fan-out 1-32), MIN_LATENCY + quality floor 3,
      3 x 262 x 4 x 384 = 1,207,296 plans
  C3  10-task layered DAG, 16 options per task, 16^10 = 1.1e12 plans,
      MIN_COST under a latency SLO (the SLO is the config-3 extension)
  C4  10,000 jobs x 6 tasks x 8 options (262,144 plans per job), MIN_COST
  C5  9-task DAG x 10 options, 1e9 plans, Pareto frontier (quality constant,
      so the reference's 4-D dominance is the 3-D (cost, latency, energy) one)
"""
from __future__ import annotations

import json
import random
from dataclasses import dataclass
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"


@dataclass
class Workload:
    name: str
    dag: dict
    library: dict
    bounds: dict
    objective: dict

    def texts(self) -> tuple[str, str, str, str]:
        return (json.dumps(self.dag), json.dumps(self.library), json.dumps(self.objective),
                json.dumps(self.bounds))


def _u(rng: random.Random, lo: float, hi: float) -> float:
    return lo + (hi - lo) * rng.random()


def _i(rng: random.Random, lo: int, hi: int) -> int:
    return lo + min(hi - lo, int(rng.random() * (hi - lo + 1)))


def _sku(id_, cls, busy, idle, rate):
    return {"id": id_, "class": cls, "generation": id_, "capacity_unit": "core" if cls == "cpu" else "device",
            "busy_watts_per_unit": busy, "idle_watts_per_unit": idle, "dollars_per_unit_hour": rate}


def _agent(cap, consumes="text", produces="text"):
    return {"capability": cap, "schema": [], "consumes": consumes, "produces": produces}


def _impl(name, cap, quality, classes):
    return {"name": name, "capability": cap, "quality": quality, "supported_classes": classes}


def _prof(impl, sku, units, thr, setup=0.0):
    return {"implementation": impl, "sku": sku, "units": units, "throughput": thr, "setup_seconds": setup}


def _node(id_, cap, work, splittable, min_chunk=0.0, multi_path=False, ceiling=None, consumes=("text",),
          produces="text"):
    n = {"id": id_, "capability": cap, "work_units": work, "splittable": splittable, "min_chunk": min_chunk,
         "multi_path": multi_path, "origin": "hinted", "consumes": list(consumes), "produces": produces,
         "tool_calls": []}
    if ceiling is not None:
        n["path_quality_ceiling"] = ceiling
    return n


def _layered_edges(rng: random.Random, ids: list[str], skip_p: float) -> list[dict]:
    edges = []
    for i in range(1, len(ids)):
        for p in range(i):
            if p == i - 1 or rng.random() < skip_p:
                edges.append({"from": ids[p], "to": ids[i], "kind": "text"})
    return edges


# ---------------------------------------------------------------------------
def config1() -> Workload:
    d = GOLDEN / "c1"
    return Workload("c1_video_min_cost", json.loads((d / "dag.json").read_text()),
                    json.loads((d / "library.json").read_text()), json.loads((d / "bounds.json").read_text()),
                    {"constraint": "MIN_COST"})


# ---------------------------------------------------------------------------
C2_LEXICON = [
    {"keywords": ["extract", "extraction", "frames", "frame", "video", "videos", "sample"],
     "capability": "frame_extraction", "consumes": "video", "produces": "image",
     "defaults": {"start_time": 0.0, "frame_rate": 0.16666666666666666}, "splittable": False,
     "work_factor": 0.16666666666666666},
    {"keywords": ["speech", "text", "transcribe", "transcription", "transcript", "audio"],
     "capability": "speech_to_text", "consumes": "video", "produces": "text", "defaults": {"language": "en"},
     "splittable": True, "min_chunk": 18.75, "work_factor": 2.0},
    {"keywords": ["detect", "detection", "objects", "object", "recognize"], "capability": "object_detection",
     "consumes": "image", "produces": "text", "defaults": {"top_k": 5}, "splittable": False, "work_factor": 2.2},
    {"keywords": ["summarize", "summary", "describe", "scenes", "scene", "caption"], "capability": "summarization",
     "consumes": ["image", "text"], "produces": "text", "defaults": {"context_len": 4096}, "splittable": True,
     "min_chunk": 47.5, "work_factor": 1.0, "multi_path": True, "path_quality_ceiling": 4},
    {"keywords": ["list", "objects", "shown", "mentioned", "videos", "video", "understanding"],
     "capability": "video_understanding",
     "expansion": ["frame_extraction", "speech_to_text", "object_detection", "summarization"]},
]

C2_SPEC = {
    "description": "List objects shown/mentioned in the videos",
    "tasks": ["Extract frames from each video", "Run speech-to-text on all scenes", "Detect objects in the frames",
              "Summarize the scenes using frames, detected objects and transcripts"],
    "inputs": [{"id": "cats.mov", "media_kind": "video", "work_units": 300},
               {"id": "formula_1.mov", "media_kind": "video", "work_units": 300}],
    "constraint": "MIN_LATENCY", "quality_floor": 3, "mode": "declarative"}


def config2_library() -> dict:
    skus = [_sku("cpu-epyc", "cpu", 25.0, 5.0, 0.05), _sku("gpu-a100", "gpu", 400.0, 60.0, 3.0),
            _sku("gpu-h100", "gpu", 700.0, 90.0, 4.5), _sku("gpu-b200", "gpu", 1000.0, 140.0, 7.0)]
    agents = [_agent("frame_extraction", "video", "image"), _agent("speech_to_text", "video", "text"),
              _agent("object_detection", "image", "text"), _agent("summarization", ["image", "text"], "text")]
    impls = [_impl("ffmpeg-keyframes", "frame_extraction", 3, ["cpu"]),
             _impl("opencv-frame-extractor", "frame_extraction", 2, ["cpu"]),
             _impl("pyav-sampler", "frame_extraction", 1, ["cpu"]),
             _impl("whisper-large", "speech_to_text", 3, ["cpu", "gpu"]),
             _impl("whisper", "speech_to_text", 2, ["cpu", "gpu"]),
             _impl("owlvit-l", "object_detection", 3, ["cpu", "gpu"]),
             _impl("clip", "object_detection", 2, ["cpu"]),
             _impl("nvlm", "summarization", 3, ["gpu"]),
             _impl("llava-next", "summarization", 2, ["gpu"])]
    profs = [_prof("ffmpeg-keyframes", "cpu-epyc", 16, 28.0), _prof("opencv-frame-extractor", "cpu-epyc", 16, 32.0),
             _prof("pyav-sampler", "cpu-epyc", 16, 40.0)]
    for name, scale in (("whisper-large", 0.7), ("whisper", 1.0)):
        profs += [_prof(name, "cpu-epyc", 16, 3.3333333333333335 * scale), _prof(name, "gpu-a100", 1, 4.8 * scale),
                  _prof(name, "gpu-h100", 1, 8.5 * scale), _prof(name, "gpu-b200", 1, 14.0 * scale)]
    profs += [_prof("owlvit-l", "cpu-epyc", 16, 3.5), _prof("owlvit-l", "gpu-a100", 1, 9.0),
              _prof("owlvit-l", "gpu-h100", 1, 16.0), _prof("clip", "cpu-epyc", 16, 5.0)]
    for name, scale in (("nvlm", 1.0), ("llava-next", 1.4)):
        profs += [_prof(name, "gpu-a100", 2, 10.0 * scale), _prof(name, "gpu-h100", 2, 18.0 * scale),
                  _prof(name, "gpu-b200", 1, 16.0 * scale)]
    return {"skus": skus, "agents": agents, "implementations": impls, "profiles": profs}


def config2_dag() -> dict:
    """What the reference planner emits for C2_SPEC with C2_LEXICON (pinned by
    tests/golden/make_golden.py against the compiled reference)."""
    ids = ["t0_frame_extraction", "t1_speech_to_text", "t2_object_detection", "t3_summarization"]
    nodes = [_node(ids[0], "frame_extraction", 600.0, False, consumes=("video",), produces="image"),
             _node(ids[1], "speech_to_text", 600.0, True, 18.75, consumes=("video",)),
             _node(ids[2], "object_detection", 100.0, False, consumes=("image",)),
             _node(ids[3], "summarization", 1520.0, True, 47.5, True, 4, consumes=("image", "text"))]
    edges = [{"from": ids[0], "to": ids[2], "kind": "image"}, {"from": ids[0], "to": ids[3], "kind": "image"},
             {"from": ids[1], "to": ids[3], "kind": "text"}, {"from": ids[2], "to": ids[3], "kind": "text"}]
    return {"nodes": nodes, "edges": edges}


def config2() -> Workload:
    caps = {"cpu-epyc": 768, "gpu-a100": 64, "gpu-h100": 64, "gpu-b200": 64}
    pool = {"cpu-epyc": 96, "gpu-a100": 8, "gpu-h100": 8, "gpu-b200": 8}
    return Workload("c2_video_sweep_min_latency_q3", config2_dag(), config2_library(),
                    {"max_fanout": 32, "max_paths": 2, "sku_pool_cap": pool, "sku_total_cap": caps},
                    {"constraint": "MIN_LATENCY", "quality_floor": 3})


# ---------------------------------------------------------------------------
C3_SEED = 20250316
# 10th percentile of the latencies of 200,000 uniformly sampled plans of the
# C3 space (derived once with the oracle).  It does NOT bind at the MIN_COST
# optimum: the best all-CPU plan takes 47,258,723 us and has gpu_wh = 0, so the
# argmin is the node-local greedy seed (tests/golden/c3/full_space.json).
C3_SLO_US = 72043534
# The bench's headline SLO: below the all-CPU optimum, so every feasible plan
# puts work on GPUs, MIN_COST trades GPU energy against the critical path, and
# the argmin is not the greedy seed (checked by bench.py and the tests).
C3_BINDING_SLO_US = 40_000_000


def _two_class_library(rng: random.Random, caps: list[str], cpu_units: tuple[int, int],
                       gpus: tuple[str, str]) -> dict:
    skus = [_sku("cpu-epyc", "cpu", _u(rng, 5.0, 30.0), 1.0, _u(rng, 0.01, 0.2)),
            _sku(gpus[0], "gpu", _u(rng, 200.0, 500.0), 40.0, _u(rng, 1.0, 5.0)),
            _sku(gpus[1], "gpu", _u(rng, 400.0, 1000.0), 60.0, _u(rng, 2.0, 8.0))]
    agents, impls, profs = [], [], []
    for cap in caps:
        agents.append(_agent(cap))
        impls.append(_impl(cap + "-cpu", cap, 2, ["cpu"]))
        impls.append(_impl(cap + "-gpu", cap, 3, ["gpu"]))
        for u in cpu_units:
            profs.append(_prof(cap + "-cpu", "cpu-epyc", u, _u(rng, 0.5, 20.0) * u / cpu_units[0],
                               _u(rng, 0.0, 5.0)))
        for g in gpus:
            profs.append(_prof(cap + "-gpu", g, 1, _u(rng, 0.5, 20.0) * (2.0 if g == gpus[1] else 1.0),
                               _u(rng, 0.0, 5.0)))
    return {"skus": skus, "agents": agents, "implementations": impls, "profiles": profs}


def config3(seed: int = C3_SEED, slo_us: int | None = C3_SLO_US) -> Workload:
    rng = random.Random(seed)
    caps = [f"c{i}" for i in range(10)]
    lib = _two_class_library(rng, caps, (16, 32), ("gpu-a100", "gpu-h100"))
    ids = [f"t{i}_c{i}" for i in range(10)]
    nodes = []
    for i, cap in enumerate(caps):
        work = _u(rng, 50.0, 200.0)
        nodes.append(_node(ids[i], cap, work, True, work / _u(rng, 4.0, 8.0)))
    dag = {"nodes": nodes, "edges": _layered_edges(rng, ids, 0.15)}
    bounds = {"max_fanout": 4, "max_paths": 1, "sku_pool_cap": {"cpu-epyc": 96, "gpu-a100": 8, "gpu-h100": 8},
              "sku_total_cap": {"cpu-epyc": 192, "gpu-a100": 16, "gpu-h100": 16}}
    obj = {"constraint": "MIN_COST"}
    if slo_us is not None:
        obj["latency_slo_us"] = slo_us
    return Workload("c3_synthetic10_min_cost_slo", dag, lib, bounds, obj)


# ---------------------------------------------------------------------------
C4_SEED = 4242
C4_CAPS = 32


def config4_library(seed: int = C4_SEED) -> dict:
    rng = random.Random(seed)
    return _two_class_library(rng, [f"k{i:02d}" for i in range(C4_CAPS)], (8, 16), ("gpu-a100", "gpu-h100"))


def config4_job(j: int, seed: int = C4_SEED) -> dict:
    rng = random.Random(seed * 1_000_003 + j)
    picks: list[int] = []
    while len(picks) < 6:
        c = _i(rng, 0, C4_CAPS - 1)
        if c not in picks:
            picks.append(c)
    ids = [f"t{i}_k{c:02d}" for i, c in enumerate(picks)]
    nodes = []
    for i, c in enumerate(picks):
        work = _u(rng, 20.0, 200.0)
        nodes.append(_node(ids[i], f"k{c:02d}", work, True, work / _u(rng, 2.0, 6.0)))
    return {"nodes": nodes, "edges": _layered_edges(rng, ids, 0.25)}


C4_BOUNDS = {"max_fanout": 2, "max_paths": 1, "sku_pool_cap": {"cpu-epyc": 96, "gpu-a100": 8, "gpu-h100": 8},
             "sku_total_cap": {"cpu-epyc": 192, "gpu-a100": 16, "gpu-h100": 16}}


# C4's binding objective: every tenant asks for MIN_COST under its own latency
# SLO of 110 % of its fastest plan (the critical path with every node at its
# fastest option, loom_latency_floor).  Without an SLO every C4 winner is an
# all-CPU plan (gpu_wh = 0) that node-local choices already find.
C4_SLO_PERCENT = 110


def c4_slo_objective(latency_floor_us: int) -> dict:
    return {"constraint": "MIN_COST", "latency_slo_us": latency_floor_us * C4_SLO_PERCENT // 100}


def config4(n_jobs: int = 10_000, seed: int = C4_SEED) -> list[Workload]:
    lib = config4_library(seed)
    return [Workload(f"c4_job{j}", config4_job(j, seed), lib, C4_BOUNDS, {"constraint": "MIN_COST"})
            for j in range(n_jobs)]


# ---------------------------------------------------------------------------
C5_SEED = 9090


def config5(seed: int = C5_SEED, n_nodes: int = 9) -> Workload:
    rng = random.Random(seed)
    caps = [f"p{i}" for i in range(9)]
    skus = [_sku("cpu-epyc", "cpu", 22.0, 4.0, 0.06), _sku("gpu-h100", "gpu", 700.0, 90.0, 4.5)]
    agents, impls, profs = [], [], []
    for cap in caps:
        agents.append(_agent(cap))
        # equal quality: the reference's 4-D dominance reduces to (dollars, gpu_wh, latency)
        impls.append(_impl(cap + "-cpu", cap, 2, ["cpu"]))
        impls.append(_impl(cap + "-gpu", cap, 2, ["gpu"]))
        profs.append(_prof(cap + "-cpu", "cpu-epyc", 16, _u(rng, 0.5, 6.0), _u(rng, 0.5, 5.0)))
        profs.append(_prof(cap + "-gpu", "gpu-h100", 1, _u(rng, 4.0, 20.0), _u(rng, 0.5, 5.0)))
    lib = {"skus": skus, "agents": agents, "implementations": impls, "profiles": profs}
    ids = [f"t{i}_p{i}" for i in range(9)]
    nodes = []
    for i, cap in enumerate(caps):
        work = _u(rng, 40.0, 200.0)
        nodes.append(_node(ids[i], cap, work, True, work / _u(rng, 5.0, 9.0)))
    edges = _layered_edges(rng, ids, 0.2)
    keep = set(ids[:n_nodes])
    dag = {"nodes": nodes[:n_nodes], "edges": [e for e in edges if e["from"] in keep and e["to"] in keep]}
    bounds = {"max_fanout": 5, "max_paths": 1, "sku_pool_cap": {"cpu-epyc": 96, "gpu-h100": 8},
              "sku_total_cap": {"cpu-epyc": 192, "gpu-h100": 16}}
    return Workload(f"c5_pareto{n_nodes}", dag, lib, bounds, {"constraint": "MIN_COST"})


# ---------------------------------------------------------------------------
def random_scenario(seed: int, max_nodes: int = 4, with_setup: bool = True, ample: bool = True,
                    max_fanout: int = 4, max_paths: int = 2) -> Workload:
    """Small random instances in the spirit of the reference's
    make_random_scenario (tests/support.hpp:85-174): one cpu and one gpu sku,
    1-2 implementations per capability supporting both classes, 1-2 profile
    variants per sku, random splittable / multi-path flags, layered edges."""
    rng = random.Random(seed)
    skus = [_sku("sim-cpu", "cpu", _u(rng, 5.0, 30.0), 1.0, _u(rng, 0.01, 0.2)),
            _sku("sim-gpu", "gpu", _u(rng, 200.0, 500.0), 20.0, _u(rng, 1.0, 5.0))]
    n = _i(rng, 1, max_nodes)
    agents, impls, profs, nodes = [], [], [], []
    for i in range(n):
        cap = f"cap{i}"
        agents.append(_agent(cap))
        for m in range(_i(rng, 1, 2)):
            name = f"{cap}_impl{m}"
            impls.append(_impl(name, cap, _i(rng, 0, 3), ["cpu", "gpu"]))
            for sku in ("sim-cpu", "sim-gpu"):
                seen = set()
                for v in range(_i(rng, 1, 2)):
                    units = _i(rng, 1, 4) * (v + 1)
                    prof = _prof(name, sku, units, _u(rng, 0.5, 20.0), _u(rng, 0.0, 5.0) if with_setup else 0.0)
                    if units not in seen:
                        seen.add(units)
                        profs.append(prof)
        work = _u(rng, 5.0, 200.0)
        split = _i(rng, 0, 1) == 1
        multi = _i(rng, 0, 3) == 0
        nodes.append(_node(f"t{i}_{cap}", cap, work, split, work / _i(rng, 2, 8) if split else 0.0, multi,
                           5 if multi else None))
    ids = [x["id"] for x in nodes]
    edges = _layered_edges(rng, ids, 0.5)
    scale = 64 if ample else _i(rng, 8, 24)
    bounds = {"max_fanout": max_fanout, "max_paths": max_paths,
              "sku_pool_cap": {"sim-cpu": scale, "sim-gpu": scale},
              "sku_total_cap": {"sim-cpu": 2 * scale, "sim-gpu": 2 * scale}}
    tokens = ["MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"]
    return Workload(f"random{seed}", {"nodes": nodes, "edges": edges},
                    {"skus": skus, "agents": agents, "implementations": impls, "profiles": profs}, bounds,
                    {"constraint": tokens[seed % 4]})
