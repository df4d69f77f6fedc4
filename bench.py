"""bench.py -- plans evaluated per second for the B200 exhaustive plan search.

Workload (BASELINE.json configs[2], "C3"): a synthetic 10-task DAG with 16
lever assignments per task, 16^10 = 1.1e12 plans, MIN_COST under a binding
latency SLO.  N > 1 (torchrun, one rank per GPU): by default every rank runs
its own whole-space search (N independent scheduling requests: weak
scaling); --sharded splits ONE search's plan space by contiguous index range
across the ranks through the library's NCCL group (strong scaling; the
frontier search is latency-bound, so this barely shortens it -- DESIGN.md
§7).  configs[1] (C2, 1.2e6 plans) finishes in microseconds and is reported
under "configs" with C1/C4/C5 as time-to-plan lines, not as the headline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one exhaustive search of the whole plan space: the exact argmin of
objective_less over all 1.1e12 plans, by the default
algorithm -- branch and bound over the ConfigEnumerator tree with exact
subtree bounds, the every-plan sweep as its fallback.  "value" counts plans
COVERED per second (the whole space / step time); the plans evaluated exactly
(leaves) and the subtree bounds computed are reported beside it, and the
every-plan sweep of the same instance is its own line (configs.c3_sweep).
"value" times the search with the problem resident in HBM (CUDA events on
the launching stream, L2 flushed between steps); "e2e" times the public
drop-in call
(reference-format JSON in, selected plan out: lowering, H2D, kernel, D2H,
NCCL all-gather of winners, decode) every step.  --impl reference times the
UNMODIFIED reference (oracle/_ref, compiled from /root/reference) on the
host cores over a bounded sample of the same plan space.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "plans evaluated/sec (1/2/4/8 B200, % of roofline) vs CPU ref; time-to-plan"
WORKLOAD = ("C3: 10-task layered DAG x 16 options/task = 1.1e12 plans, MIN_COST (min gpu energy, then latency) "
            "under a BINDING 40 s latency SLO (below the 47.26 s all-CPU optimum: the argmin needs GPU nodes and is "
            "not the greedy seed)")
UNIT = "plans/s"


# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0, "fallback": True}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.  A C3 step
    takes well under a millisecond, so nvidia-smi's 100-ms loop would see no
    sample: NVML is polled from a thread every ~0.2 ms instead (the main
    thread spends the region in CUDA synchronisation, which releases the GIL).
    Falls back to nvidia-smi when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int):
        self.device = device
        self.sm: list[float] = []
        self.max_sm: list[float] = []
        self.reasons: set[str] = set()
        self.stop = threading.Event()
        self.thread = None
        self.nv = None

    def _handle(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return nv, nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:  # noqa: BLE001 -- older torch: fall back to the index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            return nv, nv.nvmlDeviceGetHandleByIndex(idx)

    def _poll(self, nv, h):
        bits = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(name for name, b in bits if b and r & b)
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.0002)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.max_sm.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001 -- no NVML: one nvidia-smi reading after the region
            self.thread = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=5)
        elif not self.sm:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=30).stdout.split(",")
                self.sm.append(float(out[0]))
                self.max_sm.append(float(out[1]))
            except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
                pass

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.max_sm) if self.max_sm else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml, polled every ~0.2 ms during the timed region" if self.thread is not None
                else "nvidia-smi after the timed region"}


# ---------------------------------------------------------------------------
def reference_arm(args) -> None:
    """The reference's own CPU implementation (oracle/_ref range driver over
    loom::estimate / meets_quality_floor / objective_less), all host threads,
    a bounded sample of the C3 plan space per step."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2501_16634_b200 import workloads as W

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    w = W.config3(slo_us=W.C3_BINDING_SLO_US)
    threads = os.cpu_count() or 1
    sample = args.ref_sample
    base = 123_456_789_012  # a slice that holds SLO-feasible plans
    times = []
    for step in range(args.warmup + args.steps):
        b = base + step * sample
        t0 = time.perf_counter()
        rc, out = O.ref_range_argmin(w.dag, w.library, w.objective, w.bounds, b, b + sample, threads)
        dt = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError(out)
        if step >= args.warmup:
            times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = sample / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+i64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "plans_per_step": sample,
                       "parallelism": f"reference CPU range driver, {threads} host threads",
                       "sample": "a bounded slice of the same plan space per step (the full space would take "
                                 "~1e6 s on the host)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{sample} consecutive plan indices of C3 per step, range driver over the "
                                       f"reference's estimate/objective_less on {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def cpu_baseline(seconds_budget: float = 12.0) -> dict:
    """The compiled reference on this box's host cores over a bounded C3
    sample (rank 0, N=1 only)."""
    from oracle import oracle as O
    from paper_2501_16634_b200 import workloads as W

    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref missing"}
    w = W.config3(slo_us=W.C3_BINDING_SLO_US)
    threads = os.cpu_count() or 1
    b = 123_456_789_012
    probe = 20_000 * threads
    rc, out = O.ref_range_argmin(w.dag, w.library, w.objective, w.bounds, b, b + probe, threads)
    rate = probe / max(out["seconds"], 1e-6)
    sample = int(max(probe, min(rate * seconds_budget, 5e8)))
    rc, out = O.ref_range_argmin(w.dag, w.library, w.objective, w.bounds, b, b + sample, threads)
    # the same whole-space answer by the oracle's plain-C branch and bound on
    # the host cores (a port, not the reference): what a CPU caller gets from
    # the bounding idea alone
    p = O.problem(w.dag, w.library, w.bounds)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r, visited = O.argmin_bnb(p, w.objective, threads)
        ts.append(time.perf_counter() - t0)
    return {"value": sample / out["seconds"], "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{sample} consecutive C3 plans from index {b}: reference estimate + objective_less "
                      f"(oracle/_ref range driver, g++ -O2) on {threads} host threads, {out['seconds']:.1f} s",
            "cpu_branch_and_bound_port": {"ms": 1e3 * min(ts), "threads": threads, "plan_index": r["index"],
                                          "subtrees_and_leaves_visited": visited,
                                          "what": "oracle/flat_oracle.c oracle_argmin_bnb over the whole space"}}


def flush_l2(torch, buf) -> None:
    buf.add_(1)  # 256 MiB read+write > 126 MB L2


def b200_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2501_16634_b200 import dist as D, loom, workloads as W

    world, rank, local = dist_env()
    # one process per GPU; LOOM_DIST_BACKEND=gloo lets ranks share a GPU when
    # validating the multi-rank path on a single-GPU box
    backend = os.environ.get("LOOM_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.Stream()
    # N > 1, default: N independent searches, one per GPU (weak scaling: each
    # rank serves its own scheduling request over the whole C3 space).  The
    # frontier branch and bound finishes one request in ~0.2 ms, bound by its
    # per-level critical path, so splitting ONE request's plan space across
    # GPUs barely shortens it (max shard time 0.20 ms at N = 8).
    # --sharded: one request split by plan-index range instead -- over NCCL
    # through the library's own multi-GPU group (loom_group_create_rank: its
    # NCCL communicator, the sharded search and the ncclAllGather of the
    # per-rank records all live in libloom_b200.so; torch.distributed only
    # hands rank 0's NCCL id to the other ranks and times the ranks).
    sharded = world > 1 and args.sharded
    replicas = world > 1 and not sharded
    use_group = sharded and backend == "nccl"
    group = None
    if use_group:
        ids = [loom.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        group = loom.Group(device=local, rank=rank, world=world, nccl_id=ids[0], stream=stream.cuda_stream)
        ctx = None
    else:
        ctx = loom.Context(local, stream.cuda_stream)
    w = W.config3(slo_us=W.C3_BINDING_SLO_US)
    dag_t, lib_t, obj_t, bounds_t = w.texts()

    lw = loom.Lowered(w.dag, w.library, w.bounds)
    obj = loom.objective(w.objective)
    total = lw.total
    begin, end = D.shard_range(total, rank, world) if sharded else (0, total)
    dp = loom.DeviceProblem(ctx, lw.problem, obj) if not use_group else None
    scratch = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    group_out = {}

    def shard_result():
        if use_group:
            return group_out["w"]
        try:
            return dp.result()
        except loom.NoFeasibleConfigError:  # nothing feasible in this rank's shard
            return D.empty_winner()

    # ---- value: resident problem, device-timed -------------------------------
    # N > 1: each rank searches its index range plus the greedy seed as a common
    # incumbent (loom_search_argmin_shard), so every shard prunes like the
    # whole-space search; the reduce over ranks is still the exact argmin.
    def search(b, e):
        if use_group:  # the whole space, sharded and exchanged inside the library
            group_out["w"] = group.search_argmin(lw.problem, obj)
        elif sharded:
            dp.search_shard_async(b, e)
        else:
            dp.search_async(b, e)

    for _ in range(args.warmup):
        search(begin, end)
        shard_result()
    count_launches = (lambda: group.launches()) if use_group else (lambda: ctx.launches)
    launches0 = count_launches()
    step_ms = []
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush_l2(torch, scratch)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            search(begin, end)
            e1.record(stream)
            shard_result()
            step_ms.append(e0.elapsed_time(e1))
        barrier()
    launches = count_launches() - launches0
    bnb = loom.bnb_last_stats()  # the last timed launch (this rank's job)
    local_ms = sum(step_ms) / len(step_ms)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([local_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    units = total * (world if replicas else 1)  # plans covered by all ranks per step
    value = units / (ms / 1e3)

    # winners must agree with a full-space reduce (checked every run)
    local_w = shard_result()
    winners = D.allgather_winners(local_w, device=red_dev) if sharded and not use_group else [local_w]
    chosen = D.combine(winners, obj)
    seed = greedy_seed_index(loom, lw, obj)
    # the headline is a real search: the SLO binds and the argmin is not the
    # node-local greedy seed the kernels may start from
    assert chosen["plan_index"] != seed and chosen["latency_us"] <= W.C3_BINDING_SLO_US, (chosen, seed)

    # ---- e2e: the public drop-in call, host JSON in / plan out ---------------
    def e2e_step():
        if not sharded:
            return loom.exhaustive_search(dag_t, lib_t, obj_t, bounds_t, ctx=ctx)
        if use_group:
            return group.exhaustive_search(dag_t, lib_t, obj_t, bounds_t)
        low = loom.Lowered(dag_t, lib_t, bounds_t)
        o = loom.objective(obj_t)
        mine = D.search_shard(ctx, low.problem, o, rank, world)
        best = D.combine(D.allgather_winners(mine, device=red_dev), o)
        return low.config(best["plan_index"]) | best

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        out = e2e_step()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    te = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units / (float(te.item()) / 1e3)
    assert out["plan_index"] == chosen["plan_index"], (out, chosen)

    if dp is not None:
        image_bytes = dp.image_bytes
    else:
        probe = loom.DeviceProblem(group.context(0), lw.problem, obj)
        image_bytes = probe.image_bytes
        probe.close()
    if rank == 0:
        pk = peaks()
        clk = clocks.summary()
        f_mhz = clk["sm_mhz"] or pk.get("sm_max_mhz", 1965.0)
        props = torch.cuda.get_device_properties(local)
        sms = props.multi_processor_count
        issue = sms * 4 * 32 * f_mhz * 1e6  # thread-instructions per second
        # Dominant kernel: bfs_kernel, the frontier branch and bound (the whole
        # timed step is one graph launch: this kernel, a conditional node that
        # stays closed unless the frontier overflows, and the 48-byte D2H).
        # Its duration is read live from the kernel's own %globaltimer trace
        # (CTA 0's start to the last CTA's exit) over a few extra searches.
        kern_us, levels = [], None
        for _ in range(5):
            search(begin, end)
            shard_result()
            tr = loom.bfs_trace()
            if tr["total_us"]:
                kern_us.append(tr["total_us"])
                levels = tr["levels"]
        kernel_s = statistics.median(kern_us) / 1e6 if kern_us else local_ms / 1e3
        n_nodes, n_edges = lw.problem.n_nodes, lw.problem.n_edges
        i_eval = 12 * n_nodes + 3 * n_edges + 20  # SURVEY.md §8(d) full-evaluation count
        evals = bnb["child_evaluations"]
        prof_p = ROOT / "profiles" / "ncu_summary.json"
        prof = json.loads(prof_p.read_text()) if prof_p.exists() else {}
        fr = prof.get("bfs_kernel", {})
        inst = fr.get("warp_inst_per_launch")
        issue_peak = sms * 4 * f_mhz * 1e6  # warp instructions per second (one issue per SMSP per clock)
        roofline = {
            "bound": "instruction issue (latency-limited: level-synchronous critical path)",
            "kernel": "bfs_kernel" if not bnb["depth_first"] else "bnb_kernel",
            "achieved": inst / kernel_s if inst else None, "peak": issue_peak, "unit": "warp instructions/s",
            "frac": inst / kernel_s / issue_peak if inst else None,
            "traffic": fr.get("dram_bytes_per_launch"),
            "kernel_us": 1e6 * kernel_s,
            "warp_inst_per_launch": inst,
            "work": {"unit": "subtree bounds + leaf evaluations (children) per second",
                     "children_per_launch": evals, "achieved": evals / kernel_s,
                     "full_evaluation_ceiling": issue * 1.0 / i_eval,
                     "frac": evals / kernel_s / (issue / i_eval),
                     "inst_per_evaluation": i_eval},
            "levels": levels,
            "note": "achieved = warp instructions of one launch (ncu smsp__inst_executed.sum, profiles/ncu_summary.json) "
                    "/ the launch's live device time; peak = SMs x 4 SMSPs x measured SM clock.  The kernel is bound "
                    "by the latency of its per-level critical path (grid barrier + one expansion chain per level, "
                    "'levels' = per-level device time), not by issue or HBM: 'work' compares the children it "
                    f"evaluates with the full-evaluation ceiling (12N+3E+20 = {i_eval} thread-instructions each, "
                    "SURVEY.md §8d).  traffic = DRAM bytes per launch (ncu)."}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if replicas else "strong",
            "vs_baseline": None, "dtype": "f64+i64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "objective": w.objective,
                       "plans_per_step": units,
                       "parallelism": (f"{world} independent whole-space searches, one per GPU" if replicas else
                                       f"plan-index range x{world}" + (" (loom_group: NCCL inside the library)"
                                                                      if use_group else "")),
                       "l2": "flushed between timed steps (256 MiB write); the problem image is 8 KB in smem",
                       "value_counts": "plans COVERED per second: every plan of the space is in the argmin's "
                                       "domain; subtrees whose exact criteria bound is infeasible or strictly "
                                       "worse than a plan already found are dropped whole",
                       "plans_exactly_evaluated": bnb["leaves"],
                       "subtree_bounds_and_leaves_evaluated": evals,
                       "plans_exactly_evaluated_per_s": bnb["leaves"] / (local_ms / 1e3),
                       "depth_first_fallback_taken": bnb["depth_first"],
                       "sweep_fallback_taken": bnb["aborted"],
                       "largest_frontier": bnb["max_frontier"],
                       "chosen_plan_index": chosen["plan_index"], "greedy_seed_index": seed,
                       "chosen_latency_us": chosen["latency_us"], "chosen_gpu_wh": chosen["gpu_wh"],
                       "golden": "tests/golden/c3/full_space.json (CPU oracle, whole space)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": float(te.item()),
                    "h2d_bytes_per_step": image_bytes + 64, "d2h_bytes_per_step": 64,
                    "path": "loom_exhaustive_search_json: JSON parse + lowering + H2D + kernel + D2H + decode"
                    if not sharded else "loom_group_exhaustive_search_json: JSON parse + lowering + per-rank shard "
                    "search (range + greedy incumbent) + ncclAllGather of the rank records + reduce + decode"},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        if not args.no_configs and world == 1:
            line["configs"] = other_configs(ctx, loom, W, issue)
        print(json.dumps(line), flush=True)
    if dp is not None:
        dp.close()
    if ctx is not None:
        ctx.close()
    if group is not None:
        group.close()
    if world > 1:
        dist.destroy_process_group()


def greedy_seed_index(loom, lw, obj) -> int:
    import ctypes as C
    d = (C.c_int32 * lw.problem.n_nodes)()
    rc = loom.lib().loom_greedy_seed(C.byref(lw.problem), C.byref(obj), d)
    assert rc == 0
    idx = 0
    for x, r in zip(d, lw.radix):
        idx = idx * r + x
    return idx


def device_ms(torch, ctx_stream, fn, reps: int) -> float:
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx_stream)
        fn()
        e1.record(ctx_stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def c3_lines(ctx, loom, W, issue: float) -> dict:
    """The C3 instance under other objectives, and the every-plan sweep of the
    headline instance (LOOM_ALGO_SWEEP: each plan gets its own compare in the
    fast path; roofline on the compiled sweep's SASS count)."""
    import torch
    stream = torch.cuda.Stream()
    sctx = loom.Context(torch.cuda.current_device(), stream.cuda_stream)
    w = W.config3(slo_us=None)
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    out = {}
    fp = FAST_PATH
    cyc_per_plan = max(fp["issue"], 2 * fp["alu"], 2 * fp["fp64"]) / fp["plans_per_lane"]
    sweep_peak = issue / cyc_per_plan
    cases = [("c3_binding_slo_sweep", {"constraint": "MIN_COST", "latency_slo_us": W.C3_BINDING_SLO_US},
              loom.ALGO_SWEEP),
             ("c3_certify_nonbinding_slo", {"constraint": "MIN_COST", "latency_slo_us": W.C3_SLO_US}, loom.ALGO_AUTO),
             ("c3_certify_nonbinding_slo_sweep", {"constraint": "MIN_COST", "latency_slo_us": W.C3_SLO_US},
              loom.ALGO_SWEEP),
             ("c3_min_latency", {"constraint": "MIN_LATENCY"}, loom.ALGO_AUTO),
             ("c3_min_dollars_binding_slo", {"constraint": "MIN_DOLLARS", "latency_slo_us": W.C3_BINDING_SLO_US},
              loom.ALGO_AUTO),
             ("c3_max_quality", {"constraint": "MAX_QUALITY"}, loom.ALGO_AUTO)]
    for name, o, algo in cases:
        ob = loom.objective(o)
        dp = loom.DeviceProblem(sctx, lw.problem, ob)
        run = lambda: dp.search_algo_async(0, None, algo)  # noqa: E731
        run()
        r = dp.result()
        t = device_ms(torch, stream, run, 3 if algo == loom.ALGO_SWEEP else 10) / 1e3
        line = {"objective": o, "algo": "sweep (every plan tested)" if algo == loom.ALGO_SWEEP else
                "default (branch and bound, sweep fallback)", "ms": 1e3 * t, "plans_covered_per_s": lw.total / t,
                "plan_index": r["plan_index"], "greedy_seed_index": greedy_seed_index(loom, lw, ob),
                "latency_us": r["latency_us"], "gpu_wh": r["gpu_wh"]}
        if algo == loom.ALGO_SWEEP:
            line["roofline"] = {"bound": "instruction issue (compiled sweep fast path)", "achieved": lw.total / t,
                                "peak": sweep_peak, "unit": "plans tested/s", "frac": lw.total / t / sweep_peak,
                                "note": f"{fp['issue']} SASS instructions per {fp['plans_per_lane']} plans per lane "
                                        "in search_kernel<4, kPrimFp, 16, paired>; flagged contexts (plans that "
                                        "pass the energy compare) take the exact slow path"}
        else:
            st = loom.bnb_last_stats()
            line.update({"plans_exactly_evaluated": st["leaves"], "subtree_bounds_and_leaves": st["child_evaluations"],
                         "depth_first_fallback_taken": st["depth_first"], "sweep_fallback_taken": st["aborted"],
                         "largest_frontier": st["max_frontier"]})
        out[name] = line
        dp.close()
    lw.close()
    sctx.close()
    return out


# Compiled fast path of the innermost contexts of search_kernel<4, kPrimFp,
# 16, true> (tools/sass_blocks.py 4 0 16 1): one fully unrolled block sweeps
# two options of the node two above the innermost x the 16 options of the
# node above it = 512 plans per lane in 675 SASS instructions -- 256
# DSETP.LE.OR and 256 ISETP.LE.OR (one compare per plan on its primary
# criterion: half the options on the FP64 pipe, half on the ALU pipe with
# high words), 66 DADD, 24 LDCU (tables from the constant bank), step flags
# -- of which 301 run on the ALU pipe and 322 on the FP64 pipe: issue-bound.
# DESIGN.md §5.
FAST_PATH = {"issue": 675, "alu": 301, "fp64": 322, "plans_per_lane": 512}


def other_configs(ctx, loom, W, issue: float) -> dict:
    """Time-to-plan for the other BASELINE configs (outside the timed region):
    C1/C2 through the JSON drop-in call; C4 = batched lowering + one batched
    search of 10,000 jobs; C5 = the full Pareto frontier."""
    out = c3_lines(ctx, loom, W, issue)
    for name, w in (("c1", W.config1()), ("c2", W.config2())):
        dag_t, lib_t, obj_t, bounds_t = w.texts()
        loom.exhaustive_search(dag_t, lib_t, obj_t, bounds_t, ctx=ctx)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            r = loom.exhaustive_search(dag_t, lib_t, obj_t, bounds_t, ctx=ctx)
            ts.append(time.perf_counter() - t0)
        out[name] = {"time_to_plan_ms": 1e3 * min(ts), "plans": r["plans"], "identifier": r["identifier"],
                     "latency_us": r["latency_us"], "gpu_wh": r["gpu_wh"]}
    jobs = W.config4(10_000)
    # the tenants' dag.json texts as the bytes a caller hands the C ABI (a
    # Python str would be re-encoded per call: ~5 ms of interpreter work for
    # 10,000 texts that is not the library's)
    dags = [json.dumps(j.dag).encode() for j in jobs]
    lib_t, bounds_t = json.dumps(jobs[0].library), json.dumps(jobs[0].bounds)
    gold_p = ROOT / "tests" / "golden" / "c4" / "all_jobs.json"
    gold = json.loads(gold_p.read_text())["objectives"] if gold_p.exists() else {}
    # MIN_LATENCY binds (off the critical path a node takes its lowest-energy
    # option with slack, so winners differ from the greedy seed); MIN_COST's
    # winners are all-CPU plans (certify case)
    for key, token in (("c4", "MIN_LATENCY"), ("c4_min_cost", "MIN_COST")):
        obj_t = json.dumps({"constraint": token})  # one objective for every tenant
        loom.exhaustive_search_batch(dags[:64], lib_t, obj_t, bounds_t, ctx=ctx)
        ts = []
        for _ in range(3):  # the whole multi-tenant call: JSON in, 10,000 winners out
            t0 = time.perf_counter()
            res = loom.exhaustive_search_batch(dags, lib_t, obj_t, bounds_t, ctx=ctx)
            ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        batch = loom.LoweredBatch(dags, lib_t, bounds_t)
        t1 = time.perf_counter()
        res2 = loom.search_lowered_batch(ctx, batch, loom.objective(token))
        t2 = time.perf_counter()
        plans = sum(batch[k].total for k in range(len(batch)))
        assert all(res[k] == res2[k] for k in range(0, len(batch), 97))
        batch.close()
        match = None
        if token in gold:
            match = sum(1 for k, g in enumerate(gold[token]) if g is not None and res[k][0] == 0 and [
                res[k][1]["plan_index"], res[k][1]["latency_us"], res[k][1]["gpu_wh"], res[k][1]["dollars"]] == g)
        out[key] = {"objective": token, "jobs": len(jobs), "plans": plans, "time_to_plan_ms": 1e3 * min(ts),
                    "lowering_ms": 1e3 * (t1 - t0), "search_ms": 1e3 * (t2 - t1),
                    "plans_covered_per_s": plans / (t2 - t1), "feasible_jobs": res.feasible(),
                    "jobs_matching_full_space_golden": match,
                    "path": "loom_exhaustive_search_batch (JSON in, winners out); lowering/search split from "
                            "LoweredBatch + loom_search_argmin_lowered"}
    # greedy_search (the reference CLI's default) on the GPU, one CTA
    w3 = W.config3(slo_us=None)
    g_args = (json.dumps(w3.dag), json.dumps(w3.library), {"constraint": "MIN_COST"}, json.dumps(w3.bounds))
    loom.greedy_search(*g_args, ctx=ctx)
    t0 = time.perf_counter()
    g = loom.greedy_search(*g_args, ctx=ctx)
    out["c3_greedy"] = {"time_to_plan_ms": 1e3 * (time.perf_counter() - t0), "latency_us": g["latency_us"],
                        "gpu_wh": g["gpu_wh"]}
    w5 = W.config5()
    lw5 = loom.Lowered(w5.dag, w5.library, w5.bounds)
    loom.search_pareto_points(ctx, lw5.problem, 0, lw5.total - 1)
    t5s = []
    for k in range(3):  # distinct ranges: the ctx caches the last frontier
        t0 = time.perf_counter()
        front = loom.search_pareto_points(ctx, lw5.problem, 0, lw5.total - (k % 2))
        t5s.append(time.perf_counter() - t0)
    front = loom.search_pareto_points(ctx, lw5.problem, 0, lw5.total)
    t5 = statistics.median(t5s)
    out["c5"] = {"plans": lw5.total, "frontier_points": len(front), "time_to_frontier_ms": 1e3 * t5,
                 "plans_per_s": lw5.total / t5}
    out["c3_score_stream"] = score_stream(ctx, loom, W)
    # dominant kernels of C4 / C5 against the instruction-issue roofline, from
    # one ncu capture each (tools/ncu_c4c5.sh -> profiles/ncu_summary.json):
    # warp instructions / kernel time vs SMs x 4 SMSPs x clock
    prof_p = ROOT / "profiles" / "ncu_summary.json"
    prof = json.loads(prof_p.read_text()) if prof_p.exists() else {}
    for key, name, kern in (("c4", "c4_bnb_kernel", "bnb_kernel (depth-first branch and bound, one CTA per job)"),
                            ("c5", "c5_pareto_eval_kernel", "pareto_eval_kernel (corner-pruned evaluation)")):
        k = prof.get(name)
        if k and key in out:
            t = k["duration_ns_under_ncu"] / 1e9
            ach = k["warp_inst_per_launch"] / t
            out[key]["roofline"] = {"bound": "instruction issue", "kernel": kern, "achieved": ach, "peak": issue / 32,
                                    "unit": "warp instructions/s", "frac": ach * 32 / issue,
                                    "traffic": k["dram_bytes_per_launch"], "kernel_ms_under_ncu": 1e3 * t,
                                    "source": "one ncu --set full capture (profiles/ncu_summary.json); the "
                                              "configuration's time_to_plan is host-inclusive"}
    return out


def score_stream(ctx, loom, W, log2: int = 28) -> dict:
    """Per-plan estimate streams (loom_estimate_range_device): estimate() of
    2^28 consecutive C3 plans written to HBM as six SoA streams (44 B/plan,
    11.8 GB per launch, larger than L2).  HBM-bound: the roofline is the
    measured copy bandwidth.  e2e = the host-buffer call (kernel + D2H of
    every stream into pinned memory)."""
    import torch
    w = W.config3()
    lw = loom.Lowered(w.dag, w.library, w.bounds)
    n, b = 1 << log2, 1000
    dt = {"int64": torch.int64, "float64": torch.float64, "int32": torch.int32}
    dev = {f: torch.empty(n, dtype=dt[t], device="cuda") for f, t in loom.STREAM_FIELDS.items()}
    bpp = sum(t.element_size() for t in dev.values())
    stream = torch.cuda.current_stream()
    sctx = loom.Context(torch.cuda.current_device(), stream.cuda_stream)
    loom.estimate_range_device(sctx, lw.problem, b, b + n, dev)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        loom.estimate_range_device(sctx, lw.problem, b, b + n, dev)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms) / 1e3
    # spot-check a few plans against the host's exact per-plan estimate
    for k in (0, n // 3, n - 1):
        ref = lw.evaluate(b + k)
        assert dev["latency_us"][k].item() == ref["latency_us"] and dev["gpu_wh"][k].item() == ref["gpu_wh"]
    del dev
    nh = 1 << 24
    host = {f: torch.empty(nh, dtype=dt[t_], pin_memory=True) for f, t_ in loom.STREAM_FIELDS.items()}
    loom.estimate_range_host(sctx, lw.problem, b, b + nh, host)
    th = []
    for _ in range(3):
        t0 = time.perf_counter()
        loom.estimate_range_host(sctx, lw.problem, b, b + nh, host)
        th.append(time.perf_counter() - t0)
    sctx.close()
    hbm = peaks().get("hbm_gbs", 6548.5)
    gbs = n * bpp / t / 1e9
    return {"plans": n, "bytes_per_plan": bpp, "ms": 1e3 * t, "plans_per_s": n / t,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "traffic_per_plan_bytes": bpp},
            "e2e": {"plans": nh, "ms": 1e3 * min(th), "plans_per_s": nh / min(th),
                    "d2h_gbs": nh * bpp / min(th) / 1e9, "d2h_bytes": nh * bpp,
                    "path": "loom_estimate_range into pinned host arrays (kernel + D2H per 4M-plan chunk)"}}



def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="N > 1: split ONE search's plan space across the ranks (strong scaling) instead of one "
                         "independent search per rank")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the time-to-plan lines of C1/C2/C4/C5 and C3 greedy")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
