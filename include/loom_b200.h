/*
 * loom_b200.h -- C ABI of the B200-native plan-evaluation library.
 *
 * This is the ONE boundary the B200 build adds to the reference (SURVEY.md
 * §1, §8b).  The reference ("loom", header-only C++20) has no process or
 * device boundary; its plugin point is the function symbol.  Each entry point
 * below names the reference interface it replaces:
 *
 *   loom_search_argmin        loom::exhaustive_search     optimizer.hpp:173-188
 *                             (ConfigEnumerator 110-150 + estimate estimator.hpp:43-78
 *                              + meets_quality_floor 118-121 + objective_less 93-116)
 *   loom_search_argmin_batch  a loop of exhaustive_search over many jobs (config 4)
 *   loom_search_pareto        loom::pareto_filter         optimizer.hpp:153-171
 *                             applied to estimate(p) for p in ConfigEnumerator order
 *   loom_winner_reduce        objective_less as a total-order reduce (multi-GPU combine)
 *   loom_evaluate_plan        loom::estimate               estimator.hpp:43-78 (one plan)
 *   loom_estimate_range(_device) / loom_estimate_plans
 *                             estimate() over an index range / an index list,
 *                             as per-plan score streams (SoA)
 *   loom_lower                node_options optimizer.hpp:51-107 + plan_node_execution
 *                             chunking.hpp:85-184 + ConfigPoint::identifier config.hpp:49-61
 *   loom_exhaustive_search_json   the whole drop-in call on reference-format JSON
 *
 * Conventions: POD arguments only, caller-owned buffers, int status return
 * (LOOM_OK / LOOM_INFEASIBLE / LOOM_INVALID / LOOM_DEVICE_ERROR), and a
 * thread-local message from loom_last_error() formatted like the reference's
 * loom::Error::what() ("<ErrorClass>: <message>", errors.hpp:17-19).  One
 * loom_ctx per host thread; a ctx is bound to one CUDA device and stream.
 * There is no CPU fallback: compute entry points fail with LOOM_DEVICE_ERROR
 * when no sm_100 device is present.
 */
#ifndef LOOM_B200_H
#define LOOM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOOM_B200_ABI_VERSION 1

/* Status codes.  INFEASIBLE <-> NoFeasibleConfigError (optimizer.hpp:184-186);
 * INVALID <-> InvalidConfigError / SchemaError / CycleError / UnknownCapabilityError. */
#define LOOM_OK 0
#define LOOM_INFEASIBLE 1
#define LOOM_INVALID 2
#define LOOM_DEVICE_ERROR 3

/* Criterion, workflow.hpp:67 (same enumerator order). */
#define LOOM_MIN_COST_DOLLARS 0
#define LOOM_MIN_ENERGY 1
#define LOOM_MIN_LATENCY 2
#define LOOM_MAX_QUALITY 3

/*
 * A lowered plan space.  Nodes are in dag.nodes order, which is the
 * ConfigEnumerator order (node 0 most significant digit, last node fastest,
 * optimizer.hpp:136-141) and also the left-fold order of the energy / dollar
 * sums in estimate (estimator.hpp:50-60).  Option arrays are node-major:
 * option o of node i sits at index offset(i) + o with offset(i) = sum of
 * radix[0..i).  Per-option values are the reference's per-node plan values
 * ALREADY multiplied by path_count exactly as estimate does (estimator.hpp:51-53).
 */
typedef struct loom_problem {
  int32_t n_nodes;
  int32_t n_edges;
  const int32_t* radix;        /* [n_nodes] node_options(...).size()                    */
  const int64_t* wall_us;      /* [sum radix] NodePlan.wall_us (chunking.hpp:171)         */
  const double* gpu_wh;        /* [sum radix] NodePlan.gpu_wh * path_count                */
  const double* cpu_wh;        /* [sum radix] NodePlan.cpu_wh * path_count                */
  const double* dollars;       /* [sum radix] NodePlan.dollars * path_count               */
  const int32_t* quality;      /* [sum radix] node_quality (estimator.hpp:32-37)          */
  const int32_t* lexrank;      /* [sum radix] rank of the option's identifier substring
                                  among the node's options (config.hpp:49-61)           */
  const uint64_t* lex_weight;  /* [n_nodes] mixed-radix weight of the node in sorted
                                  node-id order: product of radix over nodes whose id
                                  sorts after it (std::map order, config.hpp:46)        */
  const int32_t* edge_from;    /* [n_edges] node indices (dag.nodes order)                */
  const int32_t* edge_to;      /* [n_edges]                                               */
} loom_problem;

/* ObjectiveHierarchy (workflow.hpp:81-86) + the config-3 latency-SLO extension. */
typedef struct loom_objective {
  int32_t n_criteria;          /* 0..4 */
  int32_t criteria[4];         /* LOOM_MIN_* / LOOM_MAX_QUALITY, most significant first */
  int32_t has_quality_floor;
  int32_t quality_floor;
  int32_t has_latency_slo;     /* extension, not in the reference: latency_us <= slo */
  int32_t reserved;
  int64_t latency_slo_us;
} loom_objective;

/* The selected plan: ConfigEstimate (estimator.hpp:20-30) minus the strings,
 * plus its enumeration index and identifier rank.  64 bytes, POD, so it can be
 * all-gathered across ranks as raw bytes. */
typedef struct loom_winner {
  uint64_t plan_index;         /* position in ConfigEnumerator order              */
  uint64_t lexkey;             /* rank of ConfigPoint::identifier() in the space  */
  int64_t latency_us;
  double gpu_wh;
  double cpu_wh;
  double total_wh;
  double dollars;
  int32_t quality;
  int32_t found;               /* 0: no feasible plan in the searched range       */
} loom_winner;

/* One plan's Pareto coordinates (pareto_filter's dominance axes,
 * optimizer.hpp:155-161).  40 bytes, POD. */
typedef struct loom_point {
  uint64_t plan_index;
  double dollars;
  double gpu_wh;
  int64_t latency_us;
  int32_t quality;
  int32_t reserved;
} loom_point;

typedef struct loom_ctx loom_ctx;
typedef struct loom_device_problem loom_device_problem;
typedef struct loom_lowered loom_lowered;

/* ---- library / errors -------------------------------------------------- */
int loom_abi_version(void);
const char* loom_last_error(void);

/* ---- host-only helpers (no device needed) ------------------------------ */
/* Product of radices (ConfigEnumerator::total_count, optimizer.hpp:124-129);
 * LOOM_INVALID on overflow past 2^64 (the reference wraps silently). */
int loom_problem_total(const loom_problem* problem, uint64_t* total);
/* Exact reference estimate of one plan (estimator.hpp:43-78) into a winner record. */
int loom_evaluate_plan(const loom_problem* problem, uint64_t plan_index, loom_winner* out);
/* objective_less over winner records; found==0 records lose.  Deterministic. */
/* The smallest latency_us of any plan whose options meet the objective's
 * quality floor (objective may be NULL): the critical path (estimator.hpp:69-76)
 * with every node at its fastest option.  A latency SLO below it is infeasible. */
int loom_latency_floor(const loom_problem* problem, const loom_objective* objective, int64_t* out);
int loom_winner_less(const loom_winner* a, const loom_winner* b, const loom_objective* objective);
int loom_winner_reduce(const loom_winner* winners, int32_t n, const loom_objective* objective,
                       loom_winner* out);
/* Parse an objective JSON: {"constraint": "MIN_COST"} or {"criteria": [...]},
 * optional "quality_floor", optional "latency_slo_us" (workflow.hpp:91-106, 182-183). */
int loom_objective_parse(const char* objective_json, loom_objective* out);

/* ---- lowering of reference-format JSON (host) -------------------------- */
/* dag_json: WorkflowDag JSON (workflow.hpp:303-363); library_json: library
 * bundle (agent_library.hpp:327-344); bounds_json: SearchBounds as
 * {"max_fanout":4,"max_paths":2,"sku_pool_cap":{..},"sku_total_cap":{..}}. */
int loom_lower(const char* dag_json, const char* library_json, const char* bounds_json,
               loom_lowered** out);
/* Many DAGs against one library bundle and bounds (config 4: the library is
 * parsed once and the DAGs are lowered on `threads` host threads; 0 = the
 * CPUs this process may run on).
 * out[i] receives a handle or NULL; status[i] the per-DAG status. */
int loom_lower_batch(const char* library_json, const char* bounds_json, const char* const* dag_jsons,
                     int32_t n, int32_t threads, loom_lowered** out, int32_t* status);
const loom_problem* loom_lowered_problem(const loom_lowered* lowered);
/* ConfigPoint JSON (config.hpp:88-95) + "identifier" for a plan index. */
int loom_lowered_config_json(const loom_lowered* lowered, uint64_t plan_index, char* buf,
                             size_t cap, size_t* needed);
/* NodeAssignment JSON + identifier substring of one option. */
int loom_lowered_option_json(const loom_lowered* lowered, int32_t node, int32_t option, char* buf,
                             size_t cap, size_t* needed);
void loom_lowered_destroy(loom_lowered* lowered);

/* ---- device context ---------------------------------------------------- */
/* cuda_stream: a cudaStream_t to launch on (NULL: the ctx creates its own;
 * (void*)1 = cudaStreamLegacy, the legacy default stream). */
int loom_ctx_create(int32_t device, void* cuda_stream, loom_ctx** out);
int loom_ctx_destroy(loom_ctx* ctx);
/* Kernel launches issued by this ctx since creation (evidence for benches). */
uint64_t loom_ctx_launch_count(const loom_ctx* ctx);
/* The cudaStream_t the ctx launches on. */
void* loom_ctx_stream(const loom_ctx* ctx);

/* ---- multi-GPU groups ----------------------------------- */
/* A group owns one device context per local GPU and one NCCL communicator
 * (NCCL over NVLink/NVSwitch).  The plan space shards by contiguous index
 * ranges (loom_shard_range), every rank starts from the same incumbent (the
 * greedy seed), and one ncclAllGather of the per-rank results plus the
 * deterministic objective_less reduce gives every rank the same winner --
 * the caller of exhaustive_search (loom_main.cpp:140-146) sees one call.
 *   loom_group_create(mask):   this process drives every device in the mask
 *                              (bit d = device d; ncclCommInitAll; one host
 *                              thread per device per call);
 *   loom_group_create_rank():  one process per GPU (torchrun-style): rank 0
 *                              makes an id with loom_nccl_unique_id, the
 *                              caller distributes it, every rank joins. */
#define LOOM_NCCL_ID_BYTES 128
typedef struct loom_group loom_group;
int loom_nccl_unique_id(uint8_t* out /* LOOM_NCCL_ID_BYTES */);
int loom_group_create(uint64_t device_mask, loom_group** out);
int loom_group_create_rank(int32_t device, void* cuda_stream, const uint8_t* nccl_id, int32_t rank,
                           int32_t world, loom_group** out);
int loom_group_destroy(loom_group* group);
int32_t loom_group_world(const loom_group* group);  /* GPUs in the whole group    */
int32_t loom_group_local(const loom_group* group);  /* GPUs driven by this process */
int32_t loom_group_rank(const loom_group* group);   /* group rank of local GPU 0   */
loom_ctx* loom_group_ctx(loom_group* group, int32_t local_index);
/* Contiguous shard [*b, *e) of [begin, end) for rank of world (host only). */
int loom_shard_range(uint64_t begin, uint64_t end, int32_t rank, int32_t world, uint64_t* b, uint64_t* e);
/* loom_search_argmin over the group: every rank returns the same winner. */
int loom_group_search_argmin(loom_group* group, const loom_problem* problem, const loom_objective* objective,
                             uint64_t begin, uint64_t end, loom_winner* out);
/* loom_search_pareto_points over the group (per-rank frontiers, all-gathered,
 * filtered on the device, ascending plan index). */
int loom_group_search_pareto_points(loom_group* group, const loom_problem* problem, uint64_t begin, uint64_t end,
                                    loom_point* out, uint64_t capacity, uint64_t* count);
/* loom_search_argmin_batch over the group (contiguous job ranges per rank). */
int loom_group_search_argmin_batch(loom_group* group, const loom_problem* problems,
                                   const loom_objective* objectives, int32_t n_jobs, loom_winner* out,
                                   int32_t* status);
/* loom_exhaustive_search_json over the group. */
int loom_group_exhaustive_search_json(loom_group* group, const char* dag_json, const char* library_json,
                                      const char* objective_json, const char* bounds_json, char* out_json,
                                      size_t cap, size_t* needed);

/* ---- search (device) ---------------------------------------------------- */
/* Argmin over plan indices [begin, end) (end clamped to the total).  Fills
 * every field of *out from the winning index.  LOOM_INFEASIBLE when nothing in
 * the range is feasible (out->found == 0). */
int loom_search_argmin(loom_ctx* ctx, const loom_problem* problem, const loom_objective* objective,
                       uint64_t begin, uint64_t end, loom_winner* out);

/* Same, selecting the evaluation algorithm:
 *   LOOM_ALGO_AUTO  (default) branch and bound over the ConfigEnumerator tree
 *                   -- subtrees whose criteria lower bound is infeasible or
 *                   strictly worse than a plan already found are dropped --
 *                   with the exhaustive sweep as its fallback when the bound
 *                   prunes too little;
 *   LOOM_ALGO_FULL  one plan per thread, re-evaluated from scratch
 *                   (independent cross-check);
 *   LOOM_ALGO_SWEEP the hierarchical sweep alone: every plan of the range is
 *                   tested in the fast path. */
#define LOOM_ALGO_AUTO 0
#define LOOM_ALGO_FULL 1
#define LOOM_ALGO_SWEEP 2
int loom_search_argmin_algo(loom_ctx* ctx, const loom_problem* problem,
                            const loom_objective* objective, uint64_t begin, uint64_t end,
                            int32_t algo, loom_winner* out);

/* Per-job argmin over whole plan spaces (config 4).  status[j] gets the
 * per-job status; the call returns LOOM_OK unless the batch itself failed. */
int loom_search_argmin_batch(loom_ctx* ctx, const loom_problem* problems,
                             const loom_objective* objectives, int32_t n_jobs,
                             loom_winner* out, int32_t* status);

/* Multi-tenant batch on lowered handles (config 4): one objective for every
 * job; a NULL handle gets status LOOM_INVALID.  No per-job marshalling. */
int loom_search_argmin_lowered(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n,
                               const loom_objective* objective, loom_winner* out, int32_t* status);

/* Same with one objective per job (objectives[i] for lowered[i]). */
int loom_search_argmin_lowered_each(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n,
                                    const loom_objective* objectives, loom_winner* out, int32_t* status);

/* The whole multi-tenant call on reference-format JSON: n DAGs against one
 * library bundle, bounds and objective -> n winners (a loop of
 * exhaustive_search, optimizer.hpp:173-188).  On `threads` host threads
 * (0 = the CPUs this process may run on, at most 64, kept by the context),
 * blocks of 64 jobs are lowered, imaged and copied to the device while the
 * searches of the blocks already staged run.  status[i] is the job's status.
 * A context runs one batch at a time. */
/* objective_json is one objective for every job, or a JSON array of n
 * per-job objectives (e.g. per-tenant latency SLOs). */
int loom_exhaustive_search_batch(loom_ctx* ctx, const char* library_json, const char* bounds_json,
                                 const char* const* dag_jsons, int32_t n, const char* objective_json,
                                 int32_t threads, loom_winner* out, int32_t* status);

/* Shard search (multi-GPU partitions): the argmin of
 * [begin, end) u {incumbent}, where the incumbent is any plan of the space --
 * LOOM_INCUMBENT_GREEDY for the greedy seed (loom_greedy_seed).  Every rank
 * starting from the same incumbent prunes like a whole-space search, and the
 * reduce of the per-rank results over a partition of the space is still the
 * exact argmin (the incumbent is itself a plan of the space).  out->plan_index
 * may be the incumbent's, outside [begin, end). */
#define LOOM_INCUMBENT_GREEDY UINT64_MAX
int loom_search_argmin_shard(loom_ctx* ctx, const loom_problem* problem, const loom_objective* objective,
                             uint64_t begin, uint64_t end, uint64_t incumbent, loom_winner* out);

/* Resident problems: upload once, search many times (bench "value" path). */
int loom_problem_upload(loom_ctx* ctx, const loom_problem* problem, const loom_objective* objective,
                        loom_device_problem** out);
int loom_problem_release(loom_device_problem* dp);
/* Bytes of the problem image one search copies host->device (evidence for benches). */
uint64_t loom_device_problem_bytes(const loom_device_problem* dp);
/* Enqueue a search on the ctx stream without synchronising. */
int loom_search_argmin_async(loom_ctx* ctx, loom_device_problem* dp, uint64_t begin, uint64_t end);
/* loom_search_argmin_shard on a resident problem, enqueued without synchronising. */
int loom_search_argmin_shard_async(loom_ctx* ctx, loom_device_problem* dp, uint64_t begin, uint64_t end,
                                   uint64_t incumbent);
/* loom_search_argmin_async with a chosen LOOM_ALGO_* and incumbent
 * (LOOM_NO_INCUMBENT, LOOM_INCUMBENT_GREEDY or a plan index). */
#define LOOM_NO_INCUMBENT (UINT64_MAX - 1)
int loom_search_argmin_algo_async(loom_ctx* ctx, loom_device_problem* dp, uint64_t begin, uint64_t end,
                                  uint64_t incumbent, int32_t algo);
/* Evidence of the last default (LOOM_ALGO_AUTO) search, job 0 (6 entries):
 * out[0] = children evaluated (subtree bounds + leaves, all stages),
 * out[1] = bit 0: the depth-first search ran (the frontier search overflowed
 *          its buffers or did not apply); bit 1: its budget ran out and the
 *          every-plan sweep finished the search,
 * out[2] = largest frontier (frontier search) or longest work unit (depth first),
 * out[3] = CTAs of the frontier launch (or work units alive at the root),
 * out[4] = complete plans evaluated exactly (leaves),
 * out[5] = children evaluated by the depth-first search. */
int loom_bnb_last_stats(uint64_t* out);
/* Per-level timeline of the last frontier search (profiling aid): out[0] =
 * start and out[1] = end (%globaltimer ns), then per depth d out[2d+2] = end of
 * the level, out[2d+3] = parents expanded (bit 63: evaluated redundantly by
 * every CTA, without a grid barrier).  cap entries at most (<= 68). */
int loom_bfs_trace(uint64_t* out, int32_t cap);
/* Wait for the last enqueued search of dp and decode its result. */
int loom_search_argmin_result(loom_ctx* ctx, loom_device_problem* dp, loom_winner* out);

/* Pareto frontier of the plans in [begin, end) under pareto_filter's
 * dominance (raw doubles: dollars, gpu_wh; latency_us; quality, higher
 * better).  Indices are returned ascending (enumeration order).  Size query:
 * call with capacity 0 to get *count. */
int loom_search_pareto(loom_ctx* ctx, const loom_problem* problem, uint64_t begin, uint64_t end,
                       uint64_t* out_index, uint64_t capacity, uint64_t* count);
/* Same, returning the frontier's coordinates (for multi-rank merging).  A
 * call with capacity < count only reports *count; the result of the last
 * search is cached in the ctx, so the follow-up call does not search again. */
int loom_search_pareto_points(loom_ctx* ctx, const loom_problem* problem, uint64_t begin, uint64_t end,
                              loom_point* out, uint64_t capacity, uint64_t* count);
/* pareto_filter on an arbitrary point set (optimizer.hpp:153-171):
 * keep[i] = 1 iff no other point dominates point i.  Runs on the device. */
int loom_pareto_filter_points(loom_ctx* ctx, const loom_point* points, uint64_t n, uint8_t* keep);

/* ---- per-plan estimate streams (estimator.hpp:43-78) ----------------------- */
/* Structure-of-arrays score streams: element i holds one field of
 * estimate(plan) (ConfigEstimate, estimator.hpp:20-30).  A NULL stream is not
 * written (and costs no memory traffic). */
typedef struct loom_estimate_streams {
  int64_t* latency_us;
  double* gpu_wh;
  double* cpu_wh;
  double* total_wh;
  double* dollars;
  int32_t* quality;
} loom_estimate_streams;

/* estimate(p) for every plan p in [begin, end) (end clamped to the total) in
 * ConfigEnumerator order (optimizer.hpp:131-143): element i = plan begin + i.
 * The reference's equivalent is a loop of ConfigEnumerator::next + estimate.
 * HOST arrays, filled when the call returns. */
int loom_estimate_range(loom_ctx* ctx, const loom_problem* problem, uint64_t begin, uint64_t end,
                        const loom_estimate_streams* out);
/* Same into DEVICE arrays on the ctx's device, enqueued on the ctx stream
 * without synchronising (each warp stores whole aligned 32-element windows). */
int loom_estimate_range_device(loom_ctx* ctx, const loom_problem* problem, uint64_t begin, uint64_t end,
                               const loom_estimate_streams* out);
/* Batched estimate of arbitrary plans: element i =
 * estimate(indices[i]); LOOM_INVALID if an index is out of range.  HOST arrays. */
int loom_estimate_plans(loom_ctx* ctx, const loom_problem* problem, const uint64_t* indices, uint64_t n,
                        const loom_estimate_streams* out);

/* ---- greedy_search (optimizer.hpp:227-291) -------------------------------- */
/* Node-local seed of greedy_search (optimizer.hpp:194-220, 256-268): per node,
 * among options meeting the quality floor, the first minimum of the criteria
 * values of the option alone.  LOOM_INFEASIBLE if a node has none
 * (optimizer.hpp:248-251). */
int loom_greedy_seed(const loom_problem* problem, const loom_objective* objective, int32_t* digits);
/* Coordinate descent from `seed` (NULL: loom_greedy_seed), re-optimizing one
 * node at a time in `sweep_order` (NULL: index-ordered Kahn; the reference
 * uses topological_order, see loom_lowered_sweep_order) for at most
 * `max_sweeps` sweeps, stopping after a sweep without improvement.  Each
 * node step evaluates all of the node's options on the device at once; the
 * result equals the reference's sequential first-improvement scan because
 * the objective order is strict. */
int loom_search_greedy(loom_ctx* ctx, const loom_problem* problem, const loom_objective* objective,
                       const int32_t* sweep_order, const int32_t* seed, int32_t max_sweeps, loom_winner* out);
/* The reference's topological_order (workflow.hpp:467-498, peers by node id) as node indices. */
int loom_lowered_sweep_order(const loom_lowered* lowered, int32_t* out);
/* greedy_search(dag, library, objective, bounds) on reference-format JSON; same output as
 * loom_exhaustive_search_json. */
int loom_greedy_search_json(loom_ctx* ctx, const char* dag_json, const char* library_json, const char* objective_json,
                            const char* bounds_json, int32_t max_sweeps, char* out_json, size_t cap, size_t* needed);

/* ---- the drop-in call on reference-format JSON -------------------------- */
/* exhaustive_search(dag, library, objective, bounds) -> ConfigEstimate JSON:
 * {"identifier","config","latency_us","gpu_wh","cpu_wh","total_wh","dollars",
 *  "quality","plan_index","plans"}.  On error the JSON is {"error","message"}. */
int loom_exhaustive_search_json(loom_ctx* ctx, const char* dag_json, const char* library_json,
                                const char* objective_json, const char* bounds_json, char* out_json,
                                size_t cap, size_t* needed);

/* The --pin path (loom_main.cpp:125-146): parse a config point
 * (config.hpp:66-117 parse_config_point, with its SchemaError messages) and
 * return estimate(config, dag, library) (estimator.hpp:43-78) as the same
 * ConfigEstimate JSON, without "plan_index"/"plans".  Host only: one plan.
 * Missing dag tasks are rejected like the pinned-plan mode
 * (ValidationError: pinned_plan: missing assignment for task '<id>'). */
int loom_estimate_config_json(const char* dag_json, const char* library_json, const char* config_json,
                              char* out_json, size_t cap, size_t* needed);

#ifdef __cplusplus
}
#endif

#endif /* LOOM_B200_H */
