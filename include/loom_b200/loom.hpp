// loom_b200/loom.hpp -- C++ drop-in for the reference's search entry points.
//
// Same namespace, type names and signatures as the reference's hot path so a
// caller switches by changing the include and linking libloom_b200.so:
//
//   ConfigEstimate exhaustive_search(const WorkflowDag&, const AgentLibrary&,
//                                    const ObjectiveHierarchy&, const SearchBounds&);
//                                          reference: optimizer.hpp:173-176
//   std::vector<NodeAssignment> node_options(const DagNode&, const AgentLibrary&,
//                                            const SearchBounds&);   optimizer.hpp:51-53
//   NodePlan plan_node_execution(const DagNode&, const NodeAssignment&,
//                                const AgentLibrary&);               chunking.hpp:85-87
//   ConfigEstimate estimate(const ConfigPoint&, const WorkflowDag&,
//                           const AgentLibrary&);                    estimator.hpp:43-44
//   bool objective_less(const ConfigEstimate&, const ConfigEstimate&,
//                       const ObjectiveHierarchy&);                  estimator.hpp:93-94
//   std::vector<ConfigEstimate> pareto_filter(const std::vector<ConfigEstimate>&);
//                                                                    optimizer.hpp:153-154
//
// Only the data the hot path reads is modelled (no lexicon, planner, cluster
// or simulator: SURVEY.md §2 marks them out of scope).  The search itself
// runs on the GPU through the C ABI in loom_b200.h; nothing here falls back
// to a CPU search.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "loom_b200.h"

namespace loom {

using Micros = std::int64_t;

// time.hpp:15-19: one rounding onto the microsecond grid, half away from zero.
Micros to_micros(double seconds);
inline double to_seconds(Micros us) { return static_cast<double>(us) / 1e6; }

// ---- errors (errors.hpp:10-58): category drives the CLI exit code --------
enum class ErrorCategory : int { spec = 2, planning = 3, search = 4, simulation = 5 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCategory category, std::string code, const std::string& message);
  ErrorCategory category() const { return category_; }
  const std::string& code() const { return code_; }

 private:
  ErrorCategory category_;
  std::string code_;
};

#define LOOM_B200_ERROR(Name, Cat)                                              \
  struct Name : Error {                                                          \
    explicit Name(const std::string& m) : Error(ErrorCategory::Cat, #Name, m) {} \
  };
LOOM_B200_ERROR(SchemaError, spec)
LOOM_B200_ERROR(ValidationError, spec)
LOOM_B200_ERROR(CycleError, spec)
LOOM_B200_ERROR(DuplicateKeyError, spec)
LOOM_B200_ERROR(DanglingReferenceError, spec)
LOOM_B200_ERROR(UnknownCapabilityError, spec)
LOOM_B200_ERROR(InvalidConfigError, search)
LOOM_B200_ERROR(NoFeasibleConfigError, search)
#undef LOOM_B200_ERROR

// ---- profile tables (agent_library.hpp:18-80) ---------------------------
enum class HardwareClass { cpu, gpu };

struct HardwareSku {
  std::string id;
  HardwareClass hardware_class = HardwareClass::cpu;
  double busy_watts_per_unit = 0.0;
  double idle_watts_per_unit = 0.0;
  double dollars_per_unit_hour = 0.0;
};

struct Implementation {
  std::string name;
  std::string capability;
  int quality = 0;
  bool supports_cpu = false;
  bool supports_gpu = false;
  bool supports(HardwareClass c) const { return c == HardwareClass::cpu ? supports_cpu : supports_gpu; }
};

struct ExecutionProfile {
  std::string implementation;
  std::string sku;
  int units = 1;
  double throughput = 0.0;
  double setup_seconds = 0.0;
};

// Read-only catalog built from a library bundle; lookups mirror
// agent_library.hpp:251-297 (implementations best quality first, then name;
// profiles in (implementation, sku, units) order).
class AgentLibrary {
 public:
  AgentLibrary() = default;
  AgentLibrary(const AgentLibrary& other);  // copies rebuild the pointer indexes
  AgentLibrary& operator=(const AgentLibrary& other);
  AgentLibrary(AgentLibrary&&) noexcept = default;  // map nodes move with the maps
  AgentLibrary& operator=(AgentLibrary&&) noexcept = default;

  static AgentLibrary from_json_text(const std::string& bundle_json);

  void add_capability(const std::string& capability);
  void add_sku(HardwareSku sku);
  void add_implementation(Implementation impl);
  void add_profile(ExecutionProfile profile);

  const HardwareSku* sku(const std::string& id) const;
  const Implementation* implementation(const std::string& name) const;
  const ExecutionProfile* profile(const std::string& impl, const std::string& sku, int units) const;
  std::vector<const Implementation*> implementations_for(const std::string& capability) const;
  std::vector<const ExecutionProfile*> profiles_for(const std::string& implementation) const;

 private:
  std::map<std::string, bool> capabilities_;
  // std::less<>: heterogeneous lookup (no key copies on the lowering path)
  std::map<std::string, HardwareSku, std::less<>> skus_;
  std::map<std::string, Implementation, std::less<>> impls_;
  std::map<std::tuple<std::string, std::string, int>, ExecutionProfile, std::less<>> profiles_;
  // Indexes kept in lookup order as entries are added (map nodes are stable):
  // implementations per capability (quality desc, then name) and profiles
  // per implementation ((sku, units) order).
  std::map<std::string, std::vector<const Implementation*>, std::less<>> impls_by_cap_;
  std::map<std::string, std::vector<const ExecutionProfile*>, std::less<>> profiles_by_impl_;
  void rebuild_indexes();
};

// ---- dag + objective (workflow.hpp:67-106, 259-301) ---------------------
struct DagNode {
  std::string id;
  std::string capability;
  double work_units = 0.0;
  bool splittable = false;
  double min_chunk = 0.0;
  bool multi_path = false;
  std::optional<int> path_quality_ceiling;
};

struct Edge {
  std::string from;
  std::string to;
};

struct WorkflowDag {
  std::vector<DagNode> nodes;
  std::vector<Edge> edges;
  static WorkflowDag from_json_text(const std::string& dag_json);
};

enum class Criterion { min_cost_dollars, min_energy, min_latency, max_quality };

struct ObjectiveHierarchy {
  std::vector<Criterion> criteria;
  std::optional<int> quality_floor;
};

ObjectiveHierarchy objective_from_token(const std::string& token);

struct SearchBounds {
  int max_fanout = 4;
  int max_paths = 2;
  std::map<std::string, int> sku_pool_cap;
  std::map<std::string, int> sku_total_cap;
  static SearchBounds from_json_text(const std::string& bounds_json);
};

// ---- plans (config.hpp:16-64) -------------------------------------------
struct Placement {
  std::string sku;
  int units = 1;
  int workers = 1;
  bool operator==(const Placement&) const = default;
};

struct NodeAssignment {
  std::string implementation;
  std::vector<Placement> placements;
  int path_count = 1;
  int fan_out() const;
  bool operator==(const NodeAssignment&) const = default;
};

struct ConfigPoint {
  std::string label;
  std::map<std::string, NodeAssignment> nodes;
  std::string identifier() const;
  std::string to_json_text() const;
  static ConfigPoint from_json_text(const std::string& text);  // = parse_config_point
};

// A config point / --pin file (config.hpp:66-117, parse_config_point):
// SchemaError("malformed config point: ...") or the per-node checks'
// messages on bad input.
ConfigPoint parse_config_point(const std::string& text);

// Substring one node contributes to ConfigPoint::identifier().
std::string assignment_token(const std::string& node_id, const NodeAssignment& a);

struct NodePlan {
  Micros wall_us = 0;
  double gpu_wh = 0.0;
  double cpu_wh = 0.0;
  double dollars = 0.0;
};

struct ConfigEstimate {
  ConfigPoint config;
  Micros latency_us = 0;
  double gpu_wh = 0.0;
  double cpu_wh = 0.0;
  double total_wh = 0.0;
  double dollars = 0.0;
  int quality = 0;
  double latency_seconds() const { return to_seconds(latency_us); }
};

// ---- the hot path --------------------------------------------------------
int chunk_capacity(double work, double min_chunk);
std::vector<double> water_fill_split(double work, double min_chunk, const std::vector<double>& speeds);
std::vector<NodeAssignment> node_options(const DagNode& node, const AgentLibrary& library,
                                         const SearchBounds& bounds);
NodePlan plan_node_execution(const DagNode& node, const NodeAssignment& a,
                             const AgentLibrary& library);
int node_quality(const DagNode& node, const Implementation& impl, int path_count);
ConfigEstimate estimate(const ConfigPoint& config, const WorkflowDag& dag,
                        const AgentLibrary& library);
bool objective_less(const ConfigEstimate& a, const ConfigEstimate& b,
                    const ObjectiveHierarchy& objective);
bool meets_quality_floor(const ConfigEstimate& e, const ObjectiveHierarchy& objective);

// GPU-backed.  The overloads without a context use this thread's own context
// on device 0 (created on first use; concurrent callers do not serialise).
// pareto_filter: stable input order, duplicates all kept (optimizer.hpp:153-171),
// evaluated on the device (loom_pareto_filter_points).
std::vector<ConfigEstimate> pareto_filter(const std::vector<ConfigEstimate>& estimates);
std::vector<ConfigEstimate> pareto_filter(const std::vector<ConfigEstimate>& estimates, loom_ctx* ctx);
ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds);
ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds,
                                 loom_ctx* ctx, std::optional<Micros> latency_slo_us = std::nullopt);
// Multi-GPU: the plan space sharded over the group's GPUs (loom_group_create /
// loom_group_create_rank); every rank of the group returns the same estimate.
ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds,
                                 loom_group* group, std::optional<Micros> latency_slo_us = std::nullopt);

// greedy_search (optimizer.hpp:227-291) on the GPU: node-local seeds on the
// host, every sweep's per-node argmin on the device (one CTA).
ConfigEstimate greedy_search(const WorkflowDag& dag, const AgentLibrary& library, const ObjectiveHierarchy& objective,
                             const SearchBounds& bounds, int max_sweeps = 10);
ConfigEstimate greedy_search(const WorkflowDag& dag, const AgentLibrary& library, const ObjectiveHierarchy& objective,
                             const SearchBounds& bounds, int max_sweeps, loom_ctx* ctx);

// ---- lowering: the flat tables the kernels read --------------------------
struct LoweredProblem {
  std::vector<std::string> node_ids;                 // dag.nodes order
  std::vector<std::vector<NodeAssignment>> options;  // node_options per node (empty when shared_options is used)
  // node_options per node shared with a LowerCache (batch lowering): the
  // option list of a node does not depend on its work, only the numbers do
  std::vector<std::shared_ptr<const std::vector<NodeAssignment>>> shared_options;
  const std::vector<NodeAssignment>& node_opts(int i) const {
    return shared_options.empty() ? options[i] : *shared_options[i];
  }
  std::vector<int32_t> radix;
  std::vector<int64_t> wall_us;
  std::vector<double> gpu_wh, cpu_wh, dollars;       // already x path_count
  std::vector<int32_t> quality, lexrank;
  std::vector<uint64_t> lex_weight;
  std::vector<int32_t> edge_from, edge_to;
  std::vector<int32_t> sweep_order;  // topological_order (workflow.hpp:467-498): id-ordered Kahn
  uint64_t total = 0;  // 0 for an empty space
  loom_problem view() const;
  ConfigPoint config_of(uint64_t plan_index) const;
};

LoweredProblem lower(const WorkflowDag& dag, const AgentLibrary& library, const SearchBounds& bounds);

// Option sets memoised across the DAGs of a batch (one library, one set of
// bounds, one thread): per node, the options, their identifier ranks and how
// each option's numbers are computed depend only on the node's capability,
// fan-out cap, path cap and which CPU+GPU splits are possible, so a hit costs
// the per-option numbers alone.  The result equals lower() exactly.
class LowerCache;
std::shared_ptr<LowerCache> make_lower_cache();
LoweredProblem lower(const WorkflowDag& dag, const AgentLibrary& library, const SearchBounds& bounds,
                     LowerCache& cache);

}  // namespace loom
