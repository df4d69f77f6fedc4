// Host half of the C ABI (no device code): errors, problem validation, the
// exact single-plan estimate used to fill winners, the objective order over
// winner records (multi-rank combine), reference-format JSON lowering, and the
// drop-in entry points loom::exhaustive_search / loom_exhaustive_search_json.
#include <algorithm>
#include <functional>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "json.hpp"
#include "loom_b200.h"
#include "loom_b200/loom.hpp"

namespace loomi {

thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }

int fail(int status, const std::string& msg) {
  g_error = msg;
  return status;
}

int check_problem(const loom_problem* p, uint64_t* total) {
  if (!p) return fail(LOOM_INVALID, "InvalidConfigError: null problem");
  if (p->n_nodes < 0 || p->n_edges < 0) return fail(LOOM_INVALID, "InvalidConfigError: negative sizes");
  if (p->n_nodes == 0) {
    *total = 0;  // empty dag: no configs (optimizer.hpp:120)
    return LOOM_OK;
  }
  if (!p->radix) return fail(LOOM_INVALID, "InvalidConfigError: null radix");
  uint64_t t = 1;
  int64_t n_opts = 0;
  for (int i = 0; i < p->n_nodes; ++i) {
    if (p->radix[i] < 0) return fail(LOOM_INVALID, "InvalidConfigError: negative radix");
    n_opts += p->radix[i];
    if (p->radix[i] == 0) t = 0;
    else if (t && t > UINT64_MAX / static_cast<uint64_t>(p->radix[i]))
      return fail(LOOM_INVALID, "InvalidConfigError: plan space exceeds 2^64 plans");
    else t *= static_cast<uint64_t>(p->radix[i]);
  }
  if (n_opts && (!p->wall_us || !p->gpu_wh || !p->cpu_wh || !p->dollars || !p->quality || !p->lexrank))
    return fail(LOOM_INVALID, "InvalidConfigError: null option table");
  if (!p->lex_weight) return fail(LOOM_INVALID, "InvalidConfigError: null lex_weight");
  // The reference's library rejects negative watts, rates and throughputs, so
  // lowered values are finite and >= 0; the kernels' bounds rely on it (raw
  // C-ABI callers are held to the same contract).
  for (int64_t k = 0; k < n_opts; ++k) {
    const double v[3] = {p->gpu_wh[k], p->cpu_wh[k], p->dollars[k]};
    for (double x : v)
      if (!(x >= 0.0) || x == HUGE_VAL)
        return fail(LOOM_INVALID, "InvalidConfigError: option energy / dollars must be finite and >= 0");
    if (p->wall_us[k] < 0) return fail(LOOM_INVALID, "InvalidConfigError: negative wall");
  }
  if (p->n_edges && (!p->edge_from || !p->edge_to)) return fail(LOOM_INVALID, "InvalidConfigError: null edges");
  for (int e = 0; e < p->n_edges; ++e)
    if (p->edge_from[e] < 0 || p->edge_from[e] >= p->n_nodes || p->edge_to[e] < 0 || p->edge_to[e] >= p->n_nodes)
      return fail(LOOM_INVALID, "CycleError: edge references unknown node");
  *total = t;
  return LOOM_OK;
}

namespace {

std::vector<int> topo(const loom_problem* p) {
  const int n = p->n_nodes;
  std::vector<int> indeg(n, 0), order;
  std::vector<std::vector<int>> succ(n);
  for (int e = 0; e < p->n_edges; ++e) {
    succ[p->edge_from[e]].push_back(p->edge_to[e]);
    ++indeg[p->edge_to[e]];
  }
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) order.push_back(i);
  for (std::size_t k = 0; k < order.size(); ++k)
    for (int s : succ[order[k]])
      if (--indeg[s] == 0) order.push_back(s);
  return order;
}

}  // namespace

// fill_winner for dags of <= 64 nodes (every batch job): no allocations;
// predecessor masks give the critical path in any topological order (max
// and + over int64 are exact, so the order does not change the result).
static int fill_winner_small(const loom_problem* p, loom_winner* w) {
  const int n = p->n_nodes;
  int opt[64];
  uint64_t x = w->plan_index;
  int off = 0;
  for (int i = 0; i < n; ++i) off += p->radix[i];
  for (int i = n - 1; i >= 0; --i) {
    off -= p->radix[i];
    opt[i] = off + static_cast<int>(x % static_cast<uint64_t>(p->radix[i]));
    x /= static_cast<uint64_t>(p->radix[i]);
  }
  // estimator.hpp:46-67: left folds in dag.nodes order starting from 0.0
  double gpu = 0.0, cpu = 0.0, dol = 0.0;
  int q = INT_MAX;
  uint64_t lex = 0;
  for (int i = 0; i < n; ++i) {
    gpu += p->gpu_wh[opt[i]];
    cpu += p->cpu_wh[opt[i]];
    dol += p->dollars[opt[i]];
    q = std::min(q, p->quality[opt[i]]);
    lex += static_cast<uint64_t>(p->lexrank[opt[i]]) * p->lex_weight[i];
  }
  // estimator.hpp:69-76: finish(v) = max over in-edges of finish(u) + wall(v)
  uint64_t pred[64] = {};
  for (int e = 0; e < p->n_edges; ++e) pred[p->edge_to[e]] |= uint64_t(1) << p->edge_from[e];
  int64_t fin[64];
  int64_t lat = 0;
  uint64_t done = 0;
  const uint64_t all = n == 64 ? ~uint64_t(0) : (uint64_t(1) << n) - 1;
  while (done != all) {
    const uint64_t before = done;
    for (int v = 0; v < n; ++v) {
      if ((done >> v & 1) || (pred[v] & ~done)) continue;
      int64_t s = 0;
      for (uint64_t m = pred[v]; m; m &= m - 1) s = std::max(s, fin[__builtin_ctzll(m)]);
      fin[v] = s + p->wall_us[opt[v]];
      lat = std::max(lat, fin[v]);
      done |= uint64_t(1) << v;
    }
    if (done == before) return fail(LOOM_INVALID, "CycleError: dag has a cycle");
  }
  w->latency_us = lat;
  w->gpu_wh = gpu;
  w->cpu_wh = cpu;
  w->total_wh = gpu + cpu;
  w->dollars = dol;
  w->quality = q;
  w->lexkey = lex;
  w->found = 1;
  return LOOM_OK;
}

int fill_winner(const loom_problem* p, loom_winner* w) {
  uint64_t total = 0;
  if (int rc = check_problem(p, &total)) return rc;
  if (w->plan_index >= total) return fail(LOOM_INVALID, "InvalidConfigError: plan index out of range");
  const int n = p->n_nodes;
  if (n <= 64) return fill_winner_small(p, w);
  std::vector<int> opt(n), off(n + 1, 0);
  for (int i = 0; i < n; ++i) off[i + 1] = off[i] + p->radix[i];
  uint64_t x = w->plan_index;
  for (int i = n - 1; i >= 0; --i) {
    opt[i] = off[i] + static_cast<int>(x % static_cast<uint64_t>(p->radix[i]));
    x /= static_cast<uint64_t>(p->radix[i]);
  }
  // estimator.hpp:46-67: left folds in dag.nodes order starting from 0.0
  double gpu = 0.0, cpu = 0.0, dol = 0.0;
  int q = INT_MAX;
  uint64_t lex = 0;
  for (int i = 0; i < n; ++i) {
    gpu += p->gpu_wh[opt[i]];
    cpu += p->cpu_wh[opt[i]];
    dol += p->dollars[opt[i]];
    q = std::min(q, p->quality[opt[i]]);
    lex += static_cast<uint64_t>(p->lexrank[opt[i]]) * p->lex_weight[i];
  }
  // estimator.hpp:69-76: finish(v) = max over in-edges of finish(u) + wall(v)
  std::vector<std::vector<int>> preds(n);
  for (int e = 0; e < p->n_edges; ++e) preds[p->edge_to[e]].push_back(p->edge_from[e]);
  const std::vector<int> order = topo(p);
  if (static_cast<int>(order.size()) != n) return fail(LOOM_INVALID, "CycleError: dag has a cycle");
  std::vector<int64_t> fin(n, 0);
  int64_t lat = 0;
  for (int v : order) {
    int64_t s = 0;
    for (int u : preds[v]) s = std::max(s, fin[u]);
    fin[v] = s + p->wall_us[opt[v]];
    lat = std::max(lat, fin[v]);
  }
  w->latency_us = lat;
  w->gpu_wh = gpu;
  w->cpu_wh = cpu;
  w->total_wh = gpu + cpu;
  w->dollars = dol;
  w->quality = q;
  w->lexkey = lex;
  w->found = 1;
  return LOOM_OK;
}

}  // namespace loomi

namespace {

std::int64_t quantize(double v) { return static_cast<std::int64_t>(std::llround(v * 1e9)); }

int status_of(const loom::Error& e) {
  if (e.code() == "NoFeasibleConfigError") return LOOM_INFEASIBLE;
  return LOOM_INVALID;
}

loom_objective to_objective(const loom::ObjectiveHierarchy& h, std::optional<loom::Micros> slo) {
  loom_objective o;
  std::memset(&o, 0, sizeof o);
  // objective_less (estimator.hpp:93-116) accepts any criteria list; a repeat
  // of an earlier criterion compares values already found equal, so dropping
  // it (keeping the first occurrence) leaves the order unchanged and at most
  // the four distinct criteria remain
  int n = 0;
  for (const loom::Criterion c : h.criteria) {
    int32_t v = 0;
    switch (c) {
      case loom::Criterion::min_cost_dollars: v = LOOM_MIN_COST_DOLLARS; break;
      case loom::Criterion::min_energy: v = LOOM_MIN_ENERGY; break;
      case loom::Criterion::min_latency: v = LOOM_MIN_LATENCY; break;
      case loom::Criterion::max_quality: v = LOOM_MAX_QUALITY; break;
    }
    if (std::find(o.criteria, o.criteria + n, v) == o.criteria + n) o.criteria[n++] = v;
  }
  o.n_criteria = n;
  if (h.quality_floor) {
    o.has_quality_floor = 1;
    o.quality_floor = *h.quality_floor;
  }
  if (slo) {
    o.has_latency_slo = 1;
    o.latency_slo_us = *slo;
  }
  return o;
}

struct ParsedObjective {
  loom::ObjectiveHierarchy hierarchy;
  std::optional<loom::Micros> slo;
};

ParsedObjective parse_objective_value(const loomjson::Value& j);

ParsedObjective parse_objective_json(const std::string& text) {
  loomjson::Value j;
  try {
    j = loomjson::parse(text);
  } catch (const loomjson::ParseError& e) {
    throw loom::SchemaError(std::string("malformed objective: ") + e.what());
  }
  return parse_objective_value(j);
}

// One objective, or (batch calls) a JSON array of per-job objectives.
std::vector<loom_objective> parse_objectives_json(const std::string& text, int32_t n) {
  loomjson::Value j;
  try {
    j = loomjson::parse(text);
  } catch (const loomjson::ParseError& e) {
    throw loom::SchemaError(std::string("malformed objective: ") + e.what());
  }
  std::vector<loom_objective> out;
  if (!j.is_array()) {
    const ParsedObjective p = parse_objective_value(j);
    out.assign(static_cast<size_t>(std::max(n, 1)), to_objective(p.hierarchy, p.slo));
    return out;
  }
  if (static_cast<int64_t>(j.size()) != n)
    throw loom::SchemaError("objective array has " + std::to_string(j.size()) + " entries for " +
                            std::to_string(n) + " jobs");
  for (const auto& v : j.items()) {
    const ParsedObjective p = parse_objective_value(v);
    out.push_back(to_objective(p.hierarchy, p.slo));
  }
  return out;
}

ParsedObjective parse_objective_value(const loomjson::Value& j) {
  ParsedObjective out;
  try {
    if (const loomjson::Value* c = j.find("criteria")) {
      for (const auto& v : c->items()) {
        const std::string& s = v.as_string("criteria");
        if (s == "min_cost_dollars") out.hierarchy.criteria.push_back(loom::Criterion::min_cost_dollars);
        else if (s == "min_energy") out.hierarchy.criteria.push_back(loom::Criterion::min_energy);
        else if (s == "min_latency") out.hierarchy.criteria.push_back(loom::Criterion::min_latency);
        else if (s == "max_quality") out.hierarchy.criteria.push_back(loom::Criterion::max_quality);
        else throw loom::SchemaError("unknown criterion '" + s + "'");
      }
    } else {
      out.hierarchy = loom::objective_from_token(j.at("constraint").as_string("constraint"));
    }
    if (const loomjson::Value* f = j.find("quality_floor"); f && !f->is_null())
      out.hierarchy.quality_floor = static_cast<int>(f->as_int("quality_floor"));
    if (const loomjson::Value* s = j.find("latency_slo_us"); s && !s->is_null())
      out.slo = s->as_int("latency_slo_us");
  } catch (const loomjson::ParseError& e) {
    throw loom::SchemaError(std::string("objective: ") + e.what());
  }
  return out;
}

int copy_out(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
    if (n < s.size()) return loomi::fail(LOOM_INVALID, "InvalidConfigError: output buffer too small");
  }
  return LOOM_OK;
}

std::string estimate_json(const loom::ConfigEstimate& e, uint64_t plan_index, uint64_t plans) {
  using loomjson::Value;
  Value v = Value::make_object();
  v.set("identifier", Value::make_string(e.config.identifier()));
  v.set("config", loomjson::parse(e.config.to_json_text()));
  v.set("latency_us", Value::make_int(e.latency_us));
  v.set("gpu_wh", Value::make_real(e.gpu_wh));
  v.set("cpu_wh", Value::make_real(e.cpu_wh));
  v.set("total_wh", Value::make_real(e.total_wh));
  v.set("dollars", Value::make_real(e.dollars));
  v.set("quality", Value::make_int(e.quality));
  v.set("plan_index", Value::make_int(static_cast<int64_t>(plan_index)));
  v.set("plans", Value::make_int(static_cast<int64_t>(plans)));
  return v.dump();
}

std::string error_json(const std::string& what) {
  using loomjson::Value;
  Value v = Value::make_object();
  const auto colon = what.find(':');
  v.set("error", Value::make_string(colon == std::string::npos ? "Error" : what.substr(0, colon)));
  v.set("message", Value::make_string(what));
  return v.dump();
}

}  // namespace

struct loom_lowered {
  loom::LoweredProblem L;
  loom_problem view;
};

namespace loom {

// This thread's context for the overloads without one (device 0, own
// stream): a loom_ctx is re-entrant per thread, so callers on different
// threads run concurrently instead of queueing on one shared context.
namespace {
loom_ctx* thread_ctx() {
  struct Holder {
    loom_ctx* c = nullptr;
    ~Holder() {
      if (c) loom_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c && loom_ctx_create(0, nullptr, &h.c) != LOOM_OK) throw std::runtime_error(loom_last_error());
  return h.c;
}

ConfigEstimate search_lowered_one(const LoweredProblem& L, const WorkflowDag& dag, const AgentLibrary& library,
                                  const loom_objective& obj,
                                  const std::function<int(const loom_problem*, loom_winner*)>& search) {
  if (L.total == 0) throw NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
  const loom_problem view = L.view();
  loom_winner w;
  const int rc = search(&view, &w);
  if (rc == LOOM_INFEASIBLE) throw NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
  if (rc != LOOM_OK) throw std::runtime_error(loom_last_error());
  // The selected plan is re-estimated with the reference arithmetic on the
  // reference types; the GPU's latency and identifier rank must agree.
  ConfigEstimate e = estimate(L.config_of(w.plan_index), dag, library);
  if (e.latency_us != w.latency_us || e.gpu_wh != w.gpu_wh || e.dollars != w.dollars)
    throw std::runtime_error("DeviceError: GPU winner disagrees with host estimate");
  return e;
}
}  // namespace

ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds) {
  return exhaustive_search(dag, library, objective, bounds, thread_ctx());
}

ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds, loom_ctx* ctx,
                                 std::optional<Micros> latency_slo_us) {
  const LoweredProblem L = lower(dag, library, bounds);
  const loom_objective obj = to_objective(objective, latency_slo_us);
  return search_lowered_one(L, dag, library, obj, [&](const loom_problem* p, loom_winner* w) {
    return loom_search_argmin(ctx, p, &obj, 0, L.total, w);
  });
}

ConfigEstimate exhaustive_search(const WorkflowDag& dag, const AgentLibrary& library,
                                 const ObjectiveHierarchy& objective, const SearchBounds& bounds, loom_group* group,
                                 std::optional<Micros> latency_slo_us) {
  const LoweredProblem L = lower(dag, library, bounds);
  const loom_objective obj = to_objective(objective, latency_slo_us);
  return search_lowered_one(L, dag, library, obj, [&](const loom_problem* p, loom_winner* w) {
    return loom_group_search_argmin(group, p, &obj, 0, L.total, w);
  });
}

std::vector<ConfigEstimate> pareto_filter(const std::vector<ConfigEstimate>& in) {
  return pareto_filter(in, thread_ctx());
}

std::vector<ConfigEstimate> pareto_filter(const std::vector<ConfigEstimate>& in, loom_ctx* ctx) {
  // the dominance axes only (optimizer.hpp:155-161), tagged with the input
  // position; the device marks the points no other point dominates
  std::vector<loom_point> pts(in.size());
  for (std::size_t i = 0; i < in.size(); ++i)
    pts[i] = loom_point{i, in[i].dollars, in[i].gpu_wh, in[i].latency_us, in[i].quality, 0};
  std::vector<uint8_t> keep(in.size(), 0);
  if (!in.empty() && loom_pareto_filter_points(ctx, pts.data(), pts.size(), keep.data()) != LOOM_OK)
    throw std::runtime_error(loom_last_error());
  std::vector<ConfigEstimate> kept;
  for (std::size_t i = 0; i < in.size(); ++i)
    if (keep[i]) kept.push_back(in[i]);
  return kept;
}

namespace {
// greedy_search's seeding / feasibility errors carry node ids (optimizer.hpp:232-251).
void greedy_prepare(const LoweredProblem& L, const WorkflowDag& dag, const loom_objective& o, std::vector<int32_t>& seed) {
  if (dag.nodes.empty()) throw NoFeasibleConfigError("cannot search an empty dag");
  const loom_problem view = L.view();
  seed.assign(L.radix.size(), 0);
  const int rc = loom_greedy_seed(&view, &o, seed.data());
  if (rc == LOOM_INFEASIBLE) {
    const std::string msg = loom_last_error();
    const auto at = msg.find("node #");
    const int idx = at == std::string::npos ? -1 : std::atoi(msg.c_str() + at + 6);
    const std::string id = idx >= 0 && idx < static_cast<int>(L.node_ids.size()) ? L.node_ids[idx] : "?";
    throw NoFeasibleConfigError("node '" + id + "' has no lever assignment meeting the quality floor");
  }
  if (rc != LOOM_OK) throw std::runtime_error(loom_last_error());
}
}  // namespace

ConfigEstimate greedy_search(const WorkflowDag& dag, const AgentLibrary& library, const ObjectiveHierarchy& objective,
                             const SearchBounds& bounds, int max_sweeps) {
  return greedy_search(dag, library, objective, bounds, max_sweeps, thread_ctx());
}

ConfigEstimate greedy_search(const WorkflowDag& dag, const AgentLibrary& library, const ObjectiveHierarchy& objective,
                             const SearchBounds& bounds, int max_sweeps, loom_ctx* ctx) {
  const LoweredProblem L = lower(dag, library, bounds);
  const loom_objective obj = to_objective(objective, std::nullopt);
  std::vector<int32_t> seed;
  greedy_prepare(L, dag, obj, seed);
  if (L.total == 0) throw NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
  const loom_problem view = L.view();
  loom_winner w;
  const int rc = loom_search_greedy(ctx, &view, &obj, L.sweep_order.data(), seed.data(), max_sweeps, &w);
  if (rc != LOOM_OK) throw std::runtime_error(loom_last_error());
  return estimate(L.config_of(w.plan_index), dag, library);
}

}  // namespace loom

extern "C" {

int loom_abi_version(void) { return LOOM_B200_ABI_VERSION; }

int loom_greedy_seed(const loom_problem* p, const loom_objective* o, int32_t* digits) {
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  if (!o || !digits) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  int off = 0;
  for (int i = 0; i < p->n_nodes; ++i) {
    // detail::node_local_key (optimizer.hpp:194-220): the option's own
    // contribution to each criterion; std::vector<double> ordering
    // (a fixed array in the vector's lexicographic order: at most four criteria)
    int best = -1;
    double best_key[4] = {0, 0, 0, 0};
    const int nc = std::min(o->n_criteria, 4);
    for (int k = 0; k < p->radix[i]; ++k) {
      const int x = off + k;
      if (o->has_quality_floor && p->quality[x] < o->quality_floor) continue;  // optimizer.hpp:239-247
      double key[4];
      for (int c = 0; c < nc; ++c) {
        switch (o->criteria[c]) {
          case LOOM_MIN_COST_DOLLARS: key[c] = p->dollars[x]; break;
          case LOOM_MIN_ENERGY: key[c] = p->gpu_wh[x]; break;
          case LOOM_MIN_LATENCY: key[c] = static_cast<double>(p->wall_us[x]); break;
          default: key[c] = static_cast<double>(-p->quality[x]); break;
        }
      }
      if (best < 0 || std::lexicographical_compare(key, key + nc, best_key, best_key + nc)) {
        best = k;
        std::copy(key, key + nc, best_key);
      }
    }
    if (best < 0)
      return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: node #" + std::to_string(i) +
                                              " has no lever assignment meeting the quality floor");
    digits[i] = best;
    off += p->radix[i];
  }
  return LOOM_OK;
}

int loom_lowered_sweep_order(const loom_lowered* lw, int32_t* out) {
  if (!lw || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::copy(lw->L.sweep_order.begin(), lw->L.sweep_order.end(), out);
  return LOOM_OK;
}

int loom_greedy_search_json(loom_ctx* ctx, const char* dag_json, const char* library_json, const char* objective_json,
                            const char* bounds_json, int32_t max_sweeps, char* out_json, size_t cap, size_t* needed) {
  int rc = LOOM_OK;
  std::string result;
  try {
    const loom::WorkflowDag dag = loom::WorkflowDag::from_json_text(dag_json ? dag_json : "");
    const loom::AgentLibrary lib = loom::AgentLibrary::from_json_text(library_json ? library_json : "");
    const loom::SearchBounds bounds = loom::SearchBounds::from_json_text(bounds_json ? bounds_json : "{}");
    const ParsedObjective obj = parse_objective_json(objective_json ? objective_json : "");
    const loom::LoweredProblem L = loom::lower(dag, lib, bounds);
    const loom_objective o = to_objective(obj.hierarchy, obj.slo);
    std::vector<int32_t> seed;
    loom::greedy_prepare(L, dag, o, seed);
    const loom_problem view = L.view();
    loom_winner w;
    rc = loom_search_greedy(ctx, &view, &o, L.sweep_order.data(), seed.data(), max_sweeps, &w);
    if (rc == LOOM_OK) result = estimate_json(loom::estimate(L.config_of(w.plan_index), dag, lib), w.plan_index, L.total);
    else result = error_json(loom_last_error());
  } catch (const loom::Error& e) {
    rc = loomi::fail(status_of(e), e.what());
    result = error_json(e.what());
  } catch (const std::exception& e) {
    rc = loomi::fail(LOOM_INVALID, std::string("InvalidConfigError: ") + e.what());
    result = error_json(loom_last_error());
  }
  const std::string err = loom_last_error();
  const int crc = copy_out(result, out_json, cap, needed);
  if (rc == LOOM_OK) return crc;
  loomi::set_error(err);
  return rc;
}

const char* loom_last_error(void) { return loomi::g_error.c_str(); }

int loom_problem_total(const loom_problem* p, uint64_t* total) {
  if (!total) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null out");
  return loomi::check_problem(p, total);
}

int loom_evaluate_plan(const loom_problem* p, uint64_t plan_index, loom_winner* out) {
  if (!out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null out");
  std::memset(out, 0, sizeof *out);
  out->plan_index = plan_index;
  return loomi::fill_winner(p, out);
}

int loom_latency_floor(const loom_problem* p, const loom_objective* o, int64_t* out) {
  if (!p || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  const int n = p->n_nodes;
  // per node the smallest wall among options meeting the quality floor; the
  // critical path is monotone in every wall (estimator.hpp:69-76), so these
  // walls give the smallest latency of any plan
  std::vector<int64_t> w(n, INT64_MAX);
  for (int i = 0, k = 0; i < n; ++i)
    for (int j = 0; j < p->radix[i]; ++j, ++k)
      if (!o || !o->has_quality_floor || p->quality[k] >= o->quality_floor) w[i] = std::min(w[i], p->wall_us[k]);
  for (int i = 0; i < n; ++i)
    if (w[i] == INT64_MAX)
      return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
  std::vector<int32_t> indeg(n, 0);
  std::vector<std::vector<int32_t>> succ(n);
  for (int e = 0; e < p->n_edges; ++e) {
    succ[p->edge_from[e]].push_back(p->edge_to[e]);
    ++indeg[p->edge_to[e]];
  }
  std::vector<int64_t> start(n, 0);
  std::vector<int32_t> ready;
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) ready.push_back(i);
  int64_t lat = 0;
  for (std::size_t r = 0; r < ready.size(); ++r) {
    const int v = ready[r];
    const int64_t f = start[v] + w[v];
    lat = std::max(lat, f);
    for (int s2 : succ[v]) {
      start[s2] = std::max(start[s2], f);
      if (--indeg[s2] == 0) ready.push_back(s2);
    }
  }
  if (static_cast<int>(ready.size()) != n) return loomi::fail(LOOM_INVALID, "CycleError: the dag has a cycle");
  *out = n ? lat : 0;
  return LOOM_OK;
}

int loom_winner_less(const loom_winner* a, const loom_winner* b, const loom_objective* o) {
  if (!a->found) return 0;
  if (!b->found) return 1;
  for (int i = 0; i < o->n_criteria; ++i) {
    switch (o->criteria[i]) {
      case LOOM_MIN_COST_DOLLARS:
        if (quantize(a->dollars) != quantize(b->dollars)) return quantize(a->dollars) < quantize(b->dollars);
        break;
      case LOOM_MIN_ENERGY:
        if (quantize(a->gpu_wh) != quantize(b->gpu_wh)) return quantize(a->gpu_wh) < quantize(b->gpu_wh);
        break;
      case LOOM_MIN_LATENCY:
        if (a->latency_us != b->latency_us) return a->latency_us < b->latency_us;
        break;
      default:
        if (a->quality != b->quality) return a->quality > b->quality;
        break;
    }
  }
  return a->lexkey < b->lexkey;
}

int loom_winner_reduce(const loom_winner* ws, int32_t n, const loom_objective* o, loom_winner* out) {
  if (!out || !o || (n > 0 && !ws)) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::memset(out, 0, sizeof *out);
  for (int i = 0; i < n; ++i)
    if (loom_winner_less(&ws[i], out, o)) *out = ws[i];
  if (!out->found)
    return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
  return LOOM_OK;
}

int loom_objective_parse(const char* text, loom_objective* out) {
  if (!text || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  try {
    const ParsedObjective p = parse_objective_json(text);
    *out = to_objective(p.hierarchy, p.slo);
    return LOOM_OK;
  } catch (const loom::Error& e) {
    return loomi::fail(status_of(e), e.what());
  }
}

int loom_lower(const char* dag_json, const char* library_json, const char* bounds_json, loom_lowered** out) {
  if (!out || !dag_json || !library_json || !bounds_json)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  *out = nullptr;
  try {
    auto lw = std::make_unique<loom_lowered>();
    lw->L = loom::lower(loom::WorkflowDag::from_json_text(dag_json), loom::AgentLibrary::from_json_text(library_json),
                        loom::SearchBounds::from_json_text(bounds_json));
    lw->view = lw->L.view();
    *out = lw.release();
    return LOOM_OK;
  } catch (const loom::Error& e) {
    return loomi::fail(status_of(e), e.what());
  } catch (const std::exception& e) {
    return loomi::fail(LOOM_INVALID, std::string("InvalidConfigError: ") + e.what());
  }
}

int loom_lower_batch(const char* library_json, const char* bounds_json, const char* const* dag_jsons, int32_t n,
                     int32_t threads, loom_lowered** out, int32_t* status) {
  if (!library_json || !bounds_json || (n > 0 && (!dag_jsons || !out || !status)) || n < 0)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  try {
    const loom::AgentLibrary lib = loom::AgentLibrary::from_json_text(library_json);
    const loom::SearchBounds bounds = loom::SearchBounds::from_json_text(bounds_json);
    int t = threads > 0 ? threads : loomi::host_threads();
    t = std::max(1, std::min(t, n));
    std::vector<std::string> errors(n);
    std::vector<std::thread> pool;
    for (int w = 0; w < t; ++w)
      pool.emplace_back([&, w] {
        // option sets repeat across the jobs of a batch: one cache per thread
        const auto cache = loom::make_lower_cache();
        for (int i = w; i < n; i += t) {
          out[i] = nullptr;
          try {
            auto lw = std::make_unique<loom_lowered>();
            lw->L = loom::lower(loom::WorkflowDag::from_json_text(dag_jsons[i] ? dag_jsons[i] : ""), lib, bounds,
                                *cache);
            lw->view = lw->L.view();
            out[i] = lw.release();
            status[i] = LOOM_OK;
          } catch (const loom::Error& e) {
            status[i] = status_of(e);
            errors[i] = e.what();
          } catch (const std::exception& e) {
            status[i] = LOOM_INVALID;
            errors[i] = std::string("InvalidConfigError: ") + e.what();
          }
        }
      });
    for (auto& th : pool) th.join();
    for (int i = 0; i < n; ++i)
      if (status[i] != LOOM_OK) loomi::set_error(errors[i]);
    return LOOM_OK;
  } catch (const loom::Error& e) {
    return loomi::fail(status_of(e), e.what());
  }
}

const loom_problem* loom_lowered_problem(const loom_lowered* lw) { return lw ? &lw->view : nullptr; }

namespace {
int search_lowered(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n, const loom_objective* objective,
                   bool per_job, loom_winner* out, int32_t* status);
}  // namespace

int loom_search_argmin_lowered(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n,
                               const loom_objective* objective, loom_winner* out, int32_t* status) {
  return search_lowered(ctx, lowered, n, objective, false, out, status);
}

int loom_search_argmin_lowered_each(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n,
                                    const loom_objective* objectives, loom_winner* out, int32_t* status) {
  return search_lowered(ctx, lowered, n, objectives, true, out, status);
}

namespace {
int search_lowered(loom_ctx* ctx, const loom_lowered* const* lowered, int32_t n, const loom_objective* objective,
                   bool per_job, loom_winner* out, int32_t* status) {
  if (!ctx || (n > 0 && (!lowered || !out || !status)) || !objective || n < 0)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  // only the lowered jobs go to the device; the rest keep LOOM_INVALID
  std::vector<int> idx;
  std::vector<loom_problem> probs;
  for (int i = 0; i < n; ++i) {
    std::memset(&out[i], 0, sizeof out[i]);
    status[i] = LOOM_INVALID;
    if (lowered[i]) {
      idx.push_back(i);
      probs.push_back(lowered[i]->view);
    }
  }
  const int m = static_cast<int>(idx.size());
  std::vector<loom_objective> objs(m);
  for (int k = 0; k < m; ++k) objs[k] = per_job ? objective[idx[k]] : *objective;
  std::vector<loom_winner> w(m);
  std::vector<int32_t> st(m, LOOM_OK);
  const int rc = loom_search_argmin_batch(ctx, probs.data(), objs.data(), m, w.data(), st.data());
  for (int k = 0; k < m; ++k) {
    out[idx[k]] = w[k];
    status[idx[k]] = st[k];
  }
  return rc;
}
}  // namespace

int loom_exhaustive_search_batch(loom_ctx* ctx, const char* library_json, const char* bounds_json,
                                 const char* const* dag_jsons, int32_t n, const char* objective_json,
                                 int32_t threads, loom_winner* out, int32_t* status) {
  if (!ctx || !objective_json || !library_json || !bounds_json || (n > 0 && (!out || !status || !dag_jsons)) ||
      n < 0)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::vector<loom_objective> objs;
  try {
    objs = parse_objectives_json(objective_json, n);
  } catch (const loom::Error& e) {
    return loomi::fail(status_of(e), e.what());
  }
  try {
    const loom::AgentLibrary lib = loom::AgentLibrary::from_json_text(library_json ? library_json : "");
    const loom::SearchBounds bounds = loom::SearchBounds::from_json_text(bounds_json ? bounds_json : "");
    const bool per_job = objs.size() == static_cast<size_t>(n) && n > 1;
    // Each job is lowered on the host thread that then builds and stages its
    // image (loomi::argmin_batch), with one option-set cache per thread, and
    // released on the thread that finishes it.
    std::vector<loom_lowered*> lw(n, nullptr);
    std::vector<std::string> errors(n);
    std::vector<std::shared_ptr<loom::LowerCache>> caches(threads > 0 ? threads : 64);
    std::vector<loom_problem> probs(n);
    std::vector<loom_objective> objv(n);
    const loomi::BatchProduce produce = [&](int j, int w, loom_problem* p, loom_objective* o) -> int {
      if (!caches[w]) caches[w] = loom::make_lower_cache();
      try {
        auto x = std::make_unique<loom_lowered>();
        x->L = loom::lower(loom::WorkflowDag::from_json_text(dag_jsons[j] ? dag_jsons[j] : ""), lib, bounds,
                           *caches[w]);
        x->view = x->L.view();
        *p = x->view;
        *o = objs[per_job ? j : 0];
        lw[j] = x.release();
        return LOOM_OK;
      } catch (const loom::Error& e) {
        errors[j] = e.what();
        return status_of(e);
      } catch (const std::exception& e) {
        errors[j] = std::string("InvalidConfigError: ") + e.what();
        return LOOM_INVALID;
      }
    };
    const loomi::BatchRetire retire = [&](int j) {
      loom_lowered_destroy(lw[j]);
      lw[j] = nullptr;
    };
    const int rc = loomi::argmin_batch(ctx, n, threads, probs.data(), objv.data(), produce, retire, out, status);
    for (loom_lowered* h : lw) loom_lowered_destroy(h);  // the jobs an early error left
    for (int i = 0; i < n; ++i)
      if (!errors[i].empty()) loomi::set_error(errors[i]);
    return rc;
  } catch (const loom::Error& e) {
    return loomi::fail(status_of(e), e.what());
  }
}

int loom_lowered_config_json(const loom_lowered* lw, uint64_t plan_index, char* buf, size_t cap, size_t* needed) {
  if (!lw) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null lowered");
  if (plan_index >= lw->L.total) return loomi::fail(LOOM_INVALID, "InvalidConfigError: plan index out of range");
  const loom::ConfigPoint c = lw->L.config_of(plan_index);
  loomjson::Value v = loomjson::parse(c.to_json_text());
  v.set("identifier", loomjson::Value::make_string(c.identifier()));
  return copy_out(v.dump(), buf, cap, needed);
}

int loom_lowered_option_json(const loom_lowered* lw, int32_t node, int32_t option, char* buf, size_t cap,
                             size_t* needed) {
  if (!lw) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null lowered");
  if (node < 0 || node >= static_cast<int>(lw->L.radix.size()) || option < 0 ||
      option >= static_cast<int>(lw->L.node_opts(node).size()))
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: option out of range");
  loom::ConfigPoint c;
  c.nodes[lw->L.node_ids[node]] = lw->L.node_opts(node)[option];
  loomjson::Value v = loomjson::parse(c.to_json_text()).at("nodes").at(lw->L.node_ids[node]);
  v.set("identifier", loomjson::Value::make_string(c.identifier()));
  return copy_out(v.dump(), buf, cap, needed);
}

void loom_lowered_destroy(loom_lowered* lw) { delete lw; }

}  // extern "C"

namespace {
// The drop-in call on JSON with the device search supplied by the caller (one
// context, or a multi-GPU group).
using SearchFn = std::function<int(const loom_problem*, const loom_objective*, uint64_t, loom_winner*)>;
int exhaustive_json(const SearchFn& search, const char* dag_json, const char* library_json,
                    const char* objective_json, const char* bounds_json, char* out_json, size_t cap,
                    size_t* needed);
}  // namespace

extern "C" {

int loom_exhaustive_search_json(loom_ctx* ctx, const char* dag_json, const char* library_json,
                                const char* objective_json, const char* bounds_json, char* out_json, size_t cap,
                                size_t* needed) {
  return exhaustive_json(
      [ctx](const loom_problem* p, const loom_objective* o, uint64_t total, loom_winner* w) {
        return loom_search_argmin(ctx, p, o, 0, total, w);
      },
      dag_json, library_json, objective_json, bounds_json, out_json, cap, needed);
}

int loom_estimate_config_json(const char* dag_json, const char* library_json, const char* config_json,
                              char* out_json, size_t cap, size_t* needed) {
  int rc = LOOM_OK;
  std::string result;
  try {
    const loom::WorkflowDag dag = loom::WorkflowDag::from_json_text(dag_json ? dag_json : "");
    const loom::AgentLibrary lib = loom::AgentLibrary::from_json_text(library_json ? library_json : "");
    const loom::ConfigPoint config = loom::parse_config_point(config_json ? config_json : "");
    for (const auto& node : dag.nodes)
      if (!config.nodes.count(node.id))
        throw loom::ValidationError("pinned_plan: missing assignment for task '" + node.id + "'");
    const loom::ConfigEstimate e = loom::estimate(config, dag, lib);
    loomjson::Value v = loomjson::parse(estimate_json(e, 0, 0));
    loomjson::Value o = loomjson::Value::make_object();
    for (const auto& [k, x] : v.members())
      if (k != "plan_index" && k != "plans") o.set(k, x);
    result = o.dump();
  } catch (const loom::Error& e) {
    rc = loomi::fail(status_of(e), e.what());
    result = error_json(e.what());
  } catch (const std::exception& e) {
    rc = loomi::fail(LOOM_INVALID, std::string("InvalidConfigError: ") + e.what());
    result = error_json(loom_last_error());
  }
  const std::string err = loom_last_error();
  const int crc = copy_out(result, out_json, cap, needed);
  if (rc == LOOM_OK) return crc;
  loomi::set_error(err);
  return rc;
}

int loom_group_exhaustive_search_json(loom_group* g, const char* dag_json, const char* library_json,
                                      const char* objective_json, const char* bounds_json, char* out_json,
                                      size_t cap, size_t* needed) {
  return exhaustive_json(
      [g](const loom_problem* p, const loom_objective* o, uint64_t total, loom_winner* w) {
        return loom_group_search_argmin(g, p, o, 0, total, w);
      },
      dag_json, library_json, objective_json, bounds_json, out_json, cap, needed);
}

}  // extern "C"

namespace {
int exhaustive_json(const SearchFn& search, const char* dag_json, const char* library_json,
                    const char* objective_json, const char* bounds_json, char* out_json, size_t cap,
                    size_t* needed) {
  int rc = LOOM_OK;
  std::string result;
  const bool trace = std::getenv("LOOM_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[loom trace] exhaustive_json %s %.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  try {
    const loom::WorkflowDag dag = loom::WorkflowDag::from_json_text(dag_json ? dag_json : "");
    const loom::AgentLibrary lib = loom::AgentLibrary::from_json_text(library_json ? library_json : "");
    const loom::SearchBounds bounds = loom::SearchBounds::from_json_text(bounds_json ? bounds_json : "{}");
    const ParsedObjective obj = parse_objective_json(objective_json ? objective_json : "");
    mark("parse");
    const loom::LoweredProblem L = loom::lower(dag, lib, bounds);
    if (L.total == 0) throw loom::NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
    const loom_problem view = L.view();
    const loom_objective o = to_objective(obj.hierarchy, obj.slo);
    mark("lower");
    loom_winner w;
    rc = search(&view, &o, L.total, &w);
    mark("search");
    if (rc == LOOM_OK) {
      const loom::ConfigEstimate e = loom::estimate(L.config_of(w.plan_index), dag, lib);
      if (e.latency_us != w.latency_us || e.gpu_wh != w.gpu_wh || e.dollars != w.dollars)
        rc = loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: GPU winner disagrees with host estimate");
      else
        result = estimate_json(e, w.plan_index, L.total);
    }
    if (rc != LOOM_OK) result = error_json(loom_last_error());
    mark("estimate + json");
  } catch (const loom::Error& e) {
    rc = loomi::fail(status_of(e), e.what());
    result = error_json(e.what());
  } catch (const std::exception& e) {
    rc = loomi::fail(LOOM_INVALID, std::string("InvalidConfigError: ") + e.what());
    result = error_json(loom_last_error());
  }
  const std::string err = loom_last_error();
  const int crc = copy_out(result, out_json, cap, needed);
  if (rc == LOOM_OK) return crc;
  loomi::set_error(err);
  return rc;
}
}  // namespace
