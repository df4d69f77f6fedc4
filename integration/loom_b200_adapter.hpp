// loom_b200_adapter.hpp -- the binding a reference maintainer adds to use the
// B200 search from inside the reference code base.
//
// Include it AFTER the reference's own headers ("loom/loom.hpp"), link
// libloom_b200.so, and replace
//
//     loom::exhaustive_search(dag, library, objective, bounds)   // optimizer.hpp:173-188
//
// with
//
//     loom_b200_adapter::exhaustive_search(dag, library, objective, bounds)
//
// (e.g. in tools/loom_main.cpp:140-146, the `--search exhaustive` branch).
// The adapter lowers with the reference's OWN node_options
// (optimizer.hpp:51-107) and plan_node_execution (chunking.hpp:85-184), so the
// tables the GPU searches are produced by the reference itself; it then calls
// the C ABI (include/loom_b200.h), decodes the winning index through the same
// option lists and returns the reference's own estimate() of that ConfigPoint.
// Errors are raised as the reference's exception types with the reference's
// message (optimizer.hpp:184-186).
#pragma once

#include <algorithm>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "loom_b200.h"

namespace loom_b200_adapter {

struct Lowered {
  std::vector<std::string> ids;
  std::vector<std::vector<loom::NodeAssignment>> options;
  std::vector<int32_t> radix, quality, lexrank, efrom, eto;
  std::vector<int64_t> wall;
  std::vector<double> gpu, cpu, dol;
  std::vector<uint64_t> weight;
  uint64_t total = 0;

  loom_problem view() const {
    loom_problem p{};
    p.n_nodes = static_cast<int32_t>(radix.size());
    p.n_edges = static_cast<int32_t>(efrom.size());
    p.radix = radix.data();
    p.wall_us = wall.data();
    p.gpu_wh = gpu.data();
    p.cpu_wh = cpu.data();
    p.dollars = dol.data();
    p.quality = quality.data();
    p.lexrank = lexrank.data();
    p.lex_weight = weight.data();
    p.edge_from = efrom.data();
    p.edge_to = eto.data();
    return p;
  }

  loom::ConfigPoint config_of(uint64_t index) const {
    loom::ConfigPoint c;
    for (std::size_t i = radix.size(); i-- > 0;) {
      c.nodes[ids[i]] = options[i][index % static_cast<uint64_t>(radix[i])];
      index /= static_cast<uint64_t>(radix[i]);
    }
    return c;
  }
};

// Identifier substring of one node (the part ConfigPoint::identifier()
// contributes for it, config.hpp:49-61), produced by the reference itself.
inline std::string token(const std::string& id, const loom::NodeAssignment& a) {
  loom::ConfigPoint one;
  one.nodes[id] = a;
  return one.identifier();
}

inline Lowered lower(const loom::WorkflowDag& dag, const loom::AgentLibrary& library,
                     const loom::SearchBounds& bounds) {
  Lowered L;
  std::map<std::string, int> index;
  for (const auto& n : dag.nodes) {
    index[n.id] = static_cast<int>(L.ids.size());
    L.ids.push_back(n.id);
  }
  for (const auto& e : dag.edges) {
    L.efrom.push_back(index.at(e.from));
    L.eto.push_back(index.at(e.to));
  }
  L.total = dag.nodes.empty() ? 0 : 1;
  for (const auto& node : dag.nodes) {
    auto opts = loom::node_options(node, library, bounds);
    L.radix.push_back(static_cast<int32_t>(opts.size()));
    L.total *= opts.size();
    std::vector<std::string> toks;
    for (const auto& a : opts) {
      const loom::NodePlan plan = loom::plan_node_execution(node, a, library);
      L.wall.push_back(plan.wall_us);
      L.gpu.push_back(plan.gpu_wh * a.path_count);  // estimator.hpp:51-53
      L.cpu.push_back(plan.cpu_wh * a.path_count);
      L.dol.push_back(plan.dollars * a.path_count);
      L.quality.push_back(loom::node_quality(node, *library.implementation(a.implementation), a.path_count));
      toks.push_back(token(node.id, a));
      // the identifier tie-break by per-node rank is exact only when the ';'
      // that ends a node's substring is its only one (as loom::lower checks)
      if (toks.back().find(';') + 1 != toks.back().size())
        throw loom::InvalidConfigError("name in '" + toks.back() + "' contains ';', which breaks identifier ordering");
    }
    std::vector<int> order(opts.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return toks[x] < toks[y]; });
    std::vector<int32_t> rank(opts.size());
    for (std::size_t k = 0; k < order.size(); ++k) rank[order[k]] = static_cast<int32_t>(k);
    L.lexrank.insert(L.lexrank.end(), rank.begin(), rank.end());
    L.options.push_back(std::move(opts));
  }
  // mixed-radix weights in std::map (sorted node id) order
  std::vector<int> by_id(L.ids.size());
  std::iota(by_id.begin(), by_id.end(), 0);
  std::sort(by_id.begin(), by_id.end(), [&](int a, int b) { return L.ids[a] < L.ids[b]; });
  L.weight.assign(L.ids.size(), 0);
  uint64_t w = 1;
  for (std::size_t k = by_id.size(); k-- > 0;) {
    L.weight[by_id[k]] = w;
    w *= static_cast<uint64_t>(std::max<int32_t>(1, L.radix[by_id[k]]));
  }
  return L;
}

inline loom_objective objective_of(const loom::ObjectiveHierarchy& h) {
  loom_objective o{};
  // a repeated criterion never changes objective_less (estimator.hpp:93-116):
  // keep each criterion's first occurrence, which leaves at most four
  int n = 0;
  for (const loom::Criterion c : h.criteria) {
    const int32_t v = static_cast<int32_t>(c);  // same enumerator order (workflow.hpp:67)
    if (std::find(o.criteria, o.criteria + n, v) == o.criteria + n) o.criteria[n++] = v;
  }
  o.n_criteria = n;
  if (h.quality_floor) {
    o.has_quality_floor = 1;
    o.quality_floor = *h.quality_floor;
  }
  return o;
}

// Drop-in for loom::exhaustive_search (optimizer.hpp:173-188).
inline loom::ConfigEstimate exhaustive_search(const loom::WorkflowDag& dag, const loom::AgentLibrary& library,
                                              const loom::ObjectiveHierarchy& objective,
                                              const loom::SearchBounds& bounds, loom_ctx* ctx = nullptr) {
  if (!ctx) {
    // created once, thread-safely (function-local static initialisation)
    static loom_ctx* const shared = [] {
      loom_ctx* c = nullptr;
      if (loom_ctx_create(0, nullptr, &c) != LOOM_OK) throw std::runtime_error(loom_last_error());
      return c;
    }();
    ctx = shared;
  }
  const Lowered L = lower(dag, library, bounds);
  if (L.total == 0) throw loom::NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
  const loom_problem p = L.view();
  const loom_objective o = objective_of(objective);
  loom_winner w{};
  const int rc = loom_search_argmin(ctx, &p, &o, 0, L.total, &w);
  if (rc == LOOM_INFEASIBLE)
    throw loom::NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
  if (rc != LOOM_OK) throw std::runtime_error(loom_last_error());
  return loom::estimate(L.config_of(w.plan_index), dag, library);  // the reference's own estimate
}

}  // namespace loom_b200_adapter
