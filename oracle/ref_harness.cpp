// ORACLE TEST INFRASTRUCTURE -- NOT PRODUCT CODE.
//
// A thin harness around the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/loom/*.hpp), compiled from the sources where
// they lie by oracle/Makefile into oracle/_ref/ (git-ignored).  Nothing here
// re-implements the reference: every number it prints comes from a call into
// the reference's own functions:
//
//   planner      loom::LexiconPlanner::plan          planner.hpp:237
//   options      loom::node_options                  optimizer.hpp:51-107
//   node plans   loom::plan_node_execution           chunking.hpp:85-184
//   estimate     loom::estimate                      estimator.hpp:43-78
//   order        loom::objective_less                estimator.hpp:93-116
//   floor        loom::meets_quality_floor           estimator.hpp:118-121
//   search       loom::exhaustive_search             optimizer.hpp:173-188
//   greedy       loom::greedy_search                 optimizer.hpp:227-291
//   frontier     loom::pareto_filter                 optimizer.hpp:153-171
//
// The "range driver" (loomref_range_argmin) is the CPU baseline used by
// bench.py --impl reference: it decodes a plan index range into ConfigPoints
// exactly like ConfigEnumerator::next (optimizer.hpp:131-143, node 0 most
// significant) and runs the reference estimate / meets_quality_floor /
// objective_less on T host threads, then reduces the per-thread winners with
// the same objective_less.  SPEC.md:293-294 allows concurrent evaluation as
// long as the selection equals the sequential one, which the strict total
// order guarantees.
//
// The latency SLO used by config 3 is an extension the reference does not
// have: it is applied here as an extra feasibility test
// next to meets_quality_floor, nothing else changes.
//
// Exported C ABI (used via ctypes by tests/ and bench.py's reference arm):
//   loomref_plan, loomref_search, loomref_lower, loomref_enumerate,
//   loomref_pareto, loomref_range_argmin, loomref_free.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "loom/loom.hpp"

using nlohmann::json;

namespace {

struct Objective {
  loom::ObjectiveHierarchy hierarchy;
  std::optional<loom::Micros> latency_slo_us;
};

Objective parse_objective(const json& j) {
  Objective o;
  if (j.contains("criteria")) {
    for (const auto& c : j.at("criteria")) {
      const std::string s = c.get<std::string>();
      if (s == "min_cost_dollars") o.hierarchy.criteria.push_back(loom::Criterion::min_cost_dollars);
      else if (s == "min_energy") o.hierarchy.criteria.push_back(loom::Criterion::min_energy);
      else if (s == "min_latency") o.hierarchy.criteria.push_back(loom::Criterion::min_latency);
      else if (s == "max_quality") o.hierarchy.criteria.push_back(loom::Criterion::max_quality);
      else throw loom::SchemaError("unknown criterion '" + s + "'");
    }
  } else {
    o.hierarchy = loom::objective_from_token(j.at("constraint").get<std::string>());
  }
  if (j.contains("quality_floor") && !j.at("quality_floor").is_null())
    o.hierarchy.quality_floor = j.at("quality_floor").get<int>();
  if (j.contains("latency_slo_us") && !j.at("latency_slo_us").is_null())
    o.latency_slo_us = j.at("latency_slo_us").get<std::int64_t>();
  return o;
}

loom::SearchBounds parse_bounds(const json& j) {
  loom::SearchBounds b;
  b.max_fanout = j.value("max_fanout", 4);
  b.max_paths = j.value("max_paths", 2);
  if (j.contains("sku_pool_cap"))
    b.sku_pool_cap = j.at("sku_pool_cap").get<std::map<std::string, int>>();
  if (j.contains("sku_total_cap"))
    b.sku_total_cap = j.at("sku_total_cap").get<std::map<std::string, int>>();
  return b;
}

struct Problem {
  loom::WorkflowDag dag;
  loom::AgentLibrary library;
  loom::SearchBounds bounds;
};

Problem load_problem(const char* dag_json, const char* lib_json, const char* bounds_json) {
  Problem p;
  p.dag = json::parse(dag_json).get<loom::WorkflowDag>();
  p.library = loom::AgentLibrary::from_json(json::parse(lib_json));
  p.library.freeze();
  p.bounds = parse_bounds(json::parse(bounds_json));
  return p;
}

json estimate_json(const loom::ConfigEstimate& e) {
  json j;
  j["identifier"] = e.config.identifier();
  j["config"] = e.config;
  j["latency_us"] = e.latency_us;
  j["gpu_wh"] = e.gpu_wh;
  j["cpu_wh"] = e.cpu_wh;
  j["total_wh"] = e.total_wh;
  j["dollars"] = e.dollars;
  j["quality"] = e.quality;
  return j;
}

char* dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

int fail(const std::exception& e, char** out) {
  json j;
  const auto* le = dynamic_cast<const loom::Error*>(&e);
  j["error"] = le ? le->code() : std::string("internal");
  j["message"] = e.what();
  *out = dup(j.dump());
  return le ? static_cast<int>(le->category()) : 1;
}

bool feasible(const loom::ConfigEstimate& e, const Objective& o) {
  if (!loom::meets_quality_floor(e, o.hierarchy)) return false;
  if (o.latency_slo_us && e.latency_us > *o.latency_slo_us) return false;
  return true;
}

// Mixed-radix decoding of a plan index in ConfigEnumerator order
// (optimizer.hpp:136-141: last node fastest).
std::vector<std::size_t> decode(std::uint64_t index, const std::vector<std::size_t>& radix) {
  std::vector<std::size_t> d(radix.size(), 0);
  for (std::size_t i = radix.size(); i-- > 0;) {
    d[i] = static_cast<std::size_t>(index % radix[i]);
    index /= radix[i];
  }
  return d;
}

struct Options {
  std::vector<std::string> ids;
  std::vector<std::vector<loom::NodeAssignment>> opts;
  std::vector<std::size_t> radix;
  std::uint64_t total = 0;
};

Options build_options(const Problem& p) {
  Options o;
  o.total = p.dag.nodes.empty() ? 0 : 1;
  for (const auto& n : p.dag.nodes) {
    o.ids.push_back(n.id);
    o.opts.push_back(loom::node_options(n, p.library, p.bounds));
    o.radix.push_back(o.opts.back().size());
    o.total *= o.opts.back().size();
  }
  return o;
}

}  // namespace

extern "C" {

void loomref_free(char* p) { std::free(p); }

// Reference planner: job spec + library + lexicon -> dag.json text.
int loomref_plan(const char* spec_json, const char* lib_json, const char* lexicon_json, char** out) {
  try {
    const loom::JobSpec spec = loom::parse_job_spec(spec_json);
    loom::AgentLibrary library = loom::AgentLibrary::from_json(json::parse(lib_json));
    library.freeze();
    const auto lexicon = loom::CapabilityLexicon::from_json(json::parse(lexicon_json));
    const loom::WorkflowDag dag = loom::LexiconPlanner{}.plan(spec, lexicon, library);
    json j = dag;
    j["objective"] = {{"constraint", spec.constraint_token}};
    if (spec.objective.quality_floor) j["objective"]["quality_floor"] = *spec.objective.quality_floor;
    j["library"] = library.to_json();
    *out = dup(j.dump(1));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

// Reference exhaustive_search (or greedy_search) -> selected estimate JSON.
// With a latency SLO the sequential loop of exhaustive_search is re-run with
// the extra feasibility test (the reference has no SLO).
int loomref_search(const char* dag_json, const char* lib_json, const char* objective_json,
                   const char* bounds_json, const char* mode, char** out) {
  try {
    const Problem p = load_problem(dag_json, lib_json, bounds_json);
    const Objective o = parse_objective(json::parse(objective_json));
    loom::ConfigEstimate best;
    const std::string m = mode ? mode : "exhaustive";
    if (m == "greedy") {
      best = loom::greedy_search(p.dag, p.library, o.hierarchy, p.bounds);
    } else if (!o.latency_slo_us) {
      best = loom::exhaustive_search(p.dag, p.library, o.hierarchy, p.bounds);
    } else {
      loom::ConfigEnumerator stream(p.dag, p.library, p.bounds);
      std::optional<loom::ConfigEstimate> found;
      while (auto config = stream.next()) {
        loom::ConfigEstimate e = loom::estimate(*config, p.dag, p.library);
        if (!feasible(e, o)) continue;
        if (!found || loom::objective_less(e, *found, o.hierarchy)) found = std::move(e);
      }
      if (!found)
        throw loom::NoFeasibleConfigError("no configuration satisfies the quality floor and bounds");
      best = *found;
    }
    *out = dup(estimate_json(best).dump());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

// Per-node option lists (node_options order) and the per-option node plan
// (plan_node_execution) plus node_quality: the tables the B200 build lowers to.
int loomref_lower(const char* dag_json, const char* lib_json, const char* bounds_json, char** out) {
  try {
    const Problem p = load_problem(dag_json, lib_json, bounds_json);
    json nodes = json::array();
    std::uint64_t total = p.dag.nodes.empty() ? 0 : 1;
    for (const auto& n : p.dag.nodes) {
      json jn;
      jn["id"] = n.id;
      json opts = json::array();
      for (const auto& a : loom::node_options(n, p.library, p.bounds)) {
        const loom::NodePlan plan = loom::plan_node_execution(n, a, p.library);
        loom::ConfigPoint one;
        one.nodes[n.id] = a;
        json jo;
        jo["assignment"] = a;
        jo["identifier"] = one.identifier();
        jo["wall_us"] = plan.wall_us;
        jo["gpu_wh"] = plan.gpu_wh;
        jo["cpu_wh"] = plan.cpu_wh;
        jo["dollars"] = plan.dollars;
        jo["path_count"] = a.path_count;
        jo["quality"] = loom::node_quality(n, *p.library.implementation(a.implementation), a.path_count);
        opts.push_back(jo);
      }
      total *= opts.size();
      jn["options"] = opts;
      nodes.push_back(jn);
    }
    json j;
    j["nodes"] = nodes;
    j["total_count"] = total;
    j["topological_order"] = loom::topological_order(p.dag);
    *out = dup(j.dump());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

// Reference estimate for every plan index in [begin, end) (small ranges).
int loomref_enumerate(const char* dag_json, const char* lib_json, const char* bounds_json,
                      std::uint64_t begin, std::uint64_t end, char** out) {
  try {
    const Problem p = load_problem(dag_json, lib_json, bounds_json);
    const Options o = build_options(p);
    json rows = json::array();
    for (std::uint64_t i = begin; i < end && i < o.total; ++i) {
      const auto d = decode(i, o.radix);
      loom::ConfigPoint c;
      for (std::size_t k = 0; k < d.size(); ++k) c.nodes[o.ids[k]] = o.opts[k][d[k]];
      const auto e = loom::estimate(c, p.dag, p.library);
      rows.push_back({i, e.latency_us, e.gpu_wh, e.cpu_wh, e.total_wh, e.dollars, e.quality});
    }
    *out = dup(rows.dump());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

// pareto_filter over the estimates of all plans in enumeration order, mapped
// back to plan indices through the (unique) identifier.
int loomref_pareto(const char* dag_json, const char* lib_json, const char* bounds_json, char** out) {
  try {
    const Problem p = load_problem(dag_json, lib_json, bounds_json);
    loom::ConfigEnumerator stream(p.dag, p.library, p.bounds);
    std::vector<loom::ConfigEstimate> all;
    std::map<std::string, std::uint64_t> index_of;
    std::uint64_t i = 0;
    while (auto c = stream.next()) {
      index_of[c->identifier()] = i++;
      all.push_back(loom::estimate(*c, p.dag, p.library));
    }
    const auto kept = loom::pareto_filter(all);
    json rows = json::array();
    for (const auto& e : kept) {
      json r = estimate_json(e);
      r["plan_index"] = index_of.at(e.config.identifier());
      rows.push_back(r);
    }
    json j;
    j["total_count"] = i;
    j["frontier"] = rows;
    *out = dup(j.dump());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

// Range driver: reference estimate/feasibility/objective_less over plan
// indices [begin, end) on `threads` host threads.
int loomref_range_argmin(const char* dag_json, const char* lib_json, const char* objective_json,
                         const char* bounds_json, std::uint64_t begin, std::uint64_t end,
                         int threads, char** out) {
  try {
    const Problem p = load_problem(dag_json, lib_json, bounds_json);
    const Objective o = parse_objective(json::parse(objective_json));
    const Options opt = build_options(p);
    if (end > opt.total) end = opt.total;
    if (begin > end) begin = end;
    if (threads < 1) threads = 1;
    const std::uint64_t n = end - begin;
    std::vector<std::optional<loom::ConfigEstimate>> best(threads);
    std::vector<std::uint64_t> best_index(threads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        const std::uint64_t lo = begin + n * t / threads;
        const std::uint64_t hi = begin + n * (t + 1) / threads;
        if (lo >= hi) return;
        auto d = decode(lo, opt.radix);
        for (std::uint64_t i = lo; i < hi; ++i) {
          loom::ConfigPoint c;
          for (std::size_t k = 0; k < d.size(); ++k) c.nodes[opt.ids[k]] = opt.opts[k][d[k]];
          loom::ConfigEstimate e = loom::estimate(c, p.dag, p.library);
          if (feasible(e, o) && (!best[t] || loom::objective_less(e, *best[t], o.hierarchy))) {
            best[t] = std::move(e);
            best_index[t] = i;
          }
          for (std::size_t k = d.size(); k-- > 0;) {  // odometer, last node fastest
            if (++d[k] < opt.radix[k]) break;
            d[k] = 0;
          }
        }
      });
    }
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int w = -1;
    for (int t = 0; t < threads; ++t)
      if (best[t] && (w < 0 || loom::objective_less(*best[t], *best[w], o.hierarchy))) w = t;
    json j;
    j["plans"] = n;
    j["seconds"] = secs;
    j["threads"] = threads;
    j["found"] = w >= 0;
    if (w >= 0) {
      j["winner"] = estimate_json(*best[w]);
      j["winner"]["plan_index"] = best_index[w];
    }
    *out = dup(j.dump());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, out);
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// CLI: loomref <cmd> <args...>  (files in, JSON on stdout)
// ---------------------------------------------------------------------------
namespace {
std::string slurp(const char* path) {
  std::ifstream in(path);
  if (!in) {
    std::fprintf(stderr, "cannot open %s\n", path);
    std::exit(2);
  }
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}
int emit(int rc, char** out) {
  std::printf("%s\n", *out);
  loomref_free(*out);
  return rc;
}
}  // namespace

#ifndef LOOMREF_NO_MAIN
int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: loomref plan SPEC LIB LEXICON\n"
                 "       loomref search DAG LIB OBJECTIVE BOUNDS [exhaustive|greedy]\n"
                 "       loomref lower DAG LIB BOUNDS\n"
                 "       loomref pareto DAG LIB BOUNDS\n"
                 "       loomref range DAG LIB OBJECTIVE BOUNDS BEGIN END THREADS\n");
    return 2;
  }
  const std::string cmd = argv[1];
  char* out = nullptr;
  if (cmd == "plan" && argc == 5)
    return emit(loomref_plan(slurp(argv[2]).c_str(), slurp(argv[3]).c_str(), slurp(argv[4]).c_str(), &out), &out);
  if (cmd == "search" && (argc == 6 || argc == 7))
    return emit(loomref_search(slurp(argv[2]).c_str(), slurp(argv[3]).c_str(), slurp(argv[4]).c_str(),
                               slurp(argv[5]).c_str(), argc == 7 ? argv[6] : "exhaustive", &out),
                &out);
  if (cmd == "lower" && argc == 5)
    return emit(loomref_lower(slurp(argv[2]).c_str(), slurp(argv[3]).c_str(), slurp(argv[4]).c_str(), &out), &out);
  if (cmd == "pareto" && argc == 5)
    return emit(loomref_pareto(slurp(argv[2]).c_str(), slurp(argv[3]).c_str(), slurp(argv[4]).c_str(), &out), &out);
  if (cmd == "range" && argc == 9)
    return emit(loomref_range_argmin(slurp(argv[2]).c_str(), slurp(argv[3]).c_str(), slurp(argv[4]).c_str(),
                                     slurp(argv[5]).c_str(), std::strtoull(argv[6], nullptr, 10),
                                     std::strtoull(argv[7], nullptr, 10), std::atoi(argv[8]), &out),
                &out);
  std::fprintf(stderr, "bad command line\n");
  return 2;
}
#endif
