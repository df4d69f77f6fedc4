// GPU check of the C++ drop-in (include/loom_b200/loom.hpp) -- TEST DRIVER.
//
//   pareto   loom::pareto_filter on the reference's own test shapes:
//            test_optimizer.cpp:259-327 (the two SECTION cases; 20 random sets
//            of 100 integer-valued points in [0,5]^3 x [0,3]) and
//            acceptance.cpp:202-234 (100 sets of 60 points in [0,6]^3 x
//            [0,3]) -- heavy duplicates and ties -- against the quadratic
//            dominance oracle those tests use: same size, same order (stable
//            input order), duplicates kept, every removed point covered.
//   group    loom::exhaustive_search through a single-process multi-GPU group
//            (loom_group_create(mask)) equals the single-context call.
//
// Prints "ok <what>" lines; exits non-zero on the first mismatch.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "loom_b200/loom.hpp"

using loom::ConfigEstimate;

static ConfigEstimate make(double dollars, double wh, long long latency, int quality) {
  ConfigEstimate e;
  e.dollars = dollars;
  e.gpu_wh = wh;
  e.latency_us = latency;
  e.quality = quality;
  return e;
}

static bool dominates(const ConfigEstimate& a, const ConfigEstimate& b) {
  const bool no_worse = a.dollars <= b.dollars && a.gpu_wh <= b.gpu_wh && a.latency_us <= b.latency_us &&
                        a.quality >= b.quality;
  const bool strict = a.dollars < b.dollars || a.gpu_wh < b.gpu_wh || a.latency_us < b.latency_us ||
                      a.quality > b.quality;
  return no_worse && strict;
}

static bool same(const ConfigEstimate& a, const ConfigEstimate& b) {
  return a.dollars == b.dollars && a.gpu_wh == b.gpu_wh && a.latency_us == b.latency_us && a.quality == b.quality;
}

static int check_set(const std::vector<ConfigEstimate>& points, const char* what, int trial) {
  const auto kept = loom::pareto_filter(points);
  std::vector<ConfigEstimate> oracle;
  for (std::size_t i = 0; i < points.size(); ++i) {
    bool dominated = false;
    for (std::size_t j = 0; j < points.size(); ++j)
      if (j != i && dominates(points[j], points[i])) dominated = true;
    if (!dominated) oracle.push_back(points[i]);
  }
  if (kept.size() != oracle.size()) {
    std::printf("FAIL %s trial %d: kept %zu, oracle %zu\n", what, trial, kept.size(), oracle.size());
    return 1;
  }
  for (std::size_t i = 0; i < kept.size(); ++i)
    if (!same(kept[i], oracle[i])) {
      std::printf("FAIL %s trial %d: position %zu differs\n", what, trial, i);
      return 1;
    }
  for (const auto& p : points) {
    bool in_kept = false, covered = false;
    for (const auto& k : kept) {
      in_kept |= same(k, p);
      covered |= dominates(k, p);
    }
    if (!in_kept && !covered) {
      std::printf("FAIL %s trial %d: a removed point is not covered\n", what, trial);
      return 1;
    }
  }
  return 0;
}

static int pareto() {
  {
    const auto kept = loom::pareto_filter({make(1, 1, 1, 0), make(2, 2, 2, 0)});
    if (kept.size() != 1 || kept[0].dollars != 1) return std::puts("FAIL strict dominance"), 1;
    if (loom::pareto_filter({make(1, 2, 1, 0), make(2, 1, 1, 0)}).size() != 2) return std::puts("FAIL incomparable"), 1;
    if (!loom::pareto_filter({}).empty()) return std::puts("FAIL empty"), 1;
    const auto dup = loom::pareto_filter({make(1, 1, 1, 1), make(1, 1, 1, 1), make(2, 2, 2, 0)});
    if (dup.size() != 2) return std::puts("FAIL duplicates are all kept"), 1;
  }
  std::mt19937_64 rng(99);
  auto uni = [&](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  for (int trial = 0; trial < 20; ++trial) {  // test_optimizer.cpp:279-326
    std::vector<ConfigEstimate> pts;
    for (int i = 0; i < 100; ++i) pts.push_back(make(uni(0, 5), uni(0, 5), uni(0, 5), uni(0, 3)));
    if (check_set(pts, "test_optimizer", trial)) return 1;
  }
  for (int set = 0; set < 100; ++set) {  // acceptance.cpp:202-234
    std::vector<ConfigEstimate> pts;
    for (int i = 0; i < 60; ++i) pts.push_back(make(uni(0, 6), uni(0, 6), uni(0, 6), uni(0, 3)));
    if (check_set(pts, "acceptance", set)) return 1;
  }
  for (int set = 0; set < 5; ++set) {  // larger sets: the device filter's blocked path
    std::vector<ConfigEstimate> pts;
    for (int i = 0; i < 20000; ++i) pts.push_back(make(uni(0, 40), uni(0, 40), uni(0, 40), uni(0, 3)));
    const auto kept = loom::pareto_filter(pts);
    std::vector<ConfigEstimate> oracle;
    for (std::size_t i = 0; i < pts.size(); ++i) {
      bool d = false;
      for (std::size_t j = 0; j < pts.size() && !d; ++j) d = dominates(pts[j], pts[i]);
      if (!d) oracle.push_back(pts[i]);
    }
    if (kept.size() != oracle.size()) return std::printf("FAIL large set %d\n", set), 1;
    for (std::size_t i = 0; i < kept.size(); ++i)
      if (!same(kept[i], oracle[i])) return std::printf("FAIL large set %d order\n", set), 1;
  }
  std::puts("ok pareto");
  return 0;
}

static std::string slurp(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return {};
  std::string s;
  char buf[65536];
  std::size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, n);
  std::fclose(f);
  return s;
}

static int group(const char* dag, const char* lib, const char* bounds) {
  const loom::WorkflowDag d = loom::WorkflowDag::from_json_text(slurp(dag));
  const loom::AgentLibrary l = loom::AgentLibrary::from_json_text(slurp(lib));
  const loom::SearchBounds b = loom::SearchBounds::from_json_text(slurp(bounds));
  loom_group* g = nullptr;
  if (loom_group_create(1, &g) != LOOM_OK) return std::printf("FAIL group: %s\n", loom_last_error()), 1;
  for (const char* token : {"MIN_COST", "MIN_DOLLARS", "MIN_LATENCY", "MAX_QUALITY"}) {
    const loom::ObjectiveHierarchy o = loom::objective_from_token(token);
    const ConfigEstimate one = loom::exhaustive_search(d, l, o, b);
    const ConfigEstimate grp = loom::exhaustive_search(d, l, o, b, g);
    if (one.config.identifier() != grp.config.identifier() || one.latency_us != grp.latency_us ||
        one.gpu_wh != grp.gpu_wh)
      return std::printf("FAIL group %s\n", token), 1;
  }
  loom_group_destroy(g);
  std::puts("ok group");
  return 0;
}

int main(int argc, char** argv) {
  try {
    if (argc >= 2 && std::string(argv[1]) == "pareto") return pareto();
    if (argc >= 5 && std::string(argv[1]) == "group") return group(argv[2], argv[3], argv[4]);
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1;
  }
  std::puts("usage: dropin_check pareto | group dag.json library.json bounds.json");
  return 2;
}
