// ORACLE TEST INFRASTRUCTURE.  Compiled against the UNMODIFIED reference
// headers (oracle/Makefile target `adapter`), this binary runs the
// reference's loom::exhaustive_search and the drop-in
// loom_b200_adapter::exhaustive_search (integration/loom_b200_adapter.hpp ->
// libloom_b200.so -> sm_100a kernel) on the same inputs and compares the
// selected ConfigPoint and every metric bit for bit.
//
//   adapter_check DAG LIB BOUNDS TOKEN [FLOOR]     -> prints JSON, exit 0 iff equal
#include <cstdio>
#include <fstream>
#include <sstream>

#include "loom/loom.hpp"
#include "loom_b200_adapter.hpp"

using nlohmann::json;

static std::string slurp(const char* p) {
  std::ifstream in(p);
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: adapter_check DAG LIB BOUNDS TOKEN [FLOOR]\n");
    return 2;
  }
  const auto dag = json::parse(slurp(argv[1])).get<loom::WorkflowDag>();
  auto library = loom::AgentLibrary::from_json(json::parse(slurp(argv[2])));
  library.freeze();
  const json bj = json::parse(slurp(argv[3]));
  loom::SearchBounds bounds;
  bounds.max_fanout = bj.value("max_fanout", 4);
  bounds.max_paths = bj.value("max_paths", 2);
  if (bj.contains("sku_pool_cap")) bounds.sku_pool_cap = bj.at("sku_pool_cap").get<std::map<std::string, int>>();
  if (bj.contains("sku_total_cap")) bounds.sku_total_cap = bj.at("sku_total_cap").get<std::map<std::string, int>>();
  auto objective = loom::objective_from_token(argv[4]);
  if (argc > 5) objective.quality_floor = std::atoi(argv[5]);

  json out;
  std::string ref_err, gpu_err;
  loom::ConfigEstimate ref, gpu;
  try {
    ref = loom::exhaustive_search(dag, library, objective, bounds);
  } catch (const loom::Error& e) {
    ref_err = e.what();
  }
  try {
    gpu = loom_b200_adapter::exhaustive_search(dag, library, objective, bounds);
  } catch (const std::exception& e) {
    gpu_err = e.what();
  }
  bool same;
  if (!ref_err.empty() || !gpu_err.empty()) {
    same = ref_err == gpu_err;
  } else {
    same = ref.config.identifier() == gpu.config.identifier() && ref.latency_us == gpu.latency_us &&
           ref.gpu_wh == gpu.gpu_wh && ref.cpu_wh == gpu.cpu_wh && ref.total_wh == gpu.total_wh &&
           ref.dollars == gpu.dollars && ref.quality == gpu.quality;
  }
  out["same"] = same;
  out["reference"] = ref_err.empty() ? json(ref.config.identifier()) : json(ref_err);
  out["b200"] = gpu_err.empty() ? json(gpu.config.identifier()) : json(gpu_err);
  std::printf("%s\n", out.dump().c_str());
  return same ? 0 : 1;
}
