// Internal glue shared by the host (.cpp) and device (.cu) halves of
// libloom_b200.so.  Not part of the public ABI.
#pragma once

#include <sched.h>

#include <algorithm>
#include <functional>
#include <string>
#include <thread>

#include "loom_b200.h"

namespace loomi {

// Thread-local message returned by loom_last_error(); formatted like the
// reference's loom::Error::what(): "<ErrorClass>: <message>".
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);

// Validates a problem and computes its plan count (host, no device).
int check_problem(const loom_problem* p, uint64_t* total);

// Fills every metric of *w from w->plan_index with the reference's exact
// arithmetic (estimator.hpp:43-78).  Sets found = 1.
int fill_winner(const loom_problem* p, loom_winner* w);

// Host threads this process may run on (its CPU affinity mask; the machine's
// count when unavailable): the default width of the host-side batch work
// (more threads than cores only add switching, measured on C4).
inline int host_threads() {
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof set, &set) == 0) {
    const int n = CPU_COUNT(&set);
    if (n > 0) return n;
  }
  return static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
}

// The batch search (loom_search_argmin_batch) with its jobs produced on the
// host threads that build the problem images: produce(j, worker, &problems[j],
// &objectives[j]) fills job j (worker < threads, for per-thread caches) or
// returns its failure status; retire(j) runs once job j's winner is final.
// Either callback may be empty (problems/objectives are then read as given).
using BatchProduce = std::function<int(int job, int worker, loom_problem* p, loom_objective* o)>;
using BatchRetire = std::function<void(int job)>;
int argmin_batch(loom_ctx* c, int n_jobs, int threads, loom_problem* problems, loom_objective* objectives,
                 const BatchProduce& produce, const BatchRetire& retire, loom_winner* out, int32_t* status);

}  // namespace loomi
