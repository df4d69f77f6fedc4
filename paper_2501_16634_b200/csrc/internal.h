// Internal glue shared by the host (.cpp) and device (.cu) halves of
// libloom_b200.so.  Not part of the public ABI.
#pragma once

#include <string>

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

}  // namespace loomi
