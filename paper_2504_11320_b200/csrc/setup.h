// setup.h -- host-side threshold / fluid setup (internal to libsched)
#pragma once
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/sched.h"

namespace waitsim {

typedef std::vector<std::pair<uint16_t, uint64_t>> Table;  // (value, weight)

struct SetupInput {
  std::vector<double> lambda;
  std::vector<Table> l, lp;
  double d0_s, d1_s;
  int64_t M;
  int policy;
  std::vector<uint32_t> thresholds;  // empty = choose
  std::vector<uint16_t> seg_end;
  uint32_t B;
  std::vector<std::vector<std::pair<double, double>>> rf;  // per class (start s, rate); empty = constant
};

// returns 0, -2 (unstable; report filled), -3 (infeasible), -1 (invalid)
int compute_thresholds(const SetupInput& in, int mode, double delta, double budget_B,
                       sched_threshold_report* out, std::vector<uint32_t>* chosen,
                       std::string* err);

}  // namespace waitsim
