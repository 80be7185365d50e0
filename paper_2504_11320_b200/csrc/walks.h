// walks.h -- parameters of the random-walk kernel (internal to libsched)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace waitsim {

constexpr int kWalkFields = 10;  // W_B, stuck, sumW, maxW, Wt_B, viol, sumX, maxS, minS, S_B

struct WalkParams {
  int32_t kind;        // 0: Poisson(mu) arrivals; 1: Binomial(n_prev, p) arrivals
  int64_t n;           // threshold
  double mu;           // Poisson mean (kind 0)
  int64_t kmax;        // kind 0: cap of the inversion loop
  int64_t n_prev;      // kind 1: Binomial trials
  double p0;           // pmf at 0: exp(-mu) or (1-p)^n_prev
  double ratio;        // kind 1: p / (1-p)
  uint64_t seed;
  uint64_t walk_begin; // global index of local walk 0
  uint32_t n_walks;
  uint32_t B;          // steps per walk
  int64_t* out;        // device, field-major [kWalkFields][n_walks]
};

cudaError_t launch_walks(const WalkParams& p, cudaStream_t s);

}  // namespace waitsim
