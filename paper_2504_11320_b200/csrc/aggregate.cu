// aggregate.cu -- S6/S7: per-policy sums over the replications of one launch
// (the vector the cross-GPU all-reduce adds; PAPER.md:1235-1242 metrics).
// One block of 1024 threads: each thread sums a strided subset of the
// replications, then a fixed-order warp-shuffle tree and a fixed-order sum of
// the 32 warp partials -- deterministic for a given n_reps.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sched.h"

namespace waitsim {
namespace {

constexpr int kAggInt = 13, kAggF64 = 6;
constexpr double kTicksPerSecond = 1e12;

__device__ __forceinline__ double u128_seconds(uint64_t lo, uint64_t hi) {
  return ((double)lo + (double)hi * 18446744073709551616.0) / kTicksPerSecond;
}

__global__ void __launch_bounds__(1024) agg_kernel(const uint64_t* __restrict__ rows, uint64_t ld, uint32_t n,
                                                   double horizon_s, int64_t* __restrict__ out_i,
                                                   double* __restrict__ out_f) {
  __shared__ int64_t wi[32][kAggInt];
  __shared__ double wf[32][kAggF64];
  int64_t si[kAggInt] = {};
  double sf[kAggF64] = {};
  const int fi[kAggInt - 1] = {SCHED_F_ARRIVALS, SCHED_F_ADMITTED, SCHED_F_COMPLETED, SCHED_F_COMPLETED_AFTER_T,
                               SCHED_F_COMPLETED_TOKENS, SCHED_F_FIRST_TOKENS, SCHED_F_BATCHES,
                               SCHED_F_REQUEST_STEPS, SCHED_F_PREFILL_STEPS, SCHED_F_EVICTIONS,
                               SCHED_F_FINAL_WAITING, SCHED_F_FINAL_RESIDENT};
  for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
    auto v = [&](int f) { return __ldg(rows + (size_t)f * ld + r); };
#pragma unroll
    for (int k = 0; k < kAggInt - 1; ++k) si[k] += (int64_t)v(fi[k]);
    si[kAggInt - 1] += v(SCHED_F_STATUS) != 0;  // replications with a nonzero status
    const double lat = u128_seconds(v(SCHED_F_LAT_LO), v(SCHED_F_LAT_HI));
    const uint64_t comp = v(SCHED_F_COMPLETED);
    const double mean_lat = lat / (double)(comp ? comp : 1);
    const double thr = (double)v(SCHED_F_COMPLETED_TOKENS) / horizon_s;
    sf[0] += lat;
    sf[1] += u128_seconds(v(SCHED_F_TTFT_LO), v(SCHED_F_TTFT_HI));
    sf[2] += u128_seconds(v(SCHED_F_SOJ_LO), v(SCHED_F_SOJ_HI));
    sf[3] += (double)v(SCHED_F_BUSY_TICKS) / kTicksPerSecond;
    sf[4] += mean_lat * mean_lat;
    sf[5] += thr * thr;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kAggInt; ++k) {
    for (int d = 16; d >= 1; d >>= 1) si[k] += __shfl_xor_sync(0xffffffffu, si[k], d);
    if (lane == 0) wi[w][k] = si[k];
  }
#pragma unroll
  for (int k = 0; k < kAggF64; ++k) {
    for (int d = 16; d >= 1; d >>= 1) sf[k] += __shfl_xor_sync(0xffffffffu, sf[k], d);
    if (lane == 0) wf[w][k] = sf[k];
  }
  __syncthreads();
  const int nw = (int)(blockDim.x >> 5);
  if (threadIdx.x < kAggInt) {
    int64_t t = 0;
    for (int j = 0; j < nw; ++j) t += wi[j][threadIdx.x];
    out_i[threadIdx.x] = t;
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 + kAggF64) {
    double t = 0;
    for (int j = 0; j < nw; ++j) t += wf[j][threadIdx.x - 32];
    out_f[threadIdx.x - 32] = t;
  }
}

}  // namespace
}  // namespace waitsim

namespace waitsim {
cudaError_t launch_aggregate(const uint64_t* rows, uint64_t ld, uint32_t n, double horizon_s, int64_t* out_i,
                             double* out_f, cudaStream_t s) {
  agg_kernel<<<1, 1024, 0, s>>>(rows, ld, n, horizon_s, out_i, out_f);
  return cudaGetLastError();
}
}  // namespace waitsim
