// sim_k_trace.cu -- explicit-trace kernels (sched_run_trace): member engine
// for every policy, segment engine for Nested
#include "sim_kernel.cuh"

namespace waitsim {

cudaError_t launch_trace(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s) {
  if (p.seg_engine) return launch_t<SCHED_NESTED, true, false, true>(p, grid, block, smem, s);
  switch (p.policy) {
    case SCHED_WAIT: return launch_t<SCHED_WAIT, true>(p, grid, block, smem, s);
    case SCHED_NESTED: return launch_t<SCHED_NESTED, true>(p, grid, block, smem, s);
    case SCHED_FCFS_ONGOING: return launch_t<SCHED_FCFS_ONGOING, true>(p, grid, block, smem, s);
    default: return launch_t<SCHED_FCFS, true>(p, grid, block, smem, s);
  }
}

cudaError_t occ_trace(int policy, int block, size_t smem, int* bps, int seg) {
  if (seg) return occ_t<SCHED_NESTED, true, false, true>(block, smem, bps);
  switch (policy) {
    case SCHED_WAIT: return occ_t<SCHED_WAIT, true>(block, smem, bps);
    case SCHED_NESTED: return occ_t<SCHED_NESTED, true>(block, smem, bps);
    case SCHED_FCFS_ONGOING: return occ_t<SCHED_FCFS_ONGOING, true>(block, smem, bps);
    default: return occ_t<SCHED_FCFS, true>(block, smem, bps);
  }
}

}  // namespace waitsim
