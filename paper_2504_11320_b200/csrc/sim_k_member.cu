// sim_k_member.cu -- member-engine kernels (sched_run), one translation unit
// per engine so the sm_100a build compiles them in parallel
#include "sim_kernel.cuh"

namespace waitsim {

cudaError_t launch_member(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s) {
  if (p.K == 1 && p.policy == SCHED_NESTED) return launch_t<SCHED_NESTED, false, false, false, 1>(p, grid, block, smem, s);
  if (p.K == 1 && p.policy == SCHED_FCFS) return launch_t<SCHED_FCFS, false, false, false, 1>(p, grid, block, smem, s);
  switch (p.policy) {
    case SCHED_WAIT: return launch_t<SCHED_WAIT, false>(p, grid, block, smem, s);
    case SCHED_NESTED: return launch_t<SCHED_NESTED, false>(p, grid, block, smem, s);
    case SCHED_FCFS_ONGOING: return launch_t<SCHED_FCFS_ONGOING, false>(p, grid, block, smem, s);
    default: return launch_t<SCHED_FCFS, false>(p, grid, block, smem, s);
  }
}

cudaError_t occ_member(int policy, int K, int block, size_t smem, int* bps) {
  if (K == 1 && policy == SCHED_NESTED) return occ_t<SCHED_NESTED, false, false, false, 1>(block, smem, bps);
  if (K == 1 && policy == SCHED_FCFS) return occ_t<SCHED_FCFS, false, false, false, 1>(block, smem, bps);
  switch (policy) {
    case SCHED_WAIT: return occ_t<SCHED_WAIT, false>(block, smem, bps);
    case SCHED_NESTED: return occ_t<SCHED_NESTED, false>(block, smem, bps);
    case SCHED_FCFS_ONGOING: return occ_t<SCHED_FCFS_ONGOING, false>(block, smem, bps);
    default: return occ_t<SCHED_FCFS, false>(block, smem, bps);
  }
}

}  // namespace waitsim
