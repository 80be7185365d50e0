// sim_k_seg.cu -- Nested segment-engine kernels (sched_run), specialised on
// the class count of the bench workloads (C3a: 4, C3b: 1, C4: 3)
#include "sim_kernel.cuh"

namespace waitsim {

cudaError_t launch_seg(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s) {
  if (p.K == 1) return launch_t<SCHED_NESTED, false, false, true, 1>(p, grid, block, smem, s);
  if (p.K == 3) return launch_t<SCHED_NESTED, false, false, true, 3>(p, grid, block, smem, s);
  if (p.K == 4) return launch_t<SCHED_NESTED, false, false, true, 4>(p, grid, block, smem, s);
  return launch_t<SCHED_NESTED, false, false, true>(p, grid, block, smem, s);
}

cudaError_t occ_seg(int K, int block, size_t smem, int* bps) {
  if (K == 1) return occ_t<SCHED_NESTED, false, false, true, 1>(block, smem, bps);
  if (K == 3) return occ_t<SCHED_NESTED, false, false, true, 3>(block, smem, bps);
  if (K == 4) return occ_t<SCHED_NESTED, false, false, true, 4>(block, smem, bps);
  return occ_t<SCHED_NESTED, false, false, true>(block, smem, bps);
}

}  // namespace waitsim
