// sim_kernel.cu -- launch dispatch of the sm_100a simulation kernels
// (sim_kernel.cuh: the kernel; sim_k_*.cu: its instantiations per engine).
#include <cuda_runtime.h>

#include "../../include/sched.h"
#include "sim_internal.h"

namespace waitsim {

cudaError_t launch_member(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t launch_ring(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t launch_seg(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t launch_trace(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t occ_member(int policy, int K, int block, size_t smem, int* bps);
cudaError_t occ_ring(int policy, int K, int block, size_t smem, int* bps);
cudaError_t occ_seg(int K, int block, size_t smem, int* bps);
cudaError_t occ_trace(int policy, int block, size_t smem, int* bps, int seg);

cudaError_t launch_sim(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s) {
  if (p.trace_mode) return launch_trace(p, grid, block, smem, s);
  if (p.seg_engine) return launch_seg(p, grid, block, smem, s);
  if (p.ring_engine) return launch_ring(p, grid, block, smem, s);
  return launch_member(p, grid, block, smem, s);
}

cudaError_t sim_occupancy(int policy, int trace, int block, size_t smem, int* bps, int ring, int K) {
  if (trace) return occ_trace(policy, block, smem, bps, ring == 2);
  if (ring == 2) return occ_seg(K, block, smem, bps);
  if (ring) return occ_ring(policy, K, block, smem, bps);
  return occ_member(policy, K, block, smem, bps);
}

}  // namespace waitsim
