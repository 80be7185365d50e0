// walks.cu -- NEXT(4): the appendix's embedded random-walk chains as a
// second GPU workload (App. B-C, 2150-2373).  One thread = one
// walk; walks are independent, B steps each.
//
//   kind 0 (WAIT, Lemma "Queue Length and Stuck Time"):
//     X^b ~ Poisson(mu);  W^{b+1} = W^b + X^b - n 1{W^b + X^b >= n};
//     coupled W~^0 = 2n, W~^{b+1} = max(2n, W~^b + X^b - n)   (Lemma, 2169)
//   kind 1 (Nested segment k >= 2):
//     Y^b ~ Binomial(n_prev, p);  W^{b+1} = W^b + Y^b - n 1{W^b + Y^b >= n};
//     coupled W~^0 = n, W~^{b+1} = max(n, W~^b + Y^b - n)
//
// Draws are bit-exact with the oracle: step b of walk w uses
// Philox4x32-10(ctr=(b, w, 0x80000000|kind, 0), key=seed) words x0, x1 ->
// U = (2 u52 + 1) 2^-53, then inversion of the pmf with one rounded IEEE op
// per line.
#include <cuda_runtime.h>
#include <stdint.h>

#include "walks.h"

namespace waitsim {
namespace {

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint32_t k0, uint32_t k1, uint32_t& o0, uint32_t& o1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  o0 = c0; o1 = c1;
}

__global__ void __launch_bounds__(256) walk_kernel(const WalkParams P) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= P.n_walks) return;
  const uint32_t wg = (uint32_t)(P.walk_begin + w);
  const int64_t n = P.n;
  const int64_t c0 = P.kind == 0 ? 2 * n : n;  // coupled process start / floor
  int64_t W = 0, Wt = c0, S = 0, maxS = 0, minS = 0, maxW = 0;
  int64_t stuck = 0, viol = 0, sumX = 0, sumW = 0;
  for (uint32_t b = 0; b < P.B; ++b) {
    uint32_t x0, x1;
    philox(b, wg, 0x80000000u | (uint32_t)P.kind, 0u, (uint32_t)P.seed, (uint32_t)(P.seed >> 32),
           x0, x1);
    const uint64_t v = ((((uint64_t)x0 << 20) | (uint64_t)(x1 >> 12)) << 1) | 1ull;
    const double U = __dmul_rn((double)v, 0x1p-53);
    // inversion of the pmf
    int64_t k = 0;
    double pk = P.p0, F = P.p0;
    if (P.kind == 0) {
      while (U > F && k < P.kmax) {
        ++k;
        pk = __ddiv_rn(__dmul_rn(pk, P.mu), (double)k);
        F = __dadd_rn(F, pk);
      }
    } else {
      while (U > F && k < P.n_prev) {
        pk = __dmul_rn(__ddiv_rn(__dmul_rn(pk, (double)(P.n_prev - k)), (double)(k + 1)), P.ratio);
        ++k;
        F = __dadd_rn(F, pk);
      }
    }
    const int64_t X = k;
    sumX += X;
    W += X;
    if (W >= n) W -= n; else ++stuck;      // batch processed / stuck iteration
    const int64_t t = Wt + X - n;
    Wt = t > c0 ? t : c0;                  // coupled dominating process
    if (P.kind == 0 ? (Wt < W + n) : (Wt < W)) ++viol;
    S += X - n;
    if (S > maxS) maxS = S;
    if (S < minS) minS = S;
    if (W > maxW) maxW = W;
    sumW += W;
  }
  const size_t N = P.n_walks;
  int64_t* o = P.out;
  o[0 * N + w] = W;     o[1 * N + w] = stuck; o[2 * N + w] = sumW; o[3 * N + w] = maxW;
  o[4 * N + w] = Wt;    o[5 * N + w] = viol;  o[6 * N + w] = sumX; o[7 * N + w] = maxS;
  o[8 * N + w] = minS;  o[9 * N + w] = S;
}

}  // namespace

cudaError_t launch_walks(const WalkParams& p, cudaStream_t s) {
  const int block = 256;
  const int grid = (int)((p.n_walks + block - 1) / block);
  walk_kernel<<<grid, block, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace waitsim
