// walks_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see des_oracle.cpp header).
//
// The appendix's embedded random-walk chains, written out one step at a
// time from the paper (App. B "Single-Type Case" 2150-2197 and
// App. C "Subsequent Segments Analysis" 2290-2325), with the draw of
// DESIGN.md §4.9 (own Philox, own pmf inversion; no code shared with the
// CUDA path).
#include <cmath>
#include <cstdint>
#include <cstring>

namespace {
void philox2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
             uint32_t* o0, uint32_t* o1) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  *o0 = c0; *o1 = c1;
}
}  // namespace

extern "C" int orc_walks(int32_t kind, int64_t n, double mu, int64_t n_prev, double p,
                         uint64_t seed, uint64_t walk_begin, uint32_t n_walks, uint32_t B,
                         int64_t* out) {
  // pmf inversion constants
  const double p0 = kind == 0 ? std::exp(-mu) : std::pow(1.0 - p, (double)n_prev);
  const double ratio = kind == 0 ? 0.0 : p / (1.0 - p);
  const int64_t kmax = kind == 0 ? (int64_t)(mu + 40.0 * std::sqrt(mu) + 100.0) : n_prev;
  for (uint32_t w = 0; w < n_walks; ++w) {
    const uint32_t wg = (uint32_t)(walk_begin + w);
    // coupled process start and floor: 2n for the WAIT chain (Lemma
    // "Coupled Dominating Process"), n for segment k
    // (Lemma "Coupled Process for Segment k")
    const int64_t c0 = kind == 0 ? 2 * n : n;
    int64_t W = 0, Wt = c0, S = 0, maxS = 0, minS = 0, maxW = 0;
    int64_t stuck = 0, viol = 0, sumX = 0, sumW = 0;
    for (uint32_t b = 0; b < B; ++b) {
      uint32_t x0, x1;
      philox2(b, wg, 0x80000000u | (uint32_t)kind, 0u, (uint32_t)seed, (uint32_t)(seed >> 32), &x0, &x1);
      const uint64_t v = 2 * (((uint64_t)x0 << 20) | (x1 >> 12)) + 1;
      const double U = (double)v * 0x1p-53;
      // arrivals this batch: Poisson(mu) or
      // Binomial(n_{k-1}, p_k), by inverting the pmf
      int64_t X = 0;
      double pk = p0, F = p0;
      if (kind == 0) {
        while (U > F && X < kmax) { ++X; pk = (pk * mu) / (double)X; F = F + pk; }
      } else {
        while (U > F && X < n_prev) {
          pk = ((pk * (double)(n_prev - X)) / (double)(X + 1)) * ratio;
          ++X;
          F = F + pk;
        }
      }
      // W^{b+1} = W^b + X^b - n 1{W^b + X^b >= n}; stuck iteration otherwise
      sumX += X;
      if (W + X >= n) W = W + X - n; else { W = W + X; ++stuck; }
      // coupled process W~^{b+1} = max(c0, W~^b + X^b - n)
      Wt = std::max(c0, Wt + X - n);
      const bool dominated = kind == 0 ? (Wt >= W + n) : (Wt >= W);
      if (!dominated) ++viol;
      S += X - n;
      maxS = std::max(maxS, S);
      minS = std::min(minS, S);
      maxW = std::max(maxW, W);
      sumW += W;
    }
    const int64_t vals[10] = {W, stuck, sumW, maxW, Wt, viol, sumX, maxS, minS, S};
    for (int f = 0; f < 10; ++f) out[(int64_t)f * n_walks + w] = vals[f];
  }
  return 0;
}
