// sim_kernel.cuh -- sm_100a kernel of the batched WAIT / Nested WAIT / FCFS
// discrete-event simulation (arXiv 2504.11320).  One warp simulates one
// replication; a persistent grid pulls replication indices from a global
// counter.  Semantics: DESIGN.md §4 (event loop, policies, metrics), which
// restates the paper passages cited inline.
//
// Two resident engines, one semantics:
//   member engine (template RING = false; every policy, length marks,
//     explicit traces): residents in admission order as 16-byte records
//     {a = arrival tick, l | l' << 16 | s << 32 | meta << 48}; a batch is one
//     pass over them with ballot/popc compaction;
//   class-ring engine (RING = true; WAIT / FCFS with fixed per-class
//     lengths): residents of class c in their own ring, stage = class clock
//     - admission clock, so a batch touches only completions and admissions.
// Layout per warp (shared memory, carved from dynamic smem; warp_smem_bytes):
//   residents (member) or staged admissions + spare victim slots + class rings
//   (RING); per class a generated window and a private admission window
//   (t / l / l' of 32 arrivals each, one offset space); 32 staged restart
//   ticks; counters[64] (WAIT: residents per class; NESTED: [k] non-entry
//   residents of segment k, [32+k] residents waiting at its entry stage;
//   RING: [32+c] pending first tokens), rank[32] / snap[32] (NESTED rank
//   cursors; RING: pending first-token tick sums), WarpStats, RING eviction
//   scratch, time-varying operational-time windows.
// Per-class cursor state lives in REGISTERS of lane c (broadcast by shfl).
// Waiting prompts hold no KV: new arrivals are cursor ranges
// [k_adm, k_vis) of the class's Philox stream, regenerated at admission;
// evicted prompts go to per-FIFO restart rings in global memory.

#include <cuda_runtime.h>
#include <stdint.h>

#pragma once
#include "../../include/sched.h"
#include "sim_internal.h"

// launch-bound knobs of the FCFS class-ring kernels (blocks per SM), measured:
// K = 2: 5 (6: C2 FCFS 15.6 -> 18.5 ms, 4: -> 17.4 ms); K = 3: 4 (C4 FCFS
// 2.65 / 2.91 -> 2.55 / 2.75 ms at rho 0.9 / 0.95); K = 4: 5 (4: C3a FCFS
// 51.9 -> 54.6 ms)
// class count at which ring_append sums pending first tokens by ballot + warp
// reductions instead of shared atomics (~15 same-address atomics per class and
// batch at C2: WAIT 13.0 -> 12.3 ms, FCFS 15.4 -> 14.0 ms; K = 1 (C1: few
// admissions per batch) +2%, K = 3 / 4 (C4 / C3a FCFS) +3 / +8%)
#ifndef WAITSIM_WAIT_GEN_INL  // WAIT kernels inline the window generator (1) or call it (0: C2 WAIT 12.3 -> 13.5 ms)
#define WAITSIM_WAIT_GEN_INL 1
#endif
#ifndef WAITSIM_WAIT2_ONEWARP  // two-class WAIT ring kernel in one-warp blocks: C2 WAIT 12.3 -> 11.4 ms
#define WAITSIM_WAIT2_ONEWARP 1
#endif
#ifndef WAITSIM_FCFS4_ONEWARP  // four-class FCFS ring kernel in one-warp blocks: C3a FCFS 49.7 -> 48.3,
#define WAITSIM_FCFS4_ONEWARP 1   // C3a_tv 46.8 -> 43.3 ms (three classes: C4 FCFS +1..3%, not used)
#endif
#ifndef WAITSIM_FCFS1_ONEWARP  // (one-class FCFS ring one-warp: C1 FCFS 69.1 -> 71.9 ms: off)
#define WAITSIM_FCFS1_ONEWARP 0
#endif
#ifndef WAITSIM_MEMBER_FCFS_ONEWARP  // (one-warp member FCFS: C3b 30.1 -> 29.5 ms, C5 FCFS 71.7 -> 74.0 ms: off)
#define WAITSIM_MEMBER_FCFS_ONEWARP 0
#endif
#ifndef WAITSIM_SEG_ONEWARP  // (segment engine one-warp: C3a 54.0 -> 58.4 ms, C3b 17.2 -> 19.1 ms: 1 KB reserved smem per block)
#define WAITSIM_SEG_ONEWARP 0
#endif
#ifndef WAITSIM_WAITK_ONEWARP  // (other WAIT ring kernels one-warp: C1 / C4 within +-2%)
#define WAITSIM_WAITK_ONEWARP 0
#endif
#ifndef WAITSIM_FCFS2_ONEWARP  // (FCFS in one-warp blocks: C2 FCFS 13.0 -> 13.2 ms)
#define WAITSIM_FCFS2_ONEWARP 0
#endif
#ifndef WAITSIM_PEND_REDUCE_K
#define WAITSIM_PEND_REDUCE_K 2
#endif
#ifndef WAITSIM_WAIT2_MINB  // two-class WAIT ring kernel: 6 (80 registers); 4-warp blocks 5 / 7: 13.7 / 14.2 vs 13.0 ms; one-warp 5 / 7: 12.2 / 11.7 vs 11.4 ms
#define WAITSIM_WAIT2_MINB 6
#endif
#ifndef WAITSIM_MEMBER_FCFS_MINB  // member-engine FCFS (length marks), blocks of 8 warps: 3 (80
#define WAITSIM_MEMBER_FCFS_MINB 3   // registers): C3b FCFS 32.6 -> 30.1 ms, C5 FCFS 68 -> 71 ms per 600 s
#endif
#ifndef WAITSIM_FCFS2_MINB
#define WAITSIM_FCFS2_MINB 5
#endif
#ifndef WAITSIM_FCFS3_MINB
#define WAITSIM_FCFS3_MINB 4
#endif
#ifndef WAITSIM_FCFS4_MINB
#define WAITSIM_FCFS4_MINB 5
#endif

namespace waitsim {
namespace {

typedef unsigned __int128 u128;
constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t TMAX = INT64_MAX;
constexpr uint16_t META_FT = 0x100;  // first output token already emitted

// ------------------------------------------------------------- primitives
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27; z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds, key bumped between rounds.
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1, uint32_t& o0,
                                              uint32_t& o1, uint32_t& o2, uint32_t& o3) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// E = -ln U, U = (2 u52 + 1) 2^-53; every step one correctly rounded IEEE op
// so the CPU oracle reproduces it bit for bit.
__device__ __forceinline__ double neglog_bits(uint32_t x0, uint32_t x1) {
  const uint64_t v = ((((uint64_t)x0 << 20) | (uint64_t)(x1 >> 12)) << 1) | 1ull;
  int e = 63 - __clzll((long long)v);
  // f = v * 2^-e in [1,2): exact, built from the bits
  double f = __longlong_as_double(
      (long long)((0x3FFull << 52) | ((v << (52 - e)) & 0xFFFFFFFFFFFFFull)));
  if (f > 0x1.6a09e667f3bcdp+0) { f = __dmul_rn(f, 0.5); e += 1; }
  const double s = __ddiv_rn(__dsub_rn(f, 1.0), __dadd_rn(f, 1.0));
  const double z = __dmul_rn(s, s);
  double P = 1.0 / 19.0;
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 17.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 15.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 13.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 11.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 9.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 7.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 5.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0 / 3.0);
  P = __dadd_rn(__dmul_rn(P, z), 1.0);
  const double lnf = __dmul_rn(__dadd_rn(s, s), P);
  const double dn = (double)(e - 53);
  const double ln2_hi = __longlong_as_double(0x3fe62e42fee00000ll);
  const double ln2_lo = __longlong_as_double(0x3dea39ef35793c76ll);
  const double lnU = __dadd_rn(__dmul_rn(dn, ln2_hi), __dadd_rn(__dmul_rn(dn, ln2_lo), lnf));
  return -lnU;
}

// inverse-CDF of an integer-weight table: idx = min{i : x < thr_i}.  A guide
// table (Chen & Asau) gives the answer for the lowest x of x's bucket, the
// forward scan from it the exact same index as a binary search (usually 0-1
// steps instead of log2 n dependent loads).
__device__ __forceinline__ uint32_t cdf_sample(const uint64_t* __restrict__ thr,
                                               const uint16_t* __restrict__ val,
                                               const uint16_t* __restrict__ guide, uint32_t off,
                                               uint32_t nlg, uint32_t goff, uint32_t x) {
  if ((nlg & 0xFFFFFFu) == 1) return __ldg(val + off);
  uint32_t i = __ldg(guide + goff + (x >> (32 - (nlg >> 24))));
  while (__ldg(thr + off + i) <= (uint64_t)x) ++i;
  return __ldg(val + off + i);
}

__device__ __forceinline__ int64_t warp_incl_scan_i64(int64_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, x, d);
    if (lane >= d) x += y;
  }
  return x;
}
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, d);
    if (lane >= d) x += y;
  }
  return x;
}
__device__ __forceinline__ u128 warp_sum_u128(u128 x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const uint64_t lo = __shfl_xor_sync(FULL, (uint64_t)x, d);
    const uint64_t hi = __shfl_xor_sync(FULL, (uint64_t)(x >> 64), d);
    x += ((u128)hi << 64) | lo;
  }
  return x;
}
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
  return x;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
  return x;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// shared-memory reductions (explicit .shared: the generic atomics the
// compiler emits for smem pointers it cannot prove are slower)
__device__ __forceinline__ void sh_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void sh_add_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.shared.add.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t bcast64(int64_t v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ uint32_t bcast32(uint32_t v, int src) { return __shfl_sync(FULL, v, src); }

// ------------------------------------------------------------- the warp sim
// resident record, packed: l | l' << 16 | s << 32 | meta << 48
__device__ __forceinline__ uint64_t pack_q(uint32_t l, uint32_t lp, uint32_t s, uint32_t meta) {
  return (uint64_t)l | ((uint64_t)lp << 16) | ((uint64_t)s << 32) | ((uint64_t)meta << 48);
}
constexpr uint32_t META_RESTART = 0x200;
// one resident: arrival tick + packed record, 16 B (one LDS.128 / STS.128)
struct __align__(16) Rec {
  int64_t a;
  uint64_t q;
};
constexpr uint32_t kRingLog = 1u << 16;  // admission-log entries per warp (class-ring engine)
// segment-engine resident (NESTED), shared memory: l | l' << 16,
// cohort clock x (bits 0-30: the segment clock at which it ran its entry
// stage; stage = b_k + C_k - x) | first token emitted before a restart (bit
// 31); its arrival tick sits at the same position of a per-warp global array
struct __align__(8) SRec {
  uint32_t llp;
  uint32_t xf;
};
constexpr uint32_t SX_FT = 0x80000000u, SX_X = 0x7FFFFFFFu;
__device__ __forceinline__ uint32_t wrap(uint32_t p, uint32_t cap) { return p >= cap ? p - cap : p; }  // staging mark: came from a restart ring

// # of leading entries of the sorted array v[0..n) that precede `key`
// (v <= key if le, v < key otherwise)
__device__ __forceinline__ uint32_t count_before(const int64_t* v, uint32_t n, int64_t key, bool le) {
  uint32_t lo = 0, len = n;
  while (len > 0) {
    const uint32_t half = len >> 1;
    const int64_t x = v[lo + half];
    if (le ? (x <= key) : (x < key)) { lo += half + 1; len -= half + 1; } else { len = half; }
  }
  return lo;
}

struct WarpStats;
__device__ __noinline__ void flush_sums(WarpStats* st, int lane, uint64_t a0, uint64_t a1, uint64_t a2,
                                       uint64_t a3, uint64_t a4);

// per-replication metric accumulators, one per warp in shared memory
// (updated once per batch by lane 0; keeps them out of the register file)
struct __align__(16) WarpStats {
  u128 sum_done_t, sum_ft_t;            // sum over batches of n * t_end
  u128 acc_arr, acc_done_a, acc_ft_a;   // flushed lane-local arrival-tick sums
  uint64_t arrivals, admitted, completed, completed_after_T, completed_tokens, first_tokens,
      batches, request_steps, prefill_steps, evictions, cbi, sum_waiting, h;
  int64_t busy, idle, max_kv, log_n;
  u128 acc_adm, acc_ev;                 // segment engine: admitted / evicted arrival-tick sums
};
static_assert(sizeof(WarpStats) <= 256, "WarpStats slot");

// lane-local arrival-tick sums -> 128-bit warp totals (out of line: rarely
// run, and keeps the per-batch instruction footprint small)
__device__ __noinline__ void flush_sums(WarpStats* st, int lane, uint64_t a0, uint64_t a1, uint64_t a2,
                                       uint64_t a3, uint64_t a4) {
  const u128 s0 = warp_sum_u128(a0), s1 = warp_sum_u128(a1), s2 = warp_sum_u128(a2);
  const u128 s3 = warp_sum_u128(a3), s4 = warp_sum_u128(a4);
  if (lane == 0) {
    st->acc_arr += s0; st->acc_done_a += s1; st->acc_ft_a += s2;
    st->acc_adm += s3; st->acc_ev += s4;
  }
  __syncwarp();
}

// arrival tick at operational time tau of a time-varying class: invert the
// integrated piecewise-constant rate
__device__ __forceinline__ int64_t tv_tick_at(const int64_t* rf_B, const int64_t* rf_Lam,
                                              const double* rf_scale, uint32_t off, uint32_t n,
                                              int64_t tau) {
  uint32_t lo = 0, hi = n;  // largest p with Lam[p] <= tau (Lam[0] = 0)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(rf_Lam + off + mid) <= tau) lo = mid; else hi = mid;
  }
  const double scale = __ldg(rf_scale + off + lo);
  if (scale == 0.0) return TMAX;
  int64_t t = __ldg(rf_B + off + lo) +
              __double2ll_rz(__dmul_rn(__ll2double_rn(tau - __ldg(rf_Lam + off + lo)), scale));
  if (lo + 1 < n) t = min(t, __ldg(rf_B + off + lo + 1) - 1);
  return t;
}

// S1 arrival generation, one warp: lane i draws
// arrival base+i of class c from Philox counter (k, r, c, 0), the gaps (or
// operational-time increments) become ticks by an inclusive warp scan on top
// of `prev`, marks by inverse CDF.  Not inlined: one copy per kernel keeps
// the instruction footprint small (called at most once per 32 arrivals).
__device__ __forceinline__ void gen_window_impl(int lane, uint32_t base, int64_t prev, uint32_t rglob,
                                        uint32_t c, uint64_t seed, double gs,
                                        const uint64_t* __restrict__ cdf_thr,
                                        const uint16_t* __restrict__ cdf_val,
                                        const uint16_t* __restrict__ cdf_guide, uint32_t l_goff,
                                        uint32_t lp_goff, uint32_t l_off,
                                        uint32_t l_n, uint32_t lp_off, uint32_t lp_n,
                                        uint32_t rf_off, uint32_t rf_n, const int64_t* rf_B,
                                        const int64_t* rf_Lam, const double* rf_scale,
                                        int64_t* wt, uint16_t* wl, uint16_t* wlp, int64_t* wtau) {
  const uint32_t k = base + (uint32_t)lane;
  int64_t t = TMAX, tau = 0;
  uint32_t l = 1, lp = 1;
  if (gs != 0.0 || rf_n != 0) {
    uint32_t x0, x1, x2, x3;
    philox4x32_10(k, rglob, c, 0u, (uint32_t)seed, (uint32_t)(seed >> 32), x0, x1, x2, x3);
    const double E = neglog_bits(x0, x1);
    if (rf_n != 0) {
      // time change: tau_k = tau_{k-1} + (int64)(E 2^32), t_k = Lambda^{-1}(tau_k)
      tau = prev + warp_incl_scan_i64(__double2ll_rz(__dmul_rn(E, 4294967296.0)), lane);
      t = tv_tick_at(rf_B, rf_Lam, rf_scale, rf_off, rf_n, tau);
    } else {
      t = prev + warp_incl_scan_i64(__double2ll_rz(__dmul_rn(E, gs)), lane);
    }
    l = cdf_sample(cdf_thr, cdf_val, cdf_guide, l_off, l_n, l_goff, x2);
    lp = cdf_sample(cdf_thr, cdf_val, cdf_guide, lp_off, lp_n, lp_goff, x3);
  }
  __syncwarp();
  wt[lane] = t;
  wl[lane] = (uint16_t)l;
  wlp[lane] = (uint16_t)lp;
  if (wtau) wtau[lane] = tau;
  __syncwarp();
}

#define GEN_WINDOW_ARGS                                                                      \
  int lane, uint32_t base, int64_t prev, uint32_t rglob, uint32_t c, uint64_t seed, double gs, \
      const uint64_t *cdf_thr, const uint16_t *cdf_val, const uint16_t *cdf_guide,            \
      uint32_t l_goff, uint32_t lp_goff, uint32_t l_off, uint32_t l_n,                        \
      uint32_t lp_off, uint32_t lp_n, uint32_t rf_off, uint32_t rf_n, const int64_t *rf_B,    \
      const int64_t *rf_Lam, const double *rf_scale, int64_t *wt, uint16_t *wl, uint16_t *wlp, \
      int64_t *wtau
#define GEN_WINDOW_PASS                                                                   \
  lane, base, prev, rglob, c, seed, gs, cdf_thr, cdf_val, cdf_guide, l_goff, lp_goff, l_off, \
      l_n, lp_off, lp_n, rf_off,                                                            \
      rf_n, rf_B, rf_Lam, rf_scale, wt, wl, wlp, wtau
// one out-of-line copy (large kernels: instruction-cache footprint) ...
__device__ __noinline__ void gen_window_call(GEN_WINDOW_ARGS) { gen_window_impl(GEN_WINDOW_PASS); }
// ... or inlined (WAIT: register-bound, a call costs spills)
template <bool INLINE>
__device__ __forceinline__ void gen_window(GEN_WINDOW_ARGS) {
  if (INLINE) gen_window_impl(GEN_WINDOW_PASS);
  else gen_window_call(GEN_WINDOW_PASS);
}

template <int POL, bool TRACE, bool RING, bool SEG, int KC>
struct WarpSim {
  // class count: a compile-time constant when the kernel is specialised (KC > 0)
  __device__ __forceinline__ int nK() const { return KC ? KC : P.K; }
  // the general admission path reads each staged restart's pool record in the
  // same round trip as its eviction tick (C2 FCFS 14.1 -> 13.2 ms, C4 -1..3%);
  // the Nested member engine and the four-class kernels keep the per-candidate
  // reads (C5 Nested 588 -> 634 ms, C3a FCFS 49.4 -> 52.2 ms otherwise)
  static constexpr bool kEarlyRestart = !(POL == SCHED_NESTED && !SEG) && KC != 4;
  const DevParams& P;
  const int lane;
  // shared-memory views (this warp's slice)
  Rec* rr;                           // [Rc] residents in admission order (RING: staged admissions)
  ulonglong2* rg;                    // RING: class rings in global memory (ring c: P.rcap[c] records from P.roff[c]):
                                     //   {arrival tick | first token emitted before admission (restart) << 63,
                                     //    admission clock x}: one 16-B store per admission
  uint32_t* coh;                     // RING: [ccsize] members admitted at class clock x, slot x mod (l'_c + 1)
  int64_t* vt;                       // [K][32] generated window (t): visibility + admission
  uint16_t* vl; uint16_t* vlp;       // [K][32] generated window (l, l')
  int64_t* at;                       // [K][32] private admission windows (t)
  uint16_t* al; uint16_t* alp;       // [K][32] private admission windows (l, l')
  int64_t* re;                       // [32] staged restart-ring eviction ticks
  int64_t* vtau; int64_t* atau;      // [K][32] operational time (time-varying classes only)
  uint32_t* cnt;                     // [64] WAIT: residents per class; NESTED: [k] / [32+k]
  uint32_t* rank;                    // [32] NESTED per-segment rank cursors
  uint32_t* snap;                    // [32] NESTED entry counts at decision time
  WarpStats* st;                     // metric accumulators
  uint64_t* xs;                      // [32] RING eviction scratch (per-class sums)
  uint8_t* csum;                     // NESTED: per-chunk lowest resident segment
  uint32_t* rq;                      // [n_rings][16] restart FIFO chunks: head, head index, tail, tail index, stash
  // SEG (NESTED segment engine): residents in one array in
  // admission order = stage order; segment k is the range [P_k, P_{k-1})
  // (k = 0: [P_0, tail)), non-entry part [P_k, E_k), entry-stage part
  // [E_k, P_{k-1}); completed records stay as tombstones until compaction
  SRec* sa;                          // [seg_cap] positions [head, tail)
  int64_t* ga;                       // [seg_cap] their arrival ticks (global memory, this warp's slot)
  uint32_t* hcnt; uint32_t* hsll; uint32_t* hslp;  // [hsize] completion histograms: count, sum (l+l'), sum l'
  uint32_t* con; uint32_t* col;      // [csize] cohort rings: records | exiting << 16, sum l of the exiting

  // per-class cursor state, lane c holds class c (and ring c for WAIT; ring 0
  // otherwise).  The generated window [vbase, vbase+32) serves visibility
  // and, while the backlog fits in it, admission too ("attached":
  // k_adm >= vbase).  Pending arrivals still needed when the window advances
  // are copied to the private window [abase, abase+pcount); a deeper backlog
  // regenerates the private window from the Philox counter.  vprev/aprev:
  // tick of arrival (base - 1), the scan carry.
  uint32_t k_vis, vbase, k_adm, abase, pcount, rhead, rtail;
  int64_t vprev, aprev;
  uint32_t sv_k, sv_rhead, sv_have;  // saved admission cursor (drop/rewind); sv_prev valid
  int64_t sv_prev;
  uint32_t newc;                     // WAIT: admissions of class `lane` this epoch

  // RING: lane c holds class c's ring (head position, residents, clock =
  // batches class c took part in, sum of admission clocks) + next sequence no.
  uint32_t r_head, r_n, r_C, seq_next;
  uint32_t r_Ri;                     // r_C mod (l'_c + 1): cohort slot of the current clock
  uint32_t seq_max;                  // RING: admissions ever logged (uniform; the log keeps the last kRingLog)
  uint32_t wslot;                    // this warp's slot in the per-warp global arrays
  uint64_t r_X;
  // RING: first tokens pending at class c's next participation: count in
  // cnt[32 + c], arrival-tick sum in psum()[c] (the NESTED rank / snap slots)
  __device__ __forceinline__ uint64_t* psum() const { return (uint64_t*)rank; }

  // SEG, lane k = segment k: range starts P_k / E_k, clock C_k (batches the
  // segment took part in), C_k mod W_k, C_k mod (W_k + 1), alive non-entry /
  // entry-stage residents, T_k = sum over alive non-entry (l - x)
  uint32_t g_P, g_E, g_C, g_R, g_Rc, g_nne, g_nen;
  int64_t g_T;
  uint32_t head, tail;               // uniform
  uint32_t pf_n;                     // uniform: first tokens due at the next batch (stage 1) ...
  uint64_t pf_a;                     // ... and their arrival-tick sum
  uint64_t acc_adm, acc_ev;          // SEG / RING: lane-local arrival-tick sums of admissions / evictions

  // replication
  uint32_t rep, rglob;
  int64_t now, KV;
  uint32_t n_res, n_new, status;
  int64_t sum_new_l;
  // lane-local partial sums of arrival ticks (flushed to st before they can overflow)
  uint64_t acc_arr, acc_done_a, acc_ft_a;
  // per-epoch plan
  uint32_t Qmask;     // WAIT: qualifying classes
  int kstar;          // NESTED: last active segment
  uint32_t n_plan_res;
  bool below;         // no batch because of the threshold test (idle skip allowed)

  __device__ WarpSim(const DevParams& p, unsigned char* base, int lane_, uint32_t slot)
      : P(p), lane(lane_) {
    // layout (make_layout): the per-class windows, counters, WarpStats and
    // scratch first -- offsets that depend on the class count only, so a
    // kernel specialised on K addresses them with immediates -- then the
    // operational-time windows, Nested chunk summaries, residents / staging,
    // engine arrays; restart-FIFO cursors at the end
    const int K = KC ? KC : p.K;
    vt = (int64_t*)base;
    at = vt + K * 32;
    re = at + K * 32;
    // l / l' of both windows share one offset space with the ticks:
    // offset o < 32K is vt[o] / vl[o] / vlp[o], 32K <= o < 64K the private window
    vl = (uint16_t*)(re + 32);
    al = vl + K * 32;
    vlp = al + K * 32;
    alp = vlp + K * 32;
    cnt = (uint32_t*)(alp + K * 32);  // 768 K + 256 bytes: 16-aligned
    rank = cnt + 64;
    snap = rank + 32;
    st = (WarpStats*)(snap + 32);
    xs = (uint64_t*)((unsigned char*)st + 256);
    vtau = (int64_t*)((unsigned char*)st + 512);
    atau = vtau + K * 32;
    csum = base + p.off_csum;
    rr = (Rec*)(base + p.off_rr);
    const uint32_t Rc = p.Rc;
    if (RING) {
      rg = (ulonglong2*)p.ring_g + (size_t)slot * p.ring_stride;
      coh = (uint32_t*)(rr + Rc);
    }
    wslot = slot;
    if (SEG) {
      ga = p.seg_a + (size_t)slot * p.seg_cap;
      sa = (SRec*)(rr + Rc);
      hcnt = (uint32_t*)(sa + p.seg_cap);
      hsll = hcnt + p.hsize;
      hslp = hsll + p.hsize;
      con = hslp + p.hsize;
      col = con + p.csize;
    }
    rq = (uint32_t*)(base + p.warp_smem - p.n_rings * 80u);
    if (lane < p.n_rings) {  // this slot's chunk stash, kept in global memory between launches
      const uint4* g = reinterpret_cast<const uint4*>(p.pool_stash) + ((size_t)slot * p.n_rings + lane) * 3;
      for (int i = 0; i < 3; ++i) {  // count + kStash chunks = 12 words
        const uint4 sv = g[i];
        rq[20 * lane + 4 + 4 * i] = sv.x; rq[20 * lane + 5 + 4 * i] = sv.y;
        rq[20 * lane + 6 + 4 * i] = sv.z; rq[20 * lane + 7 + 4 * i] = sv.w;
      }
    }
  }

  __device__ void flush_acc() {
    flush_sums(st, lane, acc_arr, acc_done_a, acc_ft_a, (SEG || RING) ? acc_adm : 0ull,
               (SEG || RING) ? acc_ev : 0ull);
    acc_arr = acc_done_a = acc_ft_a = 0;
    if (SEG || RING) acc_adm = acc_ev = 0;
  }
  __device__ __forceinline__ void maybe_flush() {
    uint64_t m = acc_arr | acc_done_a | acc_ft_a;
    if (SEG || RING) m |= acc_adm | acc_ev;
    if (__any_sync(FULL, (m >> 60) != 0)) flush_acc();
  }

  // ------------------------------------------- restart FIFOs (chunk pool)
  // FIFO q holds positions [rhead, rtail) (lane q's counters) in a linked
  // list of kRestartChunk-entry chunks: rq[20q] = chunk of position rhead
  // (index rq[20q+1] = its position / kRestartChunk), rq[20q+2] = chunk of
  // the next write position rtail (index rq[20q+3]), rq[20q+16] / [20q+17] =
  // the successors of the head chunk and of the tail chunk (cached: a FIFO
  // spanning two chunks needs no link read).  Free chunks come from
  // a per-FIFO stash (rq[20q+4] = count, rq[20q+5..15] = chunks; one per warp
  // slot, kept in global memory between launches), else the device-wide
  // pool: a lock-free free stack of chunk chains (ABA tag in the high word),
  // else never-used chunks (handed out kBump at a time).  Passed and
  // released chunks go back to the stash, the overflow as ONE chain per
  // release (they are linked already): the free-stack head is one hot word,
  // so eviction-heavy runs (C4 rho >= 0.8, C5) must touch it rarely.
  static constexpr uint32_t kStash = 11, kBump = 4;  // count + kStash = 12 saved words (3 x uint4)
  __device__ uint32_t pool_alloc(int q) const {
    uint32_t* sq = rq + 20 * q;
    const uint32_t n = sq[4];
    if (n) { sq[4] = n - 1; return sq[4 + n]; }
    unsigned long long old = atomicAdd(P.pool_free, 0ull);
    while ((uint32_t)old != kNoChunk) {
      const uint32_t nxt = __ldcg(P.pool_next + (uint32_t)old);
      const unsigned long long nw = (((old >> 32) + 1ull) << 32) | nxt;
      const unsigned long long prev = atomicCAS(P.pool_free, old, nw);
      if (prev == old) return (uint32_t)old;
      old = prev;
    }
    const uint32_t c = atomicAdd(P.pool_bump, P.bump_n);
    if (c >= P.pool_chunks) return kNoChunk;
    // the rest of the batch goes to the stash (it is empty here)
    const uint32_t extra = min(P.bump_n, P.pool_chunks - c) - 1;
    for (uint32_t i = 0; i < extra; ++i) sq[5 + i] = c + 1 + i;
    sq[4] = extra;
    return c;
  }
  // push the chain first -> ... -> last (already linked) onto the free stack
  __device__ void pool_push_chain(uint32_t first, uint32_t last) const {
    unsigned long long old = atomicAdd(P.pool_free, 0ull);
    for (;;) {
      __stcg(P.pool_next + last, (uint32_t)old);
      __threadfence();
      const unsigned long long nw = (((old >> 32) + 1ull) << 32) | first;
      const unsigned long long prev = atomicCAS(P.pool_free, old, nw);
      if (prev == old) return;
      old = prev;
    }
  }
  // return the k linked chunks first -> ... (k >= 1) of FIFO q: to the stash
  // while it has room, the rest as one chain
  __device__ void pool_release_chain(int q, uint32_t first, uint32_t k) const {
    uint32_t* sq = rq + 20 * q;
    uint32_t n = sq[4];
    while (k > 0 && n < P.stash_lim) {
      sq[5 + n++] = first;
      if (--k) first = __ldcg(P.pool_next + first);
    }
    sq[4] = n;
    if (k == 0) return;
    uint32_t last = first;
    for (uint32_t i = 1; i < k; ++i) last = __ldcg(P.pool_next + last);
    pool_push_chain(first, last);
  }
  // pool entry of position pos (>= the committed head) of FIFO q
  __device__ __forceinline__ size_t fifo_entry(int q, uint32_t pos) const {
    const uint32_t want = pos / kRestartChunk, hi = rq[20 * q + 1];
    uint32_t c = rq[20 * q];
    if (want > hi) {  // the chunk after the head is cached (rq[20q+16]); further ones are walked
      c = rq[20 * q + 16];
      for (uint32_t ci = hi + 1; ci < want; ++ci) c = __ldcg(P.pool_next + c);
    }
    return (size_t)c * kRestartChunk + pos % kRestartChunk;
  }
  // pool entry of tail position pos (the tail chunk or the one after it)
  __device__ __forceinline__ size_t fifo_wentry(int q, uint32_t pos) const {
    uint32_t c = rq[20 * q + 2];
    if (pos / kRestartChunk != rq[20 * q + 3]) c = rq[20 * q + 17];  // reserved successor of the tail
    return (size_t)c * kRestartChunk + pos % kRestartChunk;
  }
  // lane q: chunks for cnt (<= 32) more entries at the tail t of FIFO q
  // (the chunk of the next write position included); false: pool exhausted
  __device__ bool fifo_reserve(int q, uint32_t t, uint32_t cnt) const {
    if (rq[20 * q + 2] == kNoChunk) {
      const uint32_t c = pool_alloc(q);
      if (c == kNoChunk) return false;
      rq[20 * q] = rq[20 * q + 2] = c;
      rq[20 * q + 1] = rq[20 * q + 3] = t / kRestartChunk;
      rq[20 * q + 16] = rq[20 * q + 17] = kNoChunk;
    }
    if ((t + cnt) / kRestartChunk > rq[20 * q + 3]) {
      const uint32_t c = pool_alloc(q);
      if (c == kNoChunk) return false;
      __stcg(P.pool_next + rq[20 * q + 2], c);
      rq[20 * q + 17] = c;
      if (rq[20 * q + 2] == rq[20 * q]) rq[20 * q + 16] = c;  // the head's successor
    }
    return true;
  }
  // lane q, after the writes: the tail chunk follows the new tail position
  __device__ void fifo_tail_done(int q, uint32_t t_new) const {
    if (t_new / kRestartChunk > rq[20 * q + 3]) {
      rq[20 * q + 2] = rq[20 * q + 17];
      rq[20 * q + 3] += 1;
      rq[20 * q + 17] = kNoChunk;
    }
  }
  // lane q: return the chunks the committed head has passed
  __device__ void fifo_commit(int q, uint32_t head) const {
    if (rq[20 * q + 2] == kNoChunk || rq[20 * q + 1] >= head / kRestartChunk) return;
    const uint32_t first = rq[20 * q], k = head / kRestartChunk - rq[20 * q + 1];
    uint32_t c = rq[20 * q + 16];  // the head's successor
    for (uint32_t i = 1; i < k; ++i) c = __ldcg(P.pool_next + c);
    rq[20 * q] = c;
    rq[20 * q + 1] += k;
    // successor of the new head: the tail's reserved successor, or a link
    rq[20 * q + 16] = c == rq[20 * q + 2] ? rq[20 * q + 17] : __ldcg(P.pool_next + c);
    pool_release_chain(q, first, k);
  }
  // lanes < n_rings: save the chunk stash of this slot (kernel exit)
  __device__ void flush_stash() const {
    if (lane < P.n_rings) {
      uint4* g = reinterpret_cast<uint4*>(P.pool_stash) + ((size_t)wslot * P.n_rings + lane) * 3;
      const uint32_t* sq = rq + 20 * lane;
      for (int i = 0; i < 3; ++i) g[i] = make_uint4(sq[4 + 4 * i], sq[5 + 4 * i], sq[6 + 4 * i], sq[7 + 4 * i]);
    }
  }
  // lane q: return every chunk of FIFO q (end of the replication)
  __device__ void fifo_release_all(int q) const {
    if (rq[20 * q + 2] == kNoChunk) return;
    const uint32_t k = rq[20 * q + 3] - rq[20 * q + 1] + 1;  // head chunk .. tail chunk
    pool_release_chain(q, rq[20 * q], k);
    rq[20 * q] = rq[20 * q + 2] = kNoChunk;
  }
  // NESTED stage info: segment index (bits 0-5), last stage of the segment
  // (bit 6), entry stage (bit 7); counter slot = segment (+32 at entry)
  __device__ __forceinline__ static uint32_t info_seg(uint32_t info) { return info & 0x3F; }
  __device__ __forceinline__ static uint32_t info_key(uint32_t info) {
    return (info & 0x3F) + ((info >> 7) ? 32u : 0u);
  }

  // ---------------------------------------------------- S1 arrival windows
  // Fill the 32 arrivals [base, base+32) of class c: lane i draws arrival
  // base+i from Philox counter (k, r, c, 0), gaps are
  // turned into ticks by an inclusive warp scan on top of `prev`.
  __device__ __forceinline__ bool is_tv(int c) const { return !TRACE && P.cls[c].rf_n != 0; }


  // S1 window fill: 32 arrivals [base, base+32) of class c into (wt, wl, wlp)
  // (+ operational time for time-varying classes).  Philox mode calls the
  // single non-inlined generator below; trace mode reads the explicit trace.
  template <bool WITH_LEN>
  __device__ __forceinline__ void fill(int c, uint32_t base, int64_t prev, int64_t* wt,
                                       uint16_t* wl, uint16_t* wlp) {
    const bool tv = is_tv(c);
    int64_t* wtau = tv ? (wt == vt ? vtau : atau) : nullptr;
    if (TRACE) {
      const uint32_t k = base + lane;
      const int64_t beg = P.tr_off[(size_t)rep * nK() + c];
      const int64_t end = P.tr_off[(size_t)rep * nK() + c + 1];
      int64_t t = TMAX;
      uint32_t l = 1, lp = 1;
      if (beg + (int64_t)k < end) {
        t = P.tr_t[beg + k];
        if (WITH_LEN) { l = P.tr_l[beg + k]; lp = P.tr_lp[beg + k]; }
      }
      __syncwarp();
      wt[c * 32 + lane] = t;
      if (WITH_LEN) { wl[c * 32 + lane] = (uint16_t)l; wlp[c * 32 + lane] = (uint16_t)lp; }
      __syncwarp();
      return;
    }
    const ClassParam& cp = P.cls[c];
    gen_window<POL == SCHED_WAIT && WAITSIM_WAIT_GEN_INL>(lane, base, prev, rglob, (uint32_t)c, P.seed, cp.gap_scale, P.cdf_thr, P.cdf_val,
               P.cdf_guide, cp.l_goff, cp.lp_goff, cp.l_off, cp.l_n, cp.lp_off, cp.lp_n, cp.rf_off, cp.rf_n, P.rf_B, P.rf_Lam,
               P.rf_scale, wt + c * 32, wl + c * 32, wlp + c * 32, wtau ? wtau + c * 32 : nullptr);
  }

  // class-c cursor fields (uniform broadcast from lane c)
  __device__ __forceinline__ uint32_t kvis(int c) const { return bcast32(k_vis, c); }
  __device__ __forceinline__ uint32_t kadm(int c) const { return bcast32(k_adm, c); }
  __device__ __forceinline__ uint32_t rcount(int q) const { return bcast32(rtail, q) - bcast32(rhead, q); }

  // scan carry of arrival k-1 of class c: its tick, or its operational time
  // for a time-varying class (k within the generated or private window)
  __device__ int64_t carry_before(int c, uint32_t k) const {
    if (k == 0) return 0;
    const bool tv = is_tv(c);
    const uint32_t vb = bcast32(vbase, c);
    if (k > vb) return (tv ? vtau : vt)[c * 32 + (k - 1 - vb)];
    if (k == vb) return bcast64(vprev, c);
    const uint32_t ab = bcast32(abase, c);
    if (k > ab) return (tv ? atau : at)[c * 32 + (k - 1 - ab)];
    return bcast64(aprev, c);
  }

  // ------------------------------------------------------ S2 ingestion
  // INGEST (DESIGN.md §4.4 step 1): arrivals with t <= now and t < T become
  // visible (join their FIFO).  Cursor only: count + arrival-time sum.
  // class c's window: arrivals due by `now` become visible; a consumed
  // window is refilled (the pending tail moves to the private window first)
  // (ACC: returns the number that became visible, else adds it to the stats)
  template <bool ACC>
  __device__ __forceinline__ uint32_t ingest_class(const int c) {
    uint32_t vis_n = 0;
    for (;;) {
      uint32_t kv = kvis(c), vb = bcast32(vbase, c);
      if (kv == vb + 32) {
        const uint32_t ka = kadm(c);
        if (ka >= vb && ka < vb + 32) {
          // pending arrivals of the old window move to the private window
          const uint32_t n = vb + 32 - ka, off = ka - vb;
          const int64_t prev = carry_before(c, ka);
          __syncwarp();
          if ((uint32_t)lane < n) {
            at[c * 32 + lane] = vt[c * 32 + off + lane];
            al[c * 32 + lane] = vl[c * 32 + off + lane];
            alp[c * 32 + lane] = vlp[c * 32 + off + lane];
            if (is_tv(c)) atau[c * 32 + lane] = vtau[c * 32 + off + lane];
          }
          __syncwarp();
          if (lane == c) { abase = ka; aprev = prev; pcount = n; }
        }
        const int64_t carry = (is_tv(c) ? vtau : vt)[c * 32 + 31];
        fill<true>(c, kv, carry, vt, vl, vlp);
        if (lane == c) { vbase = kv; vprev = carry; }
        vb = kv;
      }
      const uint32_t j = kv - vb;
      const int64_t t = vt[c * 32 + lane];
      const bool vis = (uint32_t)lane >= j && t <= now && t < P.T_t;
      const uint32_t n = __popc(__ballot_sync(FULL, vis));
      if (vis) acc_arr += (uint64_t)t;
      if (ACC) vis_n += n;
      else if (lane == 0) st->arrivals += n;
      if (lane == c) k_vis += n;
      if (j + n < 32) break;
      maybe_flush();  // a long backlog: one more tick per lane per window
    }
    return vis_n;
  }

  __device__ void ingest() {
    // specialised FCFS, K <= 3: the classes unrolled (offsets are immediates;
    // C2 FCFS 16.8 -> 15.7 ms, spills 220 -> 108 B; C4 K = 3 -3%; K = 4 loses:
    // C3a FCFS 52 -> 62 ms).  Not WAIT: it inlines the window
    // generator, and two inlined copies cost more than they save (13.7 -> 15.1 ms)
    if (KC > 0 && KC <= 3 && POL != SCHED_WAIT) {
      uint32_t n = 0;
#pragma unroll
      for (int c = 0; c < KC; ++c) n += ingest_class<true>(c);
      if (lane == 0) st->arrivals += n;
      return;
    }
    // only classes whose next window entry is due (lane c: entry k_vis; the
    // window always holds it, it is refilled before k_vis reaches its end)
    // (with one or two classes both are usually due: skip the test)
    bool due = lane < nK();
    if (nK() > 2 && due) {
      const int64_t t = vt[lane * 32 + (k_vis - vbase)];
      due = t <= now && t < P.T_t;
    }
    for (uint32_t todo = __ballot_sync(FULL, due); todo; todo &= todo - 1) ingest_class<false>(__ffs(todo) - 1);
  }

  // next not-yet-visible arrival tick (< T), TMAX if none
  __device__ int64_t next_arrival() const {
    int64_t best = TMAX;
    for (int c = 0; c < nK(); ++c) {
      const int64_t t = vt[c * 32 + (kvis(c) - bcast32(vbase, c))];
      if (t < P.T_t && t < best) best = t;
    }
    return best;
  }

  __device__ __forceinline__ static int64_t warp_min_i64(int64_t x) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) x = min(x, (int64_t)__shfl_xor_sync(FULL, (long long)x, d));
    return x;
  }

  // Idle skip.  While no batch can start because of the threshold test
  // (WAIT: no type has n_j waiting, line 1488; NESTED: fewer than n_1 wait,
  // line 1640), residents do not move and only arrivals change the decision,
  // so the epochs at the intermediate arrivals are no-ops whose idle time
  // adds up (DESIGN.md §4.4 step 3): jump straight to the arrival that can
  // start a batch.  Exact within the generated windows, else to the last
  // arrival every window still holds (an earlier epoch; ingest refills).
  __device__ int64_t idle_jump() const {
    int64_t bound = lane < nK() ? vt[lane * 32 + 31] : TMAX;
    if (POL == SCHED_WAIT || nK() == 1) {  // per FIFO: the (n - q)-th next arrival of its class
      int64_t cand = TMAX;
      if (lane < nK()) {
        const uint32_t q = k_vis - k_adm + (rtail - rhead);  // < n_j (type not qualifying)
        const uint32_t j = (k_vis - vbase) + (P.thr[lane] - q) - 1;
        cand = j < 32 ? vt[lane * 32 + j] : bound;
      }
      return warp_min_i64(cand);
    } else {
      bound = warp_min_i64(bound);
      uint32_t d = P.thr[0] - waiting_total();  // >= 1 arrivals still needed
      uint32_t ptr = lane < nK() ? k_vis - vbase : 32u;
      for (;;) {
        const int64_t h = ptr < 32 ? vt[lane * 32 + ptr] : TMAX;
        const int64_t m = warp_min_i64(h);
        if (m >= bound || --d == 0) return min(m, bound);
        if ((uint32_t)lane == (uint32_t)__ffs(__ballot_sync(FULL, h == m)) - 1) ++ptr;
      }
    }
  }

  __device__ uint32_t waiting_total() const {
    uint32_t w = lane < nK() ? k_vis - k_adm : 0u;
    if (lane < (POL == SCHED_WAIT ? nK() : 1)) w += rtail - rhead;
    return __reduce_add_sync(FULL, w);
  }

  // ------------------------------------------------------- admissions
  // Take up to `want` prompts from the head of FIFO q, in FIFO order, and
  // stage them at resident slots n_res + n_new ... (prefill -> stage 1).
  // WAIT: FIFO q = class q's arrivals + restart ring q; otherwise one FIFO
  // = all classes' arrivals + ring 0.  FIFO order: arrivals by (t, class);
  // a restart evicted at tick e precedes exactly the arrivals with t > e
  // (DESIGN.md §4.4).  Lane-parallel: each candidate's FIFO rank is the
  // number of candidates before it (binary searches over the other sources'
  // windows); FCFS additionally cuts at the first prompt failing the
  // admission test (reading R15).
  // first staging slot: after the residents (member engine) or 0 (RING)
  __device__ __forceinline__ uint32_t sbase() const { return (RING || SEG) ? 0u : n_res; }

  // FCFS admission cut: lane i holds staged candidate i (prefill length l);
  // the longest prefix passing the test of PAPER.md:1427, 1745 (R15)
  __device__ __forceinline__ uint32_t fcfs_take(uint32_t m, uint32_t l) const {
    const uint32_t pre = warp_incl_scan_u32(l, lane);
    // uniform limits: KV room (Sarathi-style ongoing-first also reserves the
    // residents' growth, R29), prefill-token budget, resident slots
    int64_t room = P.M - KV - (POL == SCHED_FCFS_ONGOING ? (int64_t)n_res : 0) - sum_new_l;
    if (P.tok_budget) room = min(room, (int64_t)P.tok_budget - sum_new_l);
    const uint32_t used = n_res + n_new, slots = P.B > used ? P.B - used : 0u;
    const bool ok = (uint32_t)lane < min(m, slots) && (int64_t)pre <= room;
    const uint32_t okm = __ballot_sync(FULL, ok);  // ok lanes form a prefix
    return okm == FULL ? 32u : (uint32_t)__ffs(~okm) - 1;
  }

  // take_fifo fast path, one source class c (WAIT, or a single class): the
  // FIFO head is arrivals k_adm .. of class c, read in order from its
  // windows.  Returns -1 capacity error, 0 done, 1 took a full chunk.
  // the first (<= 32) waiting arrivals of a class: window offsets o1 ..
  // o1+len1-1, then o2 ..
  struct Seg {
    uint32_t o1, len1, o2;
    __device__ __forceinline__ uint32_t at(uint32_t i) const { return i < len1 ? o1 + i : o2 + (i - len1); }
    __device__ __forceinline__ Seg from(int c) const {
      return Seg{__shfl_sync(FULL, o1, c), __shfl_sync(FULL, len1, c), __shfl_sync(FULL, o2, c)};
    }
  };
  // # of the first n candidates of segment sg with tick <= key (le) or < key
  __device__ __forceinline__ uint32_t count_before_seg(const Seg& sg, uint32_t n, int64_t key, bool le) const {
    uint32_t lo = 0, len = n;
    while (len > 0) {
      const uint32_t half = len >> 1;
      const int64_t x = vt[sg.at(lo + half)];
      if (le ? (x <= key) : (x < key)) { lo += half + 1; len -= half + 1; } else { len = half; }
    }
    return lo;
  }

  template <bool FCFS_COND>
  __device__ __forceinline__ int take_single(int c, uint32_t pend, const Seg& sgl, uint32_t& want) {
    const uint32_t p = bcast32(pend, c);
    const Seg sg = sgl.from(c);
    const uint32_t base = sbase() + n_new;
    uint32_t m = min(p, want);
    if (FCFS_COND) m = min(m, P.B > base ? P.B - base : 0u);
    if (m == 0) return 0;
    if (base + m > P.Rc) { status = 1; return -1; }
    uint32_t l = 0;
    if ((uint32_t)lane < m) {
      const uint32_t idx = sg.at((uint32_t)lane);
      // (class-ring engine: the class fixes l, l')
      l = RING ? (P.fl[c] & 0xFFFFu) : vl[idx];
      rr[base + lane] = Rec{vt[idx], pack_q(l, RING ? (P.fl[c] >> 16) : vlp[idx], 1, (uint32_t)c)};
    }
    const uint32_t take = FCFS_COND ? fcfs_take(m, l) : m;
    if (lane == c) { k_adm += take; newc += take; }
    n_new += take;
    sum_new_l += __reduce_add_sync(FULL, (uint32_t)lane < take ? l : 0u);
    want -= take;
    __syncwarp();
    return take < m ? 0 : m < p ? 1 : 2;
  }

  // take_fifo fast path, several classes merged by (t, class): candidate g
  // of class s ranks pos + #(earlier arrivals of the other classes), by
  // binary search over their windows.  Returns -1 capacity error, 0 done,
  // 1 took a full chunk (more may follow).
  template <bool FCFS_COND>
  __device__ __forceinline__ int take_merged(uint32_t pend, const Seg& my, uint32_t& want) {
    const uint32_t incl = warp_incl_scan_u32(pend, lane);  // lanes >= K: pend = 0
    const uint32_t ncand = __shfl_sync(FULL, incl, 31);
    if (ncand == 0) return 0;
    const uint32_t base = sbase() + n_new;
    uint32_t m = min(min(ncand, 32u), want);
    if (FCFS_COND) m = min(m, P.B > base ? P.B - base : 0u);
    if (m == 0) return 0;
    if (base + m > P.Rc) { status = 1; return -1; }
    const int K = nK();
    for (uint32_t g0 = 0; g0 < ncand; g0 += 32) {
      const uint32_t g = g0 + (uint32_t)lane;
      const bool act = g < ncand;
      int s = 0;  // source class: first class whose candidate range ends after g
      for (int c = 0; c < K; ++c) s += bcast32(incl, c) <= g;
      s = min(s, K - 1);
      const uint32_t s_n = __shfl_sync(FULL, pend, s);
      const Seg ss{__shfl_sync(FULL, my.o1, s), __shfl_sync(FULL, my.len1, s), __shfl_sync(FULL, my.o2, s)};
      const uint32_t pos = g - (__shfl_sync(FULL, incl, s) - s_n);
      const uint32_t idx = ss.at(pos);
      const int64_t t = act ? vt[idx] : 0;
      uint32_t r = pos;
      for (int c = 0; c < K; ++c) {
        const uint32_t n = bcast32(pend, c);
        const Seg sc = my.from(c);
        // ties: a lower class index precedes
        if (act && c != s && n) r += count_before_seg(sc, n, t, c < s);
      }
      if (act && r < m) {
        rr[base + r] = Rec{t, pack_q(vl[idx], vlp[idx], 1, (uint32_t)s)};
      }
    }
    __syncwarp();
    uint64_t qv = 0;
    uint32_t l = 0;
    if ((uint32_t)lane < m) { qv = rr[base + lane].q; l = (uint32_t)(qv & 0xFFFF); }
    const uint32_t take = FCFS_COND ? fcfs_take(m, l) : min(m, want);
    if (take == 0) return 0;
    const bool tk = (uint32_t)lane < take;
    const uint32_t cls = (uint32_t)(qv >> 48) & 0xFF;
    for (int c = 0; c < K; ++c) {
      const uint32_t cc = __popc(__ballot_sync(FULL, tk && cls == (uint32_t)c));
      if (lane == c) { k_adm += cc; newc += cc; }
    }
    n_new += take;
    sum_new_l += __reduce_add_sync(FULL, tk ? l : 0u);
    want -= take;
    __syncwarp();
    return take < m ? 0 : m < ncand ? 1 : 2;
  }

  // take_merged for KK <= 4 classes: each class's candidates (lane i = its
  // i-th waiting arrival) rank i + #(earlier arrivals of the other classes),
  // ties to the lower class index
  template <bool FCFS_COND, int KK>
  __device__ __forceinline__ int take_merged_k(uint32_t pend, const Seg& my, uint32_t& want) {
    uint32_t n[KK];
    Seg sg[KK];
    uint32_t ncand = 0;
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      n[c] = __shfl_sync(FULL, pend, c);
      sg[c] = my.from(c);
      ncand += n[c];
    }
    if (ncand == 0) return 0;
    const uint32_t base = sbase() + n_new;
    uint32_t m = min(min(ncand, 32u), want);
    if (FCFS_COND) m = min(m, P.B > base ? P.B - base : 0u);
    if (m == 0) return 0;
    if (base + m > P.Rc) { status = 1; return -1; }
    const uint32_t i = (uint32_t)lane;
    if (KK == 2) {
      // lane i holds both classes' i-th candidates; each candidate's rank
      // i + #(earlier arrivals of the other class) by a branch-free binary
      // search over the other class's ticks held in lanes (shuffles; ties
      // to class 0)
      uint32_t i0 = 0, i1 = 0;
      int64_t t0 = TMAX, t1 = TMAX;
      if (i < n[0]) { i0 = sg[0].at(i); t0 = vt[i0]; }
      if (i < n[1]) { i1 = sg[1].at(i); t1 = vt[i1]; }
      uint32_t r0 = 0, r1 = 0;  // # of class-1 ticks < t0, # of class-0 ticks <= t1
#pragma unroll
      for (uint32_t step = 32; step >= 1; step >>= 1) {
        const int64_t x1 = __shfl_sync(FULL, t1, (int)((r0 + step - 1) & 31u));
        const int64_t x0 = __shfl_sync(FULL, t0, (int)((r1 + step - 1) & 31u));
        if (r0 + step <= n[1] && x1 < t0) r0 += step;
        if (r1 + step <= n[0] && x0 <= t1) r1 += step;
      }
      r0 += i;
      r1 += i;
      // (class-ring engine: the class fixes l, l' -- uniform constants, no window reads)
      if (i < n[0] && r0 < m)
        rr[base + r0] = Rec{t0, RING ? pack_q(P.fl[0] & 0xFFFFu, P.fl[0] >> 16, 1, 0u) : pack_q(vl[i0], vlp[i0], 1, 0u)};
      if (i < n[1] && r1 < m)
        rr[base + r1] = Rec{t1, RING ? pack_q(P.fl[1] & 0xFFFFu, P.fl[1] >> 16, 1, 1u) : pack_q(vl[i1], vlp[i1], 1, 1u)};
    } else {
#pragma unroll
    for (int src = 0; src < KK; ++src) {
      if (i < n[src] && i < m) {
        const uint32_t idx = sg[src].at(i);
        const int64_t t = vt[idx];
        uint32_t r = i;
#pragma unroll
        for (int c = 0; c < KK; ++c) {
          if (c == src || n[c] == 0) continue;
          uint32_t lo = 0, len = n[c];
          while (len > 0) {
            const uint32_t half = len >> 1;
            const int64_t x = vt[sg[c].at(lo + half)];
            if (c < src ? (x <= t) : (x < t)) { lo += half + 1; len -= half + 1; } else { len = half; }
          }
          r += lo;
        }
        if (r < m) rr[base + r] = Rec{t, pack_q(vl[idx], vlp[idx], 1, (uint32_t)src)};
      }
    }
    }
    __syncwarp();
    uint64_t qv = 0;
    uint32_t l = 0;
    if ((uint32_t)lane < m) { qv = rr[base + lane].q; l = (uint32_t)(qv & 0xFFFF); }
    const uint32_t take = FCFS_COND ? fcfs_take(m, l) : min(m, want);
    if (take == 0) return 0;
    const bool tk = (uint32_t)lane < take;
    const uint32_t cls = (uint32_t)(qv >> 48) & 0xFF;
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      const uint32_t cc = __popc(__ballot_sync(FULL, tk && cls == (uint32_t)c));
      if (lane == c) { k_adm += cc; newc += cc; }
    }
    n_new += take;
    sum_new_l += __reduce_add_sync(FULL, tk ? l : 0u);
    want -= take;
    __syncwarp();
    return take < m ? 0 : m < ncand ? 1 : 2;
  }

  template <bool FCFS_COND>
  __device__ bool take_fifo(int q, uint32_t want) {
    const int c_lo = POL == SCHED_WAIT ? q : 0;
    const int c_hi = POL == SCHED_WAIT ? q + 1 : nK();
    while (want > 0) {
      // fast path (the common case): no restart waits in FIFO q and every
      // class's waiting arrivals sit in its generated window (backlog <= 32,
      // "attached"); lane c already holds class c's cursors
      {
        const bool in_rng = lane >= c_lo && lane < c_hi;
        const uint32_t pend = in_rng ? k_vis - k_adm : 0u;
        // class `lane`'s waiting arrivals as offsets: the generated window
        // (attached) or the private window continuing into it
        uint32_t o1 = 0, len1 = 32, o2 = 0;
        bool ok = lane != q || rtail == rhead;
        if (pend) {
          if (k_adm >= vbase) {
            o1 = lane * 32 + (k_adm - vbase);
          } else if (k_adm >= abase && abase + pcount == vbase) {
            o1 = (nK() + lane) * 32 + (k_adm - abase);
            len1 = abase + pcount - k_adm;
            o2 = lane * 32;
          } else {
            ok = false;
          }
        }
        if (__all_sync(FULL, ok)) {
          const Seg sg{o1, len1, o2};
          // each class offers its first min(pending, want, 32) arrivals: a
          // candidate's rank is at least its index in its class, so ranks
          // below `want` stay exact; when none was capped,
          // taking every offered one ends the admissions
          const uint32_t cap = min(want, 32u);
          const bool capped = __any_sync(FULL, pend > cap);
          if (c_hi - c_lo == 1) {
            const int r = take_single<FCFS_COND>(c_lo, min(pend, cap), sg, want);
            if (r < 0) return false;
            if (r == 0 || (r == 2 && !capped)) break;
            continue;
          }
          // FCFS admits whole chunks: per-class ranking wins for K <= 4
          // (measured C2 FCFS +12%, C4 +8-10%); Nested takes n_1 <= few
          const uint32_t pc = min(pend, cap);
          const int r = !FCFS_COND ? take_merged<FCFS_COND>(pc, sg, want)
                      : nK() == 2 ? take_merged_k<FCFS_COND, 2>(pc, sg, want)
                      : nK() == 3 ? take_merged_k<FCFS_COND, 3>(pc, sg, want)
                      : nK() == 4 ? take_merged_k<FCFS_COND, 4>(pc, sg, want)
                                 : take_merged<FCFS_COND>(pc, sg, want);
          if (r < 0) return false;
          if (r == 0 || (r == 2 && !capped)) break;
          continue;
        }
      }
      // (1) each class's candidate window = its first min(pending, 32)
      // waiting arrivals, as up to two sorted segments: private window part
      // (or the generated window when attached) + the generated window
      // continuing it.  Lane c keeps class c's descriptor.
      uint32_t my_o1 = 0, my_n1 = 0, my_n2 = 0, my_priv = 0, my_n = 0, total = 0;
      for (int c = c_lo; c < c_hi; ++c) {
        const uint32_t ka = kadm(c);
        const uint32_t p = kvis(c) - ka;
        if (p == 0) continue;
        const uint32_t vb = bcast32(vbase, c);
        uint32_t o1, n1, n2 = 0, priv = 0;
        if (ka >= vb) {
          o1 = ka - vb;
          n1 = p;  // k_vis <= vbase + 32
        } else {
          priv = 1;
          const uint32_t ab = bcast32(abase, c), pc = bcast32(pcount, c);
          o1 = ka - ab;
          n1 = min(p, pc - o1);
          if (n1 < p && ab + pc == vb) n2 = min(p - n1, 32u - n1);
          // ranks < m <= min(want, 32) are exact when every source offers
          // min(pending, want, 32) candidates
          if (n1 + n2 < min(p, min(want, 32u))) {
            // backlog deeper than the windows: regenerate the private window
            const int64_t prev = carry_before(c, ka);
            if (lane == c) save_carry();  // before the saved cursor's carry can leave the windows
            fill<true>(c, ka, prev, at, al, alp);
            if (lane == c) { abase = ka; aprev = prev; pcount = 32; }
            o1 = 0;
            n1 = min(p, 32u);
            n2 = 0;
          }
        }
        if (lane == c) { my_o1 = o1; my_n1 = n1; my_n2 = n2; my_priv = priv; my_n = n1 + n2; }
        total += n1 + n2;
      }
      const uint32_t nr = min(rcount(q), 32u);
      const uint32_t h0 = bcast32(rhead, q);
      // lane i: restart i's eviction tick (to shared memory, for the ranks)
      // and, in the same round trip, its arrival tick and lengths (shuffled
      // to the candidate that stages it)
      int64_t r_a = 0;
      uint32_t r_llp = 0;
      if (nr > 0) {
        __syncwarp();
        if ((uint32_t)lane < nr) {
          const size_t en = fifo_entry(q, h0 + lane);
          re[lane] = __ldcg(P.pool_e + en);
          if (kEarlyRestart) {
            r_a = __ldcg(P.pool_a + en);
            r_llp = __ldcg(P.pool_llp + en);
          }
        }
        __syncwarp();
      }
      const uint32_t ncand = total + nr;
      if (ncand == 0) break;
      const uint32_t base = sbase() + n_new;
      // stage at most what can be taken: `want` (WAIT/NESTED) or the B bound (FCFS)
      uint32_t m = min(min(ncand, 32u), want);
      if (FCFS_COND) m = min(m, P.B > base ? P.B - base : 0u);
      if (m == 0) break;
      if (base + m > P.Rc) { status = 1; return false; }
      // (2) rank candidates; rank < m -> staged at slot base + rank
      if (POL == SCHED_WAIT || (POL != SCHED_NESTED && KC == 1)) {
        // WAIT (FIFO q = class q + its restarts) or one-class FCFS: lane i holds arrival i
        // and restart i; both sources are sorted (ticks; eviction ticks in
        // FIFO order), so each rank is i + a count in the other source,
        // found by a branch-free binary search over lanes (shuffles).  A
        // restart evicted at e precedes exactly the arrivals with t > e
        // (DESIGN.md §4.4).  C1 FCFS 85.6 -> 71.5 ms.  The restarts' pool records are requested before
        // the search so their latency overlaps it.  (C4 rho = 0.9 / 0.95 WAIT
        // 2.86 / 1.93 -> 2.49 / 1.83 ms; the same merge for Nested K = 1 lost:
        // C5 584 -> 622 ms.)
        const int c = c_lo;
        const uint32_t n = bcast32(my_n, c), n1 = bcast32(my_n1, c), o1 = bcast32(my_o1, c);
        const bool priv = bcast32(my_priv, c) != 0;
        const uint32_t i = (uint32_t)lane;
        int64_t t = TMAX;
        uint32_t al_ = 0, alp_ = 0;
        if (i < n) {
          int idx;
          const int64_t* tt;
          const uint16_t *ll, *llp;
          if (i < n1) {
            idx = c * 32 + (int)(o1 + i);
            tt = priv ? at : vt; ll = priv ? al : vl; llp = priv ? alp : vlp;
          } else {
            idx = c * 32 + (int)(i - n1);
            tt = vt; ll = vl; llp = vlp;
          }
          t = tt[idx]; al_ = ll[idx]; alp_ = llp[idx];
        }
        const int64_t e = i < nr ? re[i] : TMAX;
        int64_t ra_a = 0;
        uint32_t ra_llp = 0;
        if (i < nr) {
          const size_t en = fifo_entry(q, h0 + i);
          ra_a = __ldcg(P.pool_a + en);
          ra_llp = __ldcg(P.pool_llp + en);
        }
        uint32_t ra = 0, rb = 0;  // restarts with e < t, arrivals with t <= e
#pragma unroll
        for (uint32_t step = 32; step >= 1; step >>= 1) {
          const int64_t xe = __shfl_sync(FULL, e, (int)((ra + step - 1) & 31u));
          const int64_t xt = __shfl_sync(FULL, t, (int)((rb + step - 1) & 31u));
          if (ra + step <= nr && xe < t) ra += step;
          if (rb + step <= n && xt <= e) rb += step;
        }
        ra += i;
        rb += i;
        if (i < n && ra < m) rr[base + ra] = Rec{t, pack_q(al_, alp_, 1, (uint32_t)c)};
        if (i < nr && rb < m) {
          const int64_t a = ra_a;
          const uint32_t llp = ra_llp;
          uint32_t cls = POL == SCHED_WAIT ? (uint32_t)q : 0u, l = 0, lp = 0;
          if (RING) {  // {class, ft}: the class fixes l, l'
            cls = llp & 0xFFu;
            l = P.fl[cls] & 0xFFFFu; lp = P.fl[cls] >> 16;
          } else {
            l = llp & 0xFFFFu; lp = (llp >> 16) & 0x7FFFu;
          }
          rr[base + rb] = Rec{a, pack_q(l, lp, 1, cls | ((llp >> 31) ? META_FT : 0u) | META_RESTART)};
        }
      } else
      for (uint32_t g0 = 0; g0 < ncand; g0 += 32) {
        const uint32_t g = g0 + lane;
        const bool act = g < ncand;
        int src = 32;
        uint32_t pos = 0, acc = 0;
        for (int c = c_lo; c < c_hi; ++c) {
          const uint32_t n = bcast32(my_n, c);
          if (src == 32 && g >= acc && g < acc + n) { src = c; pos = g - acc; }
          acc += n;
        }
        if (src == 32) pos = g - acc;
        const uint32_t s_o1 = __shfl_sync(FULL, my_o1, src & 31);
        const uint32_t s_n1 = __shfl_sync(FULL, my_n1, src & 31);
        const uint32_t s_priv = __shfl_sync(FULL, my_priv, src & 31);
        int64_t ra_s = 0;
        uint32_t rllp_s = 0;
        if (kEarlyRestart) {
          ra_s = __shfl_sync(FULL, r_a, (int)(pos & 31u));
          rllp_s = __shfl_sync(FULL, r_llp, (int)(pos & 31u));
        }
        int64_t key = 0, a = 0;
        uint32_t l = 0, lp = 0, meta = 0, r = pos;
        if (act) {
          if (src < 32) {
            int idx;
            const int64_t* tt;
            const uint16_t *ll, *llp;
            if (pos < s_n1) {
              idx = src * 32 + (int)(s_o1 + pos);
              tt = s_priv ? at : vt; ll = s_priv ? al : vl; llp = s_priv ? alp : vlp;
            } else {
              idx = src * 32 + (int)(pos - s_n1);
              tt = vt; ll = vl; llp = vlp;
            }
            key = tt[idx]; a = key; l = ll[idx]; lp = llp[idx]; meta = (uint32_t)src;
            r += count_before(re, nr, key, false);       // restarts with e < t
          } else {
            key = re[pos];
            uint32_t llp = rllp_s;
            a = ra_s;
            if (!kEarlyRestart) {
              const size_t e = fifo_entry(q, h0 + pos);
              a = __ldcg(P.pool_a + e);
              llp = __ldcg(P.pool_llp + e);
            }
            uint32_t cls = POL == SCHED_WAIT ? (uint32_t)q : 0u;
            if (RING) {  // {class, ft}: the class fixes l, l'
              cls = llp & 0xFFu;
              l = P.fl[cls] & 0xFFFFu; lp = P.fl[cls] >> 16;
            } else {
              l = llp & 0xFFFFu; lp = (llp >> 16) & 0x7FFFu;
            }
            meta = cls | ((llp >> 31) ? META_FT : 0u) | META_RESTART;
          }
        }
        for (int c = c_lo; c < c_hi; ++c) {
          const uint32_t n = bcast32(my_n, c);
          if (n == 0) continue;
          const uint32_t n1 = bcast32(my_n1, c), o1 = bcast32(my_o1, c);
          const int64_t* seg1 = (bcast32(my_priv, c) ? at : vt) + c * 32 + o1;
          if (act && c != src) {  // arrivals of class c before this candidate
            const bool le = src == 32 || c < src;
            uint32_t k = count_before(seg1, n1, key, le);
            if (k == n1 && n > n1) k += count_before(vt + c * 32, n - n1, key, le);
            r += k;
          }
        }
        if (act && r < m) {
          rr[base + r] = Rec{a, pack_q(l, lp, 1, meta)};
        }
      }
      __syncwarp();
      // (3) how many to take
      uint64_t qv = 0;
      uint32_t l = 0;
      if ((uint32_t)lane < m) { qv = rr[base + lane].q; l = (uint32_t)(qv & 0xFFFF); }
      const uint32_t take = FCFS_COND ? fcfs_take(m, l) : min(m, want);
      if (take == 0) break;
      // (4) consume: advance each source's cursor by what it contributed
      const bool tk = (uint32_t)lane < take;
      const uint32_t meta = (uint32_t)(qv >> 48);
      const bool rst = tk && (meta & META_RESTART);
      for (int c = c_lo; c < c_hi; ++c) {
        const uint32_t cc = __popc(__ballot_sync(FULL, tk && !(meta & META_RESTART) && (meta & 0xFF) == (uint32_t)c));
        if (lane == c) { k_adm += cc; newc += cc; }
      }
      const uint32_t crs = __popc(__ballot_sync(FULL, rst));
      if (lane == q) { rhead += crs; if (POL == SCHED_WAIT) newc += crs; }
      if (rst) rr[base + lane].q = qv & ~((uint64_t)META_RESTART << 48);
      n_new += take;
      sum_new_l += __reduce_add_sync(FULL, tk ? l : 0u);
      want -= take;
      __syncwarp();
      if (take < m) break;
    }
    return true;
  }

  // save / restore the admission cursors (rare: a drop after eviction)
  // (the scan carry of the saved cursor is read lazily: only a private-
  // window regeneration during the takes, or a restore, needs it)
  __device__ void save_cursors() {
    sv_k = k_adm;
    sv_rhead = rhead;
    sv_have = 0;
    newc = 0;
  }
  // lane < K: the scan carry of arrival sv_k - 1 of class `lane` from the
  // windows (unchanged since save_cursors unless sv_have)
  __device__ void save_carry() {
    if (lane < nK() && !sv_have) {
      sv_prev = 0;
      if (sv_k > 0) {
        const bool tv = is_tv(lane);
        if (sv_k > vbase) sv_prev = (tv ? vtau : vt)[lane * 32 + (sv_k - 1 - vbase)];
        else if (sv_k == vbase) sv_prev = vprev;
        else if (sv_k > abase) sv_prev = (tv ? atau : at)[lane * 32 + (sv_k - 1 - abase)];
        else sv_prev = aprev;
      }
      sv_have = 1;
    }
  }
  __device__ void restore_cursors() {
    save_carry();
    for (int c = 0; c < nK(); ++c) {
      const uint32_t k = bcast32(sv_k, c);
      const int64_t pv = bcast64(sv_prev, c);
      const uint32_t ab = bcast32(abase, c), pc = bcast32(pcount, c);
      if (k < bcast32(vbase, c) && !(k >= ab && k <= ab + pc)) {
        fill<true>(c, k, pv, at, al, alp);
        if (lane == c) { abase = k; aprev = pv; pcount = 32; }
      }
      if (lane == c) k_adm = k;
    }
    rhead = sv_rhead;
    newc = 0;
  }

  // ---------------------------------------------------- S3 decide + take
  __device__ bool take_wait(uint32_t limit) {
    for (int c = 0; c < nK() && limit > 0; ++c) {
      if (!((Qmask >> c) & 1u)) continue;
      const uint32_t want = min(P.thr[c], limit);
      limit -= want;
      if (!take_fifo<false>(c, want)) return false;
    }
    return true;
  }

  __device__ bool decide() {
    n_new = 0;
    sum_new_l = 0;
    below = false;
    if (POL == SCHED_WAIT) {
      // Algorithm 1: type j joins the batch iff n_j0 >= n_j;
      // all residents of qualifying types ride along (line 1490, invariant P14)
      uint32_t qq = 0, npr = 0;
      if (lane < nK()) {
        const uint32_t w = k_vis - k_adm + (rtail - rhead);
        if (w >= P.thr[lane]) { qq = 1; npr = RING ? r_n : cnt[lane]; }
      }
      Qmask = __ballot_sync(FULL, qq);
      if (!Qmask) { below = true; return false; }
      n_plan_res = __reduce_add_sync(FULL, npr);
      save_cursors();
      return take_wait(0xFFFFFFFFu);
    } else if (POL == SCHED_NESTED) {
      // Algorithm 2: largest k with Q_{k',entry} >= n_k' for all k' <= k
      // (PAPER.md:1640); batch min{n_k, Q_{k,s}} per stage (line 1642)
      if (waiting_total() < P.thr[0]) { below = true; return false; }
      const uint32_t q_entry = SEG ? g_nen : cnt[32 + lane];  // residents waiting at segment lane's entry stage
      const bool pass = lane >= 1 && lane < P.n_seg && q_entry >= P.thr[lane];
      const uint32_t fail = ~__ballot_sync(FULL, pass) & ~1u;  // bit 0 = segment 1 (passed)
      const int ks = min(__ffs(fail) - 2, P.n_seg - 1);
      kstar = ks;
      uint32_t npr = 0;
      if (lane <= ks) {
        npr = SEG ? g_nne : cnt[lane];
        if (lane >= 1) npr += min(q_entry, P.thr[lane]);
      }
      n_plan_res = __reduce_add_sync(FULL, npr);
      save_cursors();
      return take_fifo<false>(0, P.thr[0]);
    } else {
      // FCFS new-first (R15)
      n_plan_res = n_res;
      if (!take_fifo<true>(0, 0xFFFFFFFFu)) return false;
      return n_res + n_new > 0;
    }
  }

  // --------------------------------------- S4 memory check / LIFO eviction
  __device__ void memory(uint32_t& n_evict, int64_t& peak) {
    peak = KV + (int64_t)n_plan_res + sum_new_l;
    if (peak <= P.M) return;
    int64_t excess = peak - P.M;
    const uint32_t old_n = n_res;
    if (POL == SCHED_NESTED) { rank[lane] = 0; snap[lane] = cnt[32 + lane]; __syncwarp(); }
    while (excess > 0 && n_res > 0) {
      const int idx = (int)n_res - 1 - lane;  // lane 0 = last admitted
      const bool valid = idx >= 0;
      uint64_t qv = 0;
      int64_t a = 0;
      if (valid) { const Rec e = rr[idx]; qv = e.q; a = e.a; }
      const uint32_t l = (uint32_t)(qv & 0xFFFF), lp = (uint32_t)((qv >> 16) & 0xFFFF);
      const uint32_t s = (uint32_t)((qv >> 32) & 0xFFFF), meta = (uint32_t)(qv >> 48);
      uint32_t inp = 0, nkey = 0;
      if (POL == SCHED_FCFS || POL == SCHED_FCFS_ONGOING) inp = valid;
      if (POL == SCHED_WAIT) inp = valid && ((Qmask >> (meta & 0xFF)) & 1u);
      if (POL == SCHED_NESTED) {
        const uint32_t info = valid ? __ldg(P.stage_info + s) : 0u;
        const int seg = info_seg(info);
        nkey = info_key(info);
        const bool entry = valid && (info >> 7) && seg <= kstar;
        const uint32_t key = entry ? s : (0x10000u + lane);
        const uint32_t grp = __match_any_sync(FULL, key);
        if (valid && seg <= kstar) {
          if (entry) {
            const uint32_t after = rank[seg] + __popc(grp & lanemask_lt());
            inp = snap[seg] - 1 - after < P.thr[seg];  // rank from the head
          } else {
            inp = 1;
          }
        }
        __syncwarp();
        if (entry && (grp & lanemask_lt()) == 0) rank[seg] += __popc(grp);
        __syncwarp();
      }
      const uint32_t f = valid ? (l + s - 1 + inp) : 0u;
      const uint32_t cum = warp_incl_scan_u32(f, lane);
      const uint32_t hit = __ballot_sync(FULL, valid && (int64_t)cum >= excess);
      const uint32_t ne = hit ? (uint32_t)__ffs(hit) : min(n_res, 32u);
      const bool ev = (uint32_t)lane < ne;
      // restart records in eviction order (re-enter the queue)
      const int q = POL == SCHED_WAIT ? (int)(meta & 0xFF) : 0;
      const uint32_t key = ev ? (uint32_t)q : (0x100u + lane);
      const uint32_t grp = __match_any_sync(FULL, key);
      const uint32_t before = __popc(grp & lanemask_lt());
      const uint32_t tail_q = __shfl_sync(FULL, rtail, q);
      // victims per restart FIFO (lane q owns FIFO q): reserve pool chunks
      uint32_t my_cnt = POL == SCHED_WAIT ? 0u : (lane == 0 ? ne : 0u);
      if (POL == SCHED_WAIT)
        for (int c = 0; c < nK(); ++c) {
          const uint32_t mm = __ballot_sync(FULL, ev && q == c);
          if (lane == c) my_cnt = __popc(mm);
        }
      const bool res_ok = my_cnt == 0 || fifo_reserve(lane, rtail, my_cnt);
      if (__any_sync(FULL, !res_ok)) { status = 2; return; }
      __syncwarp();
      if (ev) {
        const size_t e = fifo_wentry(q, tail_q + before);
        P.pool_a[e] = a;
        P.pool_e[e] = now;
        P.pool_llp[e] = l | (lp << 16) | ((meta & META_FT) ? 0x80000000u : 0u);
        if (POL == SCHED_WAIT) sh_add_u32(&cnt[meta & 0xFF], ~0u);
        if (POL == SCHED_NESTED) sh_add_u32(&cnt[nkey], ~0u);
      }
      __syncwarp();
      if (my_cnt) { rtail += my_cnt; fifo_tail_done(lane, rtail); }
      excess -= (int64_t)__reduce_add_sync(FULL, ev ? f : 0u);
      KV -= (int64_t)__reduce_add_sync(FULL, ev ? (l + s - 1) : 0u);
      n_plan_res -= __reduce_add_sync(FULL, ev ? inp : 0u);
      n_res -= ne;
      if (lane == 0) st->evictions += ne;
      n_evict += ne;
      __syncwarp();
    }
    // close the gap between the surviving residents and the staged admissions
    if (n_res != old_n && n_new > 0) {
      for (uint32_t o = 0; o < n_new; o += 32) {
        const uint32_t i = o + lane;
        Rec e = {0, 0};
        if (i < n_new) e = rr[old_n + i];
        __syncwarp();
        if (i < n_new) rr[n_res + i] = e;
        __syncwarp();
      }
    }
    if (excess > 0) drop_admissions(excess);
    peak = P.M + excess;
  }

  // no residents left and still over M: drop the latest new admissions
  // (they stay queued) and re-take the kept prefix in FIFO order
  __device__ void drop_admissions(int64_t& excess) {
    uint32_t keep = n_new;  // n_res == 0: staged admissions start at slot 0
    while (excess > 0 && keep > 0) { excess -= (int64_t)(rr[keep - 1].q & 0xFFFF); --keep; }
    restore_cursors();
    n_new = 0;
    sum_new_l = 0;
    if (POL == SCHED_WAIT) take_wait(keep);
    else take_fifo<false>(0, keep);  // FCFS never gets here (admission bound)
  }

  // S4 for the class-ring engine: LIFO eviction of up
  // to 32 victims per round.  The admission log (global, one class byte per
  // admission in admission order, truncated by evictions) gives the LIFO
  // order across classes: the log entries of class c are its completed
  // members (oldest) followed by its r_n residents, so the j-th newest
  // class-c entry is resident iff j < r_n, at ring position tail - 1 - j.
  // A round reads the 32 newest entries, loads the residents' records, and
  // an inclusive scan of freed KV finds the cut; everything newer than the
  // cut leaves the log.
  __device__ void memory_ring(uint32_t& n_evict, int64_t& peak) {
    peak = KV + (int64_t)n_plan_res + sum_new_l;
    if (peak <= P.M) return;
    int64_t excess = peak - P.M;
    const int K = nK();
    const uint8_t* log = P.ring_log + (size_t)wslot * kRingLog;
    while (excess > 0 && n_res > 0) {
      const uint32_t lo = seq_max > kRingLog ? seq_max - kRingLog : 0u;  // oldest entry still in the log
      if (seq_next <= lo) { status = 1; return; }                       // log window exhausted
      const uint32_t avail = min(seq_next - lo, 32u);
      const bool valid = (uint32_t)lane < avail;
      const uint32_t pos = seq_next - 1 - (uint32_t)lane;  // lane 0 = the newest admission
      const uint32_t v = valid ? (uint32_t)__ldcg(log + (pos & (kRingLog - 1))) : 0u;
      const uint32_t grp = __match_any_sync(FULL, valid ? v : 0x100u + (uint32_t)lane);
      const uint32_t j = __popc(grp & lanemask_lt());  // class-v entries newer than this one
      const uint32_t rn = __shfl_sync(FULL, r_n, (int)v), head = __shfl_sync(FULL, r_head, (int)v);
      const uint32_t Cv = __shfl_sync(FULL, r_C, (int)v), Rv = __shfl_sync(FULL, r_Ri, (int)v);
      const bool res = valid && j < rn;
      ulonglong2 rr2 = make_ulonglong2(0ull, (unsigned long long)Cv);
      if (res) rr2 = __ldcg(rg + P.roff[v] + wrap(head + (rn - 1 - j), P.rcap[v]));
      const uint64_t rec = rr2.x;
      const uint32_t x = (uint32_t)rr2.y;  // admission clock
      const uint32_t fl = P.fl[v], l = fl & 0xFFFFu, lp = fl >> 16;
      const int64_t e_a = (int64_t)(rec & 0x7FFFFFFFFFFFFFFFull);
      const bool ft0 = (rec >> 63) != 0;  // first token emitted before this admission
      const uint32_t s = Cv - x;  // next stage to run
      const uint32_t inp = res && (POL == SCHED_WAIT ? ((Qmask >> v) & 1u) : 1u);
      const uint32_t f = res ? (l + s - 1 + inp) : 0u;
      const uint32_t cum = warp_incl_scan_u32(f, lane);
      const uint32_t hit = __ballot_sync(FULL, res && (int64_t)cum >= excess);
      const uint32_t ntr = hit ? (uint32_t)__ffs(hit) : avail;  // log entries removed
      const bool ev = res && (uint32_t)lane < ntr;
      const uint32_t ne = __popc(__ballot_sync(FULL, ev));
      // a first token still pending (admitted at the last participation) was not emitted
      const bool pend = ev && !ft0 && x == Cv - 1;
      // restart records in eviction order (re-enter the queue)
      const int q = POL == SCHED_WAIT ? (int)v : 0;
      const uint32_t gq = __match_any_sync(FULL, ev ? (uint32_t)q : (0x100u + (uint32_t)lane));
      const uint32_t before = __popc(gq & lanemask_lt());
      const uint32_t tail_q = __shfl_sync(FULL, rtail, q);
      uint32_t my_cnt = POL == SCHED_WAIT ? 0u : (lane == 0 ? ne : 0u);
      if (POL == SCHED_WAIT)
        for (int c = 0; c < K; ++c) {
          const uint32_t mm = __ballot_sync(FULL, ev && q == c);
          if (lane == c) my_cnt = __popc(mm);
        }
      const bool res_ok = my_cnt == 0 || fifo_reserve(lane, rtail, my_cnt);
      if (__any_sync(FULL, !res_ok)) { status = 2; return; }
      cnt[lane] = 0;
      xs[lane] = 0;
      __syncwarp();
      if (ev) {
        const size_t ri = fifo_wentry(q, tail_q + before);
        P.pool_a[ri] = e_a;
        P.pool_e[ri] = now;
        // ring engine: lengths are the class's, so the record keeps the class
        P.pool_llp[ri] = v | (!pend ? 0x80000000u : 0u);
        sh_add_u32(&cnt[v], 1u);
        sh_add_u64(&xs[v], (uint64_t)x);
        acc_ev += (uint64_t)e_a;
        // the victim leaves its cohort (stage s = C - x in 1..l')
        sh_add_u32(&coh[P.ccoff[v] + (Rv >= s ? Rv - s : Rv + lp + 1 - s)], ~0u);
        if (pend) { sh_add_u32(&cnt[32 + v], ~0u); sh_add_u64(&psum()[v], (uint64_t)(-e_a)); }
      }
      __syncwarp();
      if (lane < K) {
        const uint32_t k = cnt[lane];
        r_n -= k;
        r_X -= xs[lane];
      }
      if (my_cnt) { rtail += my_cnt; fifo_tail_done(lane, rtail); }
      if (lane == 0) st->evictions += ne;
      excess -= (int64_t)__reduce_add_sync(FULL, ev ? f : 0u);
      KV -= (int64_t)__reduce_add_sync(FULL, ev ? (l + s - 1) : 0u);
      n_plan_res -= __reduce_add_sync(FULL, ev ? inp : 0u);
      n_res -= ne;
      n_evict += ne;
      seq_next -= ntr;
      __syncwarp();
    }
    if (excess > 0) drop_admissions(excess);
    peak = P.M + excess;
  }

  // ====================================== S4/S5, NESTED segment engine (SEG)
  // Every prompt passes the stages in admission order: an entry stage takes
  // its oldest n_k first (reading R6) and every non-entry
  // stage of an active segment advances (P14), so the resident array in
  // admission order is sorted by stage and segment k is a contiguous range
  // (DESIGN.md §5.2).  A non-entry member of segment k that ran the entry
  // stage b_k at clock x (C_k = batches segment k took part in) is at stage
  // b_k + C_k - x.  Members that complete inside the segment are counted in
  // a histogram keyed by their completion clock x + l' - b_k; members that
  // reach e_k alive are counted per cohort x and leave as one block (the
  // range boundary moves).  A batch therefore touches the records of the
  // entry-stage takes and of the admissions only; completed records stay
  // as tombstones until the array is compacted.
  __device__ __forceinline__ static uint32_t wrapc(uint32_t v, uint32_t n) { return v >= n ? v - n : v; }

  // segment of position p in [head, tail): k = #{j : P_j > p}; entry stage
  // iff k >= 1 and p >= E_k (every lane runs the shuffles)
  __device__ __forceinline__ int seg_of(uint32_t p, bool& entry) const {
    int k = 0;
    for (int j = 0; j < P.n_seg; ++j) k += bcast32(g_P, j) > p;
    const uint32_t Ek = __shfl_sync(FULL, g_E, k & 31);
    entry = k >= 1 && p >= Ek;
    return k;
  }
  // cohort-ring slot of clock x in segment k (Rc = C_k mod (W_k + 1), C_k - x <= W_k)
  __device__ __forceinline__ uint32_t coh_slot(uint32_t k, uint32_t Rc, uint32_t C, uint32_t x) const {
    const uint32_t d = C - x;
    return P.coff[k] + (Rc >= d ? Rc - d : Rc + P.seg_w[k] + 1u - d);
  }

  // S4, LIFO eviction from the array tail: up to 32
  // records per round, newest first; a record's freed KV is l + s - 1 (+1
  // if it is in the plan: non-entry stages of active segments, and the
  // oldest n_k alive at an active entry stage)
  __device__ void seg_memory(uint32_t& n_evict, int64_t& peak) {
    peak = KV + (int64_t)n_plan_res + sum_new_l;
    if (peak <= P.M) return;
    int64_t excess = peak - P.M;
    const uint32_t nen0 = g_nen;   // lane k: alive entry-stage residents at decision time
    uint32_t seen = 0;             // lane k: of which evicted so far
    while (excess > 0 && n_res > 0 && tail > head) {
      const uint32_t span = tail - head;
      const bool v = (uint32_t)lane < span;
      const uint32_t p = tail - 1 - (uint32_t)lane;  // lane 0 = the newest record
      SRec r = {0, 0};
      int64_t a = 0;
      if (v) { r = sa[p]; a = ga[p]; }
      bool en = false;
      int k = 0;
      // (the usual case: the whole chunk lies in segment 1's range)
      if (tail - min(span, 32u) < bcast32(g_P, 0)) k = seg_of(v ? p : tail - 1, en);
      const uint32_t kk = (uint32_t)k & 31u;
      const uint32_t l = r.llp & 0xFFFFu, lp = r.llp >> 16, x = r.xf & SX_X;
      const uint32_t Ck = __shfl_sync(FULL, g_C, kk), Rk = __shfl_sync(FULL, g_R, kk);
      const uint32_t Rck = __shfl_sync(FULL, g_Rc, kk);
      const uint32_t seen_k = __shfl_sync(FULL, seen, kk), nen_k = __shfl_sync(FULL, nen0, kk);
      const uint32_t bk = P.seg_b[kk], Wk = P.seg_w[kk];
      const uint32_t s = en ? bk : bk + Ck - x;  // next stage to run
      const bool alive = v && (en ? lp >= bk : s <= lp);
      const bool ea = alive && en;
      const uint32_t grp = __match_any_sync(FULL, ea ? kk : 0x100u + (uint32_t)lane);
      uint32_t inp = 0;
      if (alive && k <= kstar) {
        if (!en) inp = 1u;
        else inp = nen_k - 1u - (seen_k + __popc(grp & lanemask_lt())) < P.thr[kk];  // rank from the head
      }
      const uint32_t f = alive ? l + s - 1 + inp : 0u;
      const uint32_t cum = warp_incl_scan_u32(f, lane);
      const uint32_t hit = __ballot_sync(FULL, alive && (int64_t)cum >= excess);
      const uint32_t ntr = hit ? (uint32_t)__ffs(hit) : min(span, 32u);  // records removed from the tail
      const bool tr = (uint32_t)lane < ntr;
      const bool ev = tr && alive;
      const uint32_t evm = __ballot_sync(FULL, ev);
      const uint32_t ne = __popc(evm);
      const uint32_t before = __popc(evm & lanemask_lt());
      const uint32_t tail_q = __shfl_sync(FULL, rtail, 0);
      const uint32_t my_cnt = lane == 0 ? ne : 0u;
      const bool res_ok = my_cnt == 0 || fifo_reserve(lane, rtail, my_cnt);
      if (__any_sync(FULL, !res_ok)) { status = 2; return; }
      cnt[lane] = 0;
      cnt[32 + lane] = 0;
      xs[lane] = 0;
      __syncwarp();
      if (ev) {  // restart record, in eviction order (re-enter the queue)
        const size_t e = fifo_wentry(0, tail_q + before);
        const bool emitted = (r.xf & SX_FT) || s >= 2;
        P.pool_a[e] = a;
        P.pool_e[e] = now;
        P.pool_llp[e] = l | (lp << 16) | (emitted ? 0x80000000u : 0u);
        acc_ev += (uint64_t)a;
        if (en) {
          sh_add_u32(&cnt[32 + kk], 1u);
        } else {
          sh_add_u32(&cnt[kk], 1u);
          sh_add_u64(&xs[kk], (uint64_t)((int64_t)l - (int64_t)x));
        }
      }
      if (tr && !en) {  // the record leaves its cohort, and its pending completion or exit
        const uint32_t ci = coh_slot(kk, Rck, Ck, x);
        const bool exits = lp > bk + Wk;
        sh_add_u32(&con[ci], (ev && exits) ? ~0x10000u : ~0u);  // -(1 + (1 << 16)) / -1
        if (ev && exits) sh_add_u32(&col[ci], 0u - l);
        if (ev && !exits) {  // completion due at clock x + l' - b_k >= C_k
          const uint32_t i = P.hoff[kk] + wrapc(Rk + (x + lp - bk - Ck), Wk);
          sh_add_u32(&hcnt[i], ~0u);
          sh_add_u32(&hsll[i], 0u - (l + lp));
          sh_add_u32(&hslp[i], 0u - lp);
        }
      }
      // a first token due at the next batch (stage 1) is not emitted
      const bool pf = ev && !en && k == 0 && s == 1 && !(r.xf & SX_FT);
      pf_n -= __popc(__ballot_sync(FULL, pf));
      pf_a -= warp_sum_u64(pf ? (uint64_t)a : 0ull);
      __syncwarp();
      if (lane < P.n_seg) {
        g_nne -= cnt[lane];
        g_T -= (int64_t)xs[lane];
        g_nen -= cnt[32 + lane];
        seen += cnt[32 + lane];
      }
      if (my_cnt) { rtail += my_cnt; fifo_tail_done(lane, rtail); }
      if (lane == 0) st->evictions += ne;
      excess -= (int64_t)__reduce_add_sync(FULL, ev ? f : 0u);
      KV -= (int64_t)__reduce_add_sync(FULL, ev ? (l + s - 1) : 0u);
      n_plan_res -= __reduce_add_sync(FULL, ev ? inp : 0u);
      n_res -= ne;
      n_evict += ne;
      tail -= ntr;
      g_P = min(g_P, tail);
      g_E = min(g_E, tail);
      __syncwarp();
    }
    if (excess > 0) drop_admissions(excess);
    peak = P.M + excess;
  }

  // drop the tombstones of [head, tail) and move the rest to position 0
  // (when an admission would pass the capacity); cohort record counts and
  // range starts are recomputed
  __device__ void seg_compact() {
    const int L = P.n_seg;
    for (uint32_t i = lane; i < P.csize; i += 32) con[i] &= 0xFFFF0000u;
    __syncwarp();
    uint32_t wp = 0, nP = 0xFFFFFFFFu, nE = 0xFFFFFFFFu;
    for (uint32_t p0 = head; p0 < tail; p0 += 32) {
      const uint32_t p = p0 + (uint32_t)lane;
      const bool v = p < tail;
      SRec r = {0, 0};
      int64_t a = 0;
      if (v) { r = sa[p]; a = ga[p]; }
      bool en;
      const int k = seg_of(v ? p : p0, en);
      const uint32_t kk = (uint32_t)k & 31u;
      const uint32_t lp = r.llp >> 16, x = r.xf & SX_X;
      const uint32_t Ck = __shfl_sync(FULL, g_C, kk), Rck = __shfl_sync(FULL, g_Rc, kk);
      const uint32_t bk = P.seg_b[kk];
      const bool keep = v && (en ? lp >= bk : bk + Ck - x <= lp);
      const uint32_t km = __ballot_sync(FULL, keep);
      if (lane < L) {
        if (nP == 0xFFFFFFFFu && g_P < p0 + 32) nP = wp + __popc(km & ((1u << (g_P - p0)) - 1u));
        if (nE == 0xFFFFFFFFu && g_E < p0 + 32) nE = wp + __popc(km & ((1u << (g_E - p0)) - 1u));
      }
      if (keep) {
        const uint32_t d = wp + __popc(km & lanemask_lt());
        sa[d] = r;
        ga[d] = a;
        if (!en) sh_add_u32(&con[coh_slot(kk, Rck, Ck, x)], 1u);
      }
      wp += __popc(km);
    }
    if (lane < L) {
      g_P = nP == 0xFFFFFFFFu ? wp : nP;
      g_E = nE == 0xFFFFFFFFu ? wp : nE;
    }
    head = 0;
    tail = wp;
    __syncwarp();
  }

  // S5 for the segment engine
  __device__ void seg_execute(uint32_t n_evict, int64_t peak, uint32_t waiting) {
    const int L = P.n_seg;
    const bool act = lane < L && lane <= kstar;
    const uint32_t b = lane < L ? P.seg_b[lane] : 0u, W = lane < L ? P.seg_w[lane] : 0u;
    uint32_t nd = 0, kvf = 0, dtok = 0, tok = 0;
    if (act) {
      // non-entry members run stage b_k + C_k - x: sum (l + s) = T_k + n (b_k + C_k)
      tok = (uint32_t)(g_T + (int64_t)g_nne * (int64_t)(b + g_C));
      if (W > 0) {  // members whose stage l' runs now complete (A8)
        const uint32_t i = P.hoff[lane] + g_R;
        const uint32_t c = hcnt[i], sl = hsll[i];
        nd = c;
        kvf = sl - c;
        dtok = hslp[i];
        hcnt[i] = 0; hsll[i] = 0; hslp[i] = 0;
        g_T -= (int64_t)sl - (int64_t)c * (int64_t)(b + g_C);
        g_nne -= c;
      }
    }
    // entry stage of every active segment k >= 2: the oldest min{n_k, Q}
    // alive residents join cohort x = C_k
    for (uint32_t tm = __ballot_sync(FULL, act && lane >= 1 && g_nen > 0); tm; tm &= tm - 1) {
      const int k = __ffs(tm) - 1;
      const uint32_t need0 = min(bcast32(g_nen, k), P.thr[k]);
      const uint32_t C = bcast32(g_C, k), R = bcast32(g_R, k), Rc = bcast32(g_Rc, k);
      const uint32_t bk = P.seg_b[k], Wk = P.seg_w[k], ek = bk + Wk, ho = P.hoff[k];
      const uint32_t end = bcast32(g_P, k - 1);  // entry range [E_k, P_{k-1})
      uint32_t pos = bcast32(g_E, k), need = need0, nrec = 0;
      uint32_t my_nne = 0, my_nx = 0, my_slx = 0;
      int64_t my_dT = 0;
      while (need > 0 && pos < end) {
        const uint32_t p = pos + (uint32_t)lane;
        const bool v = p < end;
        SRec r = {0, 0};
        if (v) r = sa[p];
        const uint32_t l = r.llp & 0xFFFFu, lp = r.llp >> 16;
        const bool alive = v && lp >= bk;
        const uint32_t am = __ballot_sync(FULL, alive);
        const uint32_t rk = __popc(am & lanemask_lt());
        const bool tk = alive && rk < need;
        const uint32_t last = __ballot_sync(FULL, alive && rk == need - 1);
        const uint32_t ext = last ? (uint32_t)__ffs(last) : min(32u, end - pos);
        if ((uint32_t)lane < ext) sa[p].xf = (r.xf & SX_FT) | C;
        if (tk) {
          tok += l + bk;
          if (lp == bk) {  // completes at the entry stage
            ++nd;
            kvf += l + lp - 1;
            dtok += lp;
          } else {
            ++my_nne;
            my_dT += (int64_t)l - (int64_t)C;
            if (lp <= ek) {
              const uint32_t i = ho + wrapc(R + (lp - bk), Wk);
              sh_add_u32(&hcnt[i], 1u);
              sh_add_u32(&hsll[i], l + lp);
              sh_add_u32(&hslp[i], lp);
            } else {
              ++my_nx;
              my_slx += l;
            }
          }
        }
        nrec += ext;
        pos += ext;
        need -= min((uint32_t)__popc(am), need);
      }
      const uint32_t s_nne = __reduce_add_sync(FULL, my_nne), s_nx = __reduce_add_sync(FULL, my_nx);
      const uint32_t s_slx = __reduce_add_sync(FULL, my_slx);
      const int64_t s_dT = warp_sum_i64(my_dT);
      __syncwarp();
      if (lane == k) { g_E = pos; g_nen -= need0 - need; g_nne += s_nne; g_T += s_dT; }
      if (lane == 0) {
        const uint32_t ci = P.coff[k] + Rc;
        con[ci] += nrec | (s_nx << 16);
        col[ci] += s_slx;
      }
      __syncwarp();
    }
    // a batch ending after T is the last one; its completions are not
    // counted (A19): their arrival ticks leave the completion sum here
    {
      const int64_t tokens = (int64_t)__reduce_add_sync(FULL, tok) + sum_new_l;
      const int64_t tau = P.d0_t + P.d1_t * max(tokens - P.b0, (int64_t)0);
      if (now + tau > P.T_t) seg_late_sum();
    }
    // cohort x = C_k - W_k ran stage e_k: its alive members move to the
    // entry stage of segment k+1 (the range start moves past the cohort)
    uint32_t ex_alive = 0;
    if (act) {
      const uint32_t ci = P.coff[lane] + (g_Rc == W ? 0u : g_Rc + 1);
      const uint32_t cn = con[ci], sl = col[ci];
      con[ci] = 0;
      col[ci] = 0;
      const uint32_t nx = cn >> 16;
      g_P += cn & 0xFFFFu;
      g_nne -= nx;
      g_T -= (int64_t)sl - (int64_t)nx * (int64_t)(g_C - W);
      ex_alive = nx;
    }
    {
      const uint32_t from = __shfl_up_sync(FULL, ex_alive, 1);
      if (lane >= 1 && lane < L) g_nen += from;
    }
    head = bcast32(g_P, L - 1);
    // first tokens of the prompts admitted at the previous batch (stage 1)
    const uint32_t nf = pf_n;
    const uint64_t fta = pf_a;
    pf_n = 0;
    pf_a = 0;
    // admissions (their stage-0 iteration is this batch) join cohort x = C_1 at the tail
    if (n_new > 0) {
      if (tail + n_new > P.seg_cap) {
        seg_compact();
        // a nearly full array would compact at every batch: overflow instead
        // (status 1: the replication re-runs on the member engine)
        if (tail + n_new + (P.seg_cap >> 3) > P.seg_cap) { status = 1; return; }
      }
      const uint32_t C0 = bcast32(g_C, 0), R0 = bcast32(g_R, 0), Rc0 = bcast32(g_Rc, 0), W0 = P.seg_w[0];
      uint32_t my_nx = 0, my_slx = 0, my_pf = 0, my_l = 0;
      uint64_t my_pfa = 0;
      for (uint32_t j0 = 0; j0 < n_new; j0 += 32) {
        const uint32_t j = j0 + (uint32_t)lane;
        if (j < n_new) {
          const Rec e = rr[j];
          const uint32_t l = (uint32_t)(e.q & 0xFFFF), lp = (uint32_t)((e.q >> 16) & 0xFFFF);
          const bool ft = ((uint32_t)(e.q >> 48) & META_FT) != 0;
          sa[tail + j] = SRec{l | (lp << 16), C0 | (ft ? SX_FT : 0u)};
          ga[tail + j] = e.a;
          acc_adm += (uint64_t)e.a;
          my_l += l;
          if (!ft) { ++my_pf; my_pfa += (uint64_t)e.a; }
          if (lp <= W0) {
            const uint32_t i = P.hoff[0] + wrapc(R0 + lp, W0);
            sh_add_u32(&hcnt[i], 1u);
            sh_add_u32(&hsll[i], l + lp);
            sh_add_u32(&hslp[i], lp);
          } else {
            ++my_nx;
            my_slx += l;
          }
        }
      }
      pf_n = __reduce_add_sync(FULL, my_pf);
      pf_a = warp_sum_u64(my_pfa);
      const uint32_t s_nx = __reduce_add_sync(FULL, my_nx), s_slx = __reduce_add_sync(FULL, my_slx);
      const uint32_t s_l = __reduce_add_sync(FULL, my_l);
      __syncwarp();
      if (lane == 0) {
        const uint32_t ci = P.coff[0] + Rc0;
        con[ci] += n_new | (s_nx << 16);
        col[ci] += s_slx;
        g_nne += n_new;
        g_T += (int64_t)s_l - (int64_t)n_new * (int64_t)C0;
      }
      tail += n_new;
      __syncwarp();
    }
    if (act) {
      ++g_C;
      if (W > 0) g_R = g_R + 1 == W ? 0u : g_R + 1;
      g_Rc = g_Rc == W ? 0u : g_Rc + 1;
    }
    const uint32_t tok_o = __reduce_add_sync(FULL, tok), nd_o = __reduce_add_sync(FULL, nd);
    const uint32_t kvf_o = __reduce_add_sync(FULL, kvf), dtok_o = __reduce_add_sync(FULL, dtok);
    const uint32_t gr = n_plan_res - nd_o;
    n_res = n_res - nd_o + n_new;
    epilogue(n_evict, peak, waiting, tok_o, nd_o, nf, dtok_o, kvf_o, gr, 0ull, lane == 0 ? fta : 0ull);
  }

  // arrival-tick sum of the members completing in this batch (after the
  // entry-stage takes): non-entry records of active segments whose
  // completion clock x + l' - b_k is C_k; added to the evicted sum, which
  // is subtracted from the admitted one at the end
  __device__ void seg_late_sum() {
    u128 al = 0;
    for (uint32_t p0 = head; p0 < tail; p0 += 32) {
      const uint32_t p = p0 + (uint32_t)lane;
      const bool v = p < tail;
      SRec r = {0, 0};
      if (v) r = sa[p];
      bool en;
      const int k = seg_of(v ? p : p0, en);
      const uint32_t kk = (uint32_t)k & 31u;
      const uint32_t lp = r.llp >> 16, x = r.xf & SX_X;
      const uint32_t Ck = __shfl_sync(FULL, g_C, kk);
      if (v && !en && k <= kstar && x + lp - P.seg_b[kk] == Ck) al += (uint64_t)ga[p];
    }
    al = warp_sum_u128(al);
    if (lane == 0) st->acc_ev += al;
    __syncwarp();
  }

  // end of a replication: arrival-tick sum of the residents still alive, so
  // that sum over completions by T of a = admitted - evicted - late - alive
  __device__ void seg_finish() {
    u128 ares = 0;
    for (uint32_t p0 = head; p0 < tail; p0 += 32) {
      const uint32_t p = p0 + (uint32_t)lane;
      const bool v = p < tail;
      SRec r = {0, 0};
      int64_t a = 0;
      if (v) { r = sa[p]; a = ga[p]; }
      bool en;
      const int k = seg_of(v ? p : p0, en);
      const uint32_t kk = (uint32_t)k & 31u;
      const uint32_t lp = r.llp >> 16, x = r.xf & SX_X;
      const uint32_t Ck = __shfl_sync(FULL, g_C, kk);
      const uint32_t bk = P.seg_b[kk];
      const bool alive = en ? lp >= bk : bk + Ck - x <= lp;
      if (v && alive) ares += (uint64_t)a;
    }
    ares = warp_sum_u128(ares);
    if (lane == 0) st->acc_done_a = st->acc_adm - st->acc_ev - ares;
    __syncwarp();
  }

  // per-lane batch accumulators of the execute pass
  struct Acc {
    uint32_t tok = 0, n_done = 0, done_tok = 0, n_ft = 0, kv_free = 0, grow = 0;
    uint64_t done_a = 0, ft_a = 0;
  };
  struct Upd {
    bool keep, inp;
    uint32_t l, lp, ns, meta;
    uint32_t seg;  // NESTED: segment after the step (chunk activity summary)
  };

  // S5 per-member step: membership, first token, completion or s++
  __device__ __forceinline__ Upd member(bool valid, bool fresh, int64_t a, uint64_t qv,
                                        uint32_t over, Acc& acc) {
    Upd u;
    u.l = (uint32_t)(qv & 0xFFFF);
    u.lp = (uint32_t)((qv >> 16) & 0xFFFF);
    const uint32_t s = (uint32_t)((qv >> 32) & 0xFFFF);
    u.meta = (uint32_t)(qv >> 48);
    bool inp = false;
    uint32_t key_s = 0, info_s = 0;
    if (POL == SCHED_NESTED) {
      info_s = (valid && !fresh) ? __ldg(P.stage_info + s) : 0x3Fu;
      const int seg = info_seg(info_s);
      key_s = info_key(info_s);
      const bool act = valid && !fresh && seg <= kstar;
      // entry-stage residents need a rank only in segments whose entry
      // queue holds more than n_k (first n_k in admission order batch)
      const bool ranked = act && (info_s >> 7) && ((over >> seg) & 1u);
      inp = act;
      if (__any_sync(FULL, ranked)) {
        const uint32_t key = ranked ? s : (0x10000u + lane);
        const uint32_t grp = __match_any_sync(FULL, key);
        if (ranked) inp = rank[seg] + __popc(grp & lanemask_lt()) < P.thr[seg];
        __syncwarp();
        if (ranked && (grp & lanemask_lt()) == 0) rank[seg] += __popc(grp);
        __syncwarp();
      }
    } else if (POL == SCHED_WAIT) {
      inp = valid && !fresh && ((Qmask >> (u.meta & 0xFF)) & 1u);
    } else {
      inp = valid && !fresh;
    }
    u.keep = valid;
    u.inp = inp;
    u.ns = s;
    if (POL == SCHED_NESTED) u.seg = fresh ? 0u : info_seg(info_s);
    if (inp) {
      acc.tok += u.l + s;
      // the stage-1 iteration emits the first output token
      if (s == 1 && !(u.meta & META_FT)) { u.meta |= META_FT; ++acc.n_ft; acc.ft_a += (uint64_t)a; }
      if (s == u.lp) {
        // stage l' done: complete, free KV
        u.keep = false;
        acc.kv_free += u.l + u.lp - 1;
        ++acc.n_done;
        acc.done_tok += u.lp;
        acc.done_a += (uint64_t)a;
        if (POL == SCHED_WAIT) sh_add_u32(&cnt[u.meta & 0xFF], ~0u);
        if (POL == SCHED_NESTED) sh_add_u32(&cnt[key_s], ~0u);
      } else {
        u.ns = s + 1;
        ++acc.grow;
        if (POL == SCHED_NESTED && (info_s & 0xC0)) {
          // leaving an entry stage (-> non-entry) or a segment's last stage
          // (-> the next segment's entry stage)
          const uint32_t seg = info_seg(info_s);
          const uint32_t key_n = (info_s & 0x40) ? 32u + seg + 1u : seg;
          if (info_s & 0x40) u.seg = seg + 1;
          sh_add_u32(&cnt[key_s], ~0u);
          sh_add_u32(&cnt[key_n], 1u);
        }
      }
    }
    return u;
  }

  // in-place stream compaction of one chunk (ballot + popc keeps order).
  // No __syncwarp around the stores: every lane's load of this chunk feeds
  // the ballot before any store, stores go to d <= i (slots this or earlier
  // chunks already read), and the next chunk reads beyond them.
  __device__ __forceinline__ void compact(const Upd& u, int64_t a, uint32_t& wp) {
    const uint32_t km = __ballot_sync(FULL, u.keep);
    const uint32_t d = wp + __popc(km & lanemask_lt());
    if (u.keep) rr[d] = Rec{a, pack_q(u.l, u.lp, u.ns, u.meta)};
    wp += __popc(km);
  }

  // Nested compaction + chunk activity summaries: csum[x] = the lowest
  // segment of the residents in chunk x (slots 32x..32x+31); a chunk whose
  // residents all sit in segments > k* takes no part in the batch and, while
  // nothing before it moved, is skipped
  __device__ __forceinline__ void compact_n(const Upd& u, int64_t a, uint32_t& wp) {
    const uint32_t km = __ballot_sync(FULL, u.keep);
    const uint32_t d = wp + __popc(km & lanemask_lt());
    if (u.keep) rr[d] = Rec{a, pack_q(u.l, u.lp, u.ns, u.meta)};
    const uint32_t c0 = wp >> 5, kept = __popc(km);
    const uint32_t m0 = __reduce_min_sync(FULL, (u.keep && (d >> 5) == c0) ? u.seg : 0xFFu);
    const uint32_t m1 = __reduce_min_sync(FULL, (u.keep && (d >> 5) != c0) ? u.seg : 0xFFu);
    if (lane == 0 && kept) {
      csum[c0] = (wp & 31u) ? (uint8_t)min((uint32_t)csum[c0], m0) : (uint8_t)m0;
      if (((wp + kept - 1) >> 5) != c0) csum[c0 + 1] = (uint8_t)m1;
    }
    wp += kept;
  }

  // WAIT / FCFS per-member step + compaction, branch-light: membership,
  // first token (stage 1), completion after stage l'
  // (frees l+l'-1) or s++
  __device__ __forceinline__ void step_plain(uint32_t i, bool v, const Rec& e, Acc& acc, uint32_t& wp) {
    const uint64_t q = e.q;
    const uint32_t l = (uint32_t)(q & 0xFFFF), lp = (uint32_t)((q >> 16) & 0xFFFF);
    const uint32_t s = (uint32_t)((q >> 32) & 0xFFFF), meta = (uint32_t)(q >> 48);
    bool inp = v && i < n_res;  // staged admissions (i >= n_res) just keep stage 1
    if (POL == SCHED_WAIT) inp = inp && ((Qmask >> (meta & 0xFF)) & 1u);
    const bool ft = inp && s == 1 && !(meta & META_FT);
    const bool done = inp && s == lp;
    acc.tok += inp ? l + s : 0u;
    acc.n_ft += ft;
    acc.ft_a += ft ? (uint64_t)e.a : 0ull;
    acc.n_done += done;
    acc.done_tok += done ? lp : 0u;
    acc.kv_free += done ? l + lp - 1 : 0u;
    acc.done_a += done ? (uint64_t)e.a : 0ull;
    acc.grow += inp && !done;
    if (POL == SCHED_WAIT && done) sh_add_u32(&cnt[meta & 0xFF], ~0u);
    const uint64_t nq = q + ((inp && !done) ? (1ull << 32) : 0ull) + (ft ? ((uint64_t)META_FT << 48) : 0ull);
    const bool keep = v && !done;
    const uint32_t km = __ballot_sync(FULL, keep);
    const uint32_t d = wp + __popc(km & lanemask_lt());
    if (keep) rr[d] = Rec{e.a, nq};
    wp += __popc(km);
  }

  // ------------------------------------------------------ S5 execute
  // One pass over residents (+ the staged admissions) in admission order:
  // per-member update, completions, compaction; counters updated in place.
  __device__ void execute(uint32_t n_evict, int64_t peak, uint32_t waiting) {
    if (SEG) { seg_execute(n_evict, peak, waiting); return; }
    uint32_t tok, nd, nf, dtok, kvf, gr;
    uint64_t done_a = 0, ft_a = 0;
    if (RING) {
      ring_pass(tok, nd, nf, dtok, kvf, ft_a);
      gr = n_plan_res - nd;
      if (!ring_append()) return;
      if (lane < nK() && (POL == SCHED_WAIT ? ((Qmask >> lane) & 1u) : 1u)) {
        ++r_C;
        r_Ri = r_Ri == (P.fl[lane] >> 16) ? 0u : r_Ri + 1;
      }
      n_res = n_res - nd + n_new;
    } else {
      member_pass(tok, nd, nf, dtok, kvf, gr, done_a, ft_a);
    }
    epilogue(n_evict, peak, waiting, tok, nd, nf, dtok, kvf, gr, done_a, ft_a);
  }

  // S5 for the class-ring engine: the stage of a member admitted at class
  // clock x is C_c - x, so the stage-l' completions
  // are the cohort admitted at x = C_c - l' (a count per clock slot) and
  // the stage-1 first tokens the prompts admitted at the
  // class's previous participation without one (counted at append); plan
  // tokens sum_(l + s) = n_c (l_c + C_c) - sum x.  O(K) per batch: no
  // member record is read (the arrival ticks of completions enter the
  // latency sum through admitted - evicted - late - still resident).
  __device__ void ring_pass(uint32_t& tok, uint32_t& nd, uint32_t& nf, uint32_t& dtok, uint32_t& kvf,
                            uint64_t& ft_a) {
    const bool cin = lane < nK() && (POL == SCHED_WAIT ? ((Qmask >> lane) & 1u) : 1u);
    const uint32_t fl = lane < nK() ? P.fl[lane] : 0u, l = fl & 0xFFFFu, lp = fl >> 16;
    const uint32_t tk = cin ? (uint32_t)((uint64_t)r_n * (l + r_C) - r_X) : 0u;
    tok = __reduce_add_sync(FULL, tk);
    uint32_t my_nd = 0, my_nf = 0;
    if (cin) {  // stage-1 members emit their first token
      my_nf = cnt[32 + lane];
      ft_a += psum()[lane];
      cnt[32 + lane] = 0;
      psum()[lane] = 0;
      // the cohort x = C - l' runs its last stage (slot (C + 1) mod (l' + 1))
      const uint32_t i = P.ccoff[lane] + (r_Ri == lp ? 0u : r_Ri + 1);
      my_nd = coh[i];
      coh[i] = 0;
    }
    // a batch ending after T is the last one; its completions are not
    // counted (A19): their arrival ticks leave the completion sum here
    {
      const int64_t tokens = (int64_t)tok + sum_new_l;
      const int64_t tau = P.d0_t + P.d1_t * max(tokens - P.b0, (int64_t)0);
      if (now + tau > P.T_t) {
        u128 al = 0;
        for (uint32_t cm = __ballot_sync(FULL, my_nd > 0); cm; cm &= cm - 1) {
          const int c = __ffs(cm) - 1;
          const uint32_t n = bcast32(my_nd, c), head = bcast32(r_head, c), cap = P.rcap[c];
          for (uint32_t j = lane; j < n; j += 32) al += __ldcg(&rg[P.roff[c] + wrap(head + j, cap)].x) & 0x7FFFFFFFFFFFFFFFull;
        }
        al = warp_sum_u128(al);
        if (lane == 0) st->acc_ev += al;
      }
    }
    if (cin) {
      r_head = wrap(r_head + my_nd, P.rcap[lane]);
      r_n -= my_nd;
      r_X -= (uint64_t)my_nd * (r_C - lp);
    }
    nd = __reduce_add_sync(FULL, my_nd);
    nf = __reduce_add_sync(FULL, my_nf);
    dtok = __reduce_add_sync(FULL, my_nd * lp);
    kvf = __reduce_add_sync(FULL, my_nd * (l + lp - 1));
    __syncwarp();
  }

  // append the staged admissions (stage 1 next, admission clock = C_c) to
  // their class rings (global memory), in admission order; cohort counts of
  // the current clocks; false on ring overflow (status 1)
  __device__ bool ring_append() {
    uint32_t my_new = 0;
    for (uint32_t j0 = 0; j0 < n_new; j0 += 32) {
      const uint32_t j = j0 + (uint32_t)lane;
      const bool v = j < n_new;
      Rec e = {0, 0};
      if (v) e = rr[j];
      const uint32_t meta = (uint32_t)(e.q >> 48), c = v ? (meta & 0xFFu) : 0u;
      // lanes of the same class (rank within it) and, in lane c, class c's
      // count of this chunk: one ballot per class when K is a constant
      uint32_t grp = 0, add = 0;
      if (KC > 0) {
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) {
          const uint32_t b = __ballot_sync(FULL, v && c == (uint32_t)cc);
          if (c == (uint32_t)cc) grp = b;
          if (lane == cc) add = __popc(b);
        }
      } else {
        grp = __match_any_sync(FULL, v ? c : 0x100u + (uint32_t)lane);
      }
      const uint32_t rk = __popc(grp & lanemask_lt());
      const uint32_t n = __shfl_sync(FULL, r_n, (int)c) + __shfl_sync(FULL, my_new, (int)c);
      const uint32_t head = __shfl_sync(FULL, r_head, (int)c);
      const uint32_t C = __shfl_sync(FULL, r_C, (int)c), cap = P.rcap[c];
      if (__any_sync(FULL, v && n + rk >= cap)) { status = 1; return false; }
      if (KC == 0) {
        cnt[lane] = 0;
        __syncwarp();
      }
      // a prompt without its first token emits it at the next participation
      const bool pend = v && !(meta & META_FT);
      if (v) {
        rg[P.roff[c] + wrap(head + n + rk, cap)] =
            make_ulonglong2((uint64_t)e.a | (pend ? 0ull : 1ull << 63), (unsigned long long)C);
        P.ring_log[(size_t)wslot * kRingLog + ((seq_next + j) & (kRingLog - 1))] = (uint8_t)c;
        acc_adm += (uint64_t)e.a;
        if (KC == 0 && rk == 0) cnt[c] = __popc(grp);
      }
      // per-class pending first tokens (shared: pcnt = cnt[32..], psum)
      if (KC == WAITSIM_PEND_REDUCE_K) {
        // per class: count by ballot, arrival-tick sum by three 32-bit warp
        // reductions of 24-bit pieces (ticks < 2^57: every piece sum is exact)
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) {
          const bool mine = pend && c == (uint32_t)cc;
          const uint32_t b = __ballot_sync(FULL, mine);
          if (b) {
            const uint64_t av = mine ? (uint64_t)e.a : 0ull;
            const uint32_t s0 = __reduce_add_sync(FULL, (uint32_t)(av & 0xFFFFFFu));
            const uint32_t s1 = __reduce_add_sync(FULL, (uint32_t)((av >> 24) & 0xFFFFFFu));
            const uint32_t s2 = __reduce_add_sync(FULL, (uint32_t)(av >> 48));
            if (lane == cc) {
              cnt[32 + cc] += __popc(b);
              psum()[cc] += (uint64_t)s0 + ((uint64_t)s1 << 24) + ((uint64_t)s2 << 48);
            }
          }
        }
      } else if (pend) {
        sh_add_u32(&cnt[32 + c], 1u);
        sh_add_u64(&psum()[c], (uint64_t)e.a);
      }
      if (KC > 0) {
        my_new += add;
      } else {
        __syncwarp();
        if (lane < nK()) my_new += cnt[lane];
        __syncwarp();
      }
    }
    __syncwarp();
    if (lane < nK()) {
      r_n += my_new;
      r_X += (uint64_t)my_new * r_C;
      coh[P.ccoff[lane] + r_Ri] += my_new;
    }
    seq_next += n_new;
    seq_max = max(seq_max, seq_next);
    return true;
  }

  // end of a replication (RING): arrival-tick sum of the residents still in
  // the class rings, so that the completion sum is admitted - evicted -
  // late - resident
  __device__ void ring_finish() {
    u128 ar = 0;
    for (int c = 0; c < nK(); ++c) {
      const uint32_t n = bcast32(r_n, c), head = bcast32(r_head, c), cap = P.rcap[c];
      for (uint32_t j = lane; j < n; j += 32) ar += __ldcg(&rg[P.roff[c] + wrap(head + j, cap)].x) & 0x7FFFFFFFFFFFFFFFull;
    }
    ar = warp_sum_u128(ar);
    if (lane == 0) st->acc_done_a = st->acc_adm - st->acc_ev - ar;
    __syncwarp();
  }

  // S5 for the member engine: one pass over residents (+ the staged
  // admissions) in admission order, per-member update and compaction
  __device__ void member_pass(uint32_t& tok_o, uint32_t& nd_o, uint32_t& nf_o, uint32_t& dtok_o,
                              uint32_t& kvf_o, uint32_t& gr_o, uint64_t& done_a_o, uint64_t& ft_a_o) {
    const uint32_t n_tot = n_res + n_new;
    uint32_t over = 0;  // NESTED: active segments whose entry queue exceeds n_k
    if (POL == SCHED_NESTED) {
      over = __ballot_sync(FULL, lane >= 1 && lane <= kstar && cnt[32 + lane] > P.thr[lane]);
      rank[lane] = 0;
      __syncwarp();
    }
    Acc acc;
    uint32_t wp = 0;
    if (POL != SCHED_NESTED) {
      // two chunks per iteration for ILP (chunk 0's stores land below chunk
      // 1's slots, which were loaded first)
      for (uint32_t base = 0; base < n_tot; base += 64) {
        const uint32_t i0 = base + lane, i1 = i0 + 32;
        const bool v0 = i0 < n_tot, v1 = i1 < n_tot;
        Rec e0 = {0, 0}, e1 = {0, 0};
        if (v0) e0 = rr[i0];
        if (v1) e1 = rr[i1];
        step_plain(i0, v0, e0, acc, wp);
        if (base + 32 < n_tot) step_plain(i1, v1, e1, acc, wp);
      }
    } else {
      // most residents idle (waiting at entry stages of inactive segments,
      // e.g. the thrashing C5 regime): keep chunk summaries and skip idle
      // chunks; otherwise plain passes, which mark what they wrote as active
      if (n_plan_res * 4 < n_res) {
        for (uint32_t base = 0; base < n_tot; base += 64) {
          // idle chunk pairs with nothing moved before them: skip them all at
          // once (lane i tests the pair at base + 64 i; the first non-idle
          // pair ends the run) instead of one pair per iteration
          if (wp == base) {
            for (;;) {
              const uint32_t b = base + 64u * (uint32_t)lane;
              const bool idle = b + 64 <= n_res && csum[b >> 5] > (uint32_t)kstar &&
                                csum[(b >> 5) + 1] > (uint32_t)kstar;
              const uint32_t busy = __ballot_sync(FULL, !idle);
              if (busy) { base += 64u * (uint32_t)(__ffs(busy) - 1); break; }
              base += 64u * 32u;
            }
            wp = base;
            if (base >= n_tot) break;
          }
          const uint32_t i0 = base + lane, i1 = i0 + 32;
          const bool v0 = i0 < n_tot, v1 = i1 < n_tot;
          Rec e0 = {0, 0}, e1 = {0, 0};
          if (v0) e0 = rr[i0];
          if (v1) e1 = rr[i1];
          const Upd u0 = member(v0, i0 >= n_res, e0.a, e0.q, over, acc);
          const Upd u1 = member(v1, i1 >= n_res, e1.a, e1.q, over, acc);
          compact_n(u0, e0.a, wp);
          compact_n(u1, e1.a, wp);
        }
      } else {
        for (uint32_t base = 0; base < n_tot; base += 64) {
          const uint32_t i0 = base + lane, i1 = i0 + 32;
          const bool v0 = i0 < n_tot, v1 = i1 < n_tot;
          Rec e0 = {0, 0}, e1 = {0, 0};
          if (v0) e0 = rr[i0];
          if (v1) e1 = rr[i1];
          const Upd u0 = member(v0, i0 >= n_res, e0.a, e0.q, over, acc);
          const Upd u1 = member(v1, i1 >= n_res, e1.a, e1.q, over, acc);
          compact(u0, e0.a, wp);
          compact(u1, e1.a, wp);
        }
        __syncwarp();
        for (uint32_t x = lane; x < (wp + 31) / 32; x += 32) csum[x] = 0;  // unknown: active
      }
    }
    __syncwarp();
    if (POL == SCHED_WAIT) { if (lane < nK()) cnt[lane] += newc; }
    if (POL == SCHED_NESTED) { if (lane == 0) cnt[0] += n_new; }  // stage 1 = segment 1, non-entry
    // warp-uniform batch totals
    tok_o = __reduce_add_sync(FULL, acc.tok);
    nd_o = __reduce_add_sync(FULL, acc.n_done);
    nf_o = __reduce_add_sync(FULL, acc.n_ft);
    dtok_o = __reduce_add_sync(FULL, acc.done_tok);
    kvf_o = __reduce_add_sync(FULL, acc.kv_free);
    gr_o = __reduce_add_sync(FULL, acc.grow);
    done_a_o = acc.done_a;
    ft_a_o = acc.ft_a;
    n_res = wp;
  }

  // batch epilogue: tau, clock, KV, metric accumulators, trajectory hash
  __device__ void epilogue(uint32_t n_evict, int64_t peak, uint32_t waiting, uint32_t tok, uint32_t nd,
                           uint32_t nf, uint32_t dtok, uint32_t kvf, uint32_t gr, uint64_t done_a,
                           uint64_t ft_a) {
    const int64_t tokens = (int64_t)tok + sum_new_l;
    // tau = d0 + d1 * (sum prefill l + sum decode (l+s)),
    // piecewise linear beyond b0 tokens (R31; b0 = 0: linear)
    const int64_t tau = P.d0_t + P.d1_t * max(tokens - P.b0, (int64_t)0);
    const int64_t t_end = now + tau;
    const bool by_T = t_end <= P.T_t;
    if (by_T) { acc_done_a += done_a; acc_ft_a += ft_a; }
    KV += (int64_t)gr - (int64_t)kvf + sum_new_l;
    const uint32_t plan_size = n_plan_res + n_new;
    if (lane == 0) {
      if (by_T) {
        // latency / TTFT sums = sum(t_end) - sum(a)
        st->sum_done_t += (u128)nd * (uint64_t)t_end;
        st->sum_ft_t += (u128)nf * (uint64_t)t_end;
        st->completed += nd;
        st->completed_tokens += dtok;
        st->first_tokens += nf;
        st->cbi += (uint64_t)nd * st->batches;
      } else {
        st->completed_after_T += nd;
      }
      if (TRACE && rep == 0 && st->log_n < P.log_cap) {
        int64_t* e = P.log + 7 * st->log_n;
        e[0] = now; e[1] = plan_size; e[2] = tokens; e[3] = nd; e[4] = n_evict; e[5] = n_new; e[6] = peak;
      }
      if (TRACE && rep == 0) ++st->log_n;
      uint64_t hh = st->h;
      hh = mix64(hh ^ (uint64_t)now);
      hh = mix64(hh ^ ((uint64_t)plan_size | ((uint64_t)tokens << 32)));
      hh = mix64(hh ^ ((uint64_t)nd | ((uint64_t)n_evict << 20) | ((uint64_t)n_new << 40)));
      st->h = hh;
      st->request_steps += plan_size;
      st->prefill_steps += n_new;
      st->admitted += n_new;
      st->busy += tau;
      if (peak > st->max_kv) st->max_kv = peak;
      st->sum_waiting += waiting;
      ++st->batches;
    }
    maybe_flush();
    n_new = 0;
    now = t_end;
    __syncwarp();
  }

  // ------------------------------------------------------------ run
  __device__ void run(uint32_t rep_) {
    rep = rep_;
    rglob = (uint32_t)(P.rep_begin + rep_);
    const uint64_t seed = TRACE ? 0ull : P.seed;
    now = 0; KV = 0; n_res = 0; n_new = 0; status = 0; sum_new_l = 0;
    acc_arr = acc_done_a = acc_ft_a = 0;
    __syncwarp();
    if (lane == 0) {
      WarpStats z = {};
      z.h = mix64(seed ^ ((uint64_t)(TRACE ? rep_ : rglob) * 0x9E3779B97F4A7C15ull));
      *st = z;
    }
    __syncwarp();
    k_vis = vbase = k_adm = abase = pcount = rhead = rtail = 0;
    if (lane < P.n_rings) rq[20 * lane] = rq[20 * lane + 2] = kNoChunk;
    vprev = aprev = 0;
    newc = 0;
    r_head = r_n = r_C = seq_next = 0;
    r_Ri = 0;
    seq_max = 0;
    r_X = 0;
    if (RING) {
      psum()[lane] = 0;
      acc_adm = acc_ev = 0;
      for (uint32_t i = lane; i < P.ccsize; i += 32) coh[i] = 0;
    }
    if (SEG) {
      head = tail = 0;
      pf_n = 0; pf_a = 0;
      acc_adm = acc_ev = 0;
      g_P = g_E = g_C = g_R = g_Rc = g_nne = g_nen = 0;
      g_T = 0;
      for (uint32_t i = lane; i < P.hsize; i += 32) { hcnt[i] = 0; hsll[i] = 0; hslp[i] = 0; }
      for (uint32_t i = lane; i < P.csize; i += 32) { con[i] = 0; col[i] = 0; }
    }
    for (int c = 0; c < nK(); ++c) {
      fill<true>(c, 0, 0, vt, vl, vlp);
    }
    cnt[lane] = 0;
    cnt[32 + lane] = 0;
    __syncwarp();
    for (;;) {
      ingest();
      if (now >= P.T_t) break;                     // STOP
      const uint32_t waiting = waiting_total();
      bool go = decide();
      if (status) break;
      uint32_t n_evict = 0;
      int64_t peak = 0;
      if (go) {
        if (RING) memory_ring(n_evict, peak);
        else if (SEG) seg_memory(n_evict, peak);
        else memory(n_evict, peak);
        if (status) break;
        if (n_plan_res + n_new == 0) go = false;    // empty after eviction: wait (R27)
      }
      if (!go) {
        int64_t nt = (POL == SCHED_WAIT || POL == SCHED_NESTED) && below ? idle_jump() : TMAX;
        if (nt >= P.T_t) nt = next_arrival();  // near the horizon: step arrival by arrival
        if (nt == TMAX) break;
        if (lane == 0) st->idle += nt - now;
        now = nt;
        continue;
      }
      // admissions are final: return the restart chunks the heads passed
      if (lane < P.n_rings) fifo_commit(lane, rhead);
      execute(n_evict, peak, waiting);
      if ((RING || SEG) && status) break;
    }
    finish();
  }

  __device__ void finish() {
    const uint32_t waiting = waiting_total();
    if (lane < P.n_rings) fifo_release_all(lane);
    flush_acc();
    __syncwarp();
    if (SEG) seg_finish();
    if (RING) ring_finish();
    const WarpStats S = *st;
    const uint64_t arrivals = S.arrivals, completed = S.completed;
    const u128 lat = S.sum_done_t - S.acc_done_a;
    const u128 ttft = S.sum_ft_t - S.acc_ft_a;
    // sum over arrivals of min(c, T) - a
    const u128 soj = lat + (u128)(arrivals - completed) * (u128)(uint64_t)P.T_t - (S.acc_arr - S.acc_done_a);
    uint64_t v = 0;
    switch (lane) {
      case SCHED_F_ARRIVALS: v = arrivals; break;
      case SCHED_F_ADMITTED: v = S.admitted; break;
      case SCHED_F_COMPLETED: v = completed; break;
      case SCHED_F_COMPLETED_AFTER_T: v = S.completed_after_T; break;
      case SCHED_F_COMPLETED_TOKENS: v = S.completed_tokens; break;
      case SCHED_F_FIRST_TOKENS: v = S.first_tokens; break;
      case SCHED_F_BATCHES: v = S.batches; break;
      case SCHED_F_REQUEST_STEPS: v = S.request_steps; break;
      case SCHED_F_PREFILL_STEPS: v = S.prefill_steps; break;
      case SCHED_F_EVICTIONS: v = S.evictions; break;
      case SCHED_F_BUSY_TICKS: v = (uint64_t)S.busy; break;
      case SCHED_F_IDLE_TICKS: v = (uint64_t)S.idle; break;
      case SCHED_F_LAT_LO: v = (uint64_t)lat; break;
      case SCHED_F_LAT_HI: v = (uint64_t)(lat >> 64); break;
      case SCHED_F_TTFT_LO: v = (uint64_t)ttft; break;
      case SCHED_F_TTFT_HI: v = (uint64_t)(ttft >> 64); break;
      case SCHED_F_SOJ_LO: v = (uint64_t)soj; break;
      case SCHED_F_SOJ_HI: v = (uint64_t)(soj >> 64); break;
      case SCHED_F_COMPLETION_BATCH_IDX: v = S.cbi; break;
      case SCHED_F_MAX_KV_PEAK: v = (uint64_t)S.max_kv; break;
      case SCHED_F_FINAL_WAITING: v = waiting; break;
      case SCHED_F_FINAL_RESIDENT: v = n_res; break;
      case SCHED_F_TRAJ_HASH: v = S.h; break;
      case SCHED_F_STATUS: v = status; break;
      case SCHED_F_NOW_STOP: v = (uint64_t)now; break;
      case SCHED_F_SUM_WAITING: v = S.sum_waiting; break;
      default: break;
    }
    if (lane < SCHED_NF) P.out[(size_t)lane * P.n_reps + rep] = v;
    if (TRACE && rep == 0 && lane == 0) *P.log_n = S.log_n;
  }
};

// blocks per SM the register allocation is sized for (launch bound): the
// two-class WAIT ring kernel runs best at 6 x 4 warps / 80 registers despite
// 72 B of spills (C2 WAIT 13.7 -> 13.0 ms; K = 1 and 3 lose at 6: C1 +1%,
// C4 rho=0.95 +7%), the other WAIT / class-ring kernels at 5 x 4 / 96
template <int POL, bool RING, int KC>
constexpr int kMinBlocks() {
  return (POL == SCHED_WAIT && RING && KC == 2) ? WAITSIM_WAIT2_MINB
       : (POL == SCHED_FCFS && RING && KC == 2) ? WAITSIM_FCFS2_MINB
       : (POL == SCHED_FCFS && RING && KC == 3) ? WAITSIM_FCFS3_MINB
       : (POL == SCHED_FCFS && RING && KC == 4) ? WAITSIM_FCFS4_MINB
       : (POL == SCHED_WAIT || RING) ? 5
       : (POL == SCHED_FCFS && KC == 1) ? WAITSIM_MEMBER_FCFS_MINB : 2;  // one-class member FCFS (marks)
}

// one-warp blocks (the warp's shared-memory window starts at offset 0: no
// per-warp base to rematerialise under register pressure)
template <int POL, bool RING, int KC, bool SEG = false>
__host__ __device__ constexpr bool kOneWarp() {
  return (SEG && KC > 0 && WAITSIM_SEG_ONEWARP) ||
         (!RING && !SEG && POL == SCHED_FCFS && KC == 1 && WAITSIM_MEMBER_FCFS_ONEWARP) ||
         RING && ((KC == 2 && POL == SCHED_WAIT && WAITSIM_WAIT2_ONEWARP) ||
                  (KC == 2 && POL == SCHED_FCFS && WAITSIM_FCFS2_ONEWARP) ||
                  (KC > 0 && KC != 2 && POL == SCHED_WAIT && WAITSIM_WAITK_ONEWARP) ||
                  (KC == 4 && POL == SCHED_FCFS && WAITSIM_FCFS4_ONEWARP) ||
                  (KC == 1 && POL == SCHED_FCFS && WAITSIM_FCFS1_ONEWARP));
}

template <int POL, bool TRACE, bool RING, bool SEG, int KC>
// WAIT and the class-ring engine: <= 4 warps per block, 5 blocks per SM ->
// <= 102 registers, 20 warps/SM (the ring engine's shared footprint is small,
// so registers bound its occupancy: measured C2 FCFS 128 registers / 16
// warps 20.9 ms -> 96 / 20 warps 18.7 ms; 80 / 24 warps spills, 20.7 ms);
// the member and segment engines are shared-memory bound: 128 registers
__global__ void __launch_bounds__(kOneWarp<POL, RING, KC, SEG>() ? 32 : (POL == SCHED_WAIT || RING) ? 128 : 256,
                                  kOneWarp<POL, RING, KC, SEG>() ? (SEG ? 16 : (RING ? 4 : 8) * kMinBlocks<POL, RING, KC>())
                                                                 : kMinBlocks<POL, RING, KC>())
    sim_kernel(const DevParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = kOneWarp<POL, RING, KC, SEG>() ? 0 : threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t slot = kOneWarp<POL, RING, KC, SEG>() ? blockIdx.x
                                                   : blockIdx.x * (blockDim.x >> 5) + (uint32_t)wib;  // SEG: global per-warp array
  WarpSim<POL, TRACE, RING, SEG, KC> sim(P, smem + (size_t)wib * P.warp_smem, lane, slot);
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(P.work_counter, 1u);
    i = __shfl_sync(FULL, i, 0);
    uint32_t r = i;
    if (P.fallback) {
      if (i >= *P.retry_count) break;
      r = P.retry_list[i];
    } else if (i >= P.n_reps) {
      break;
    }
    sim.run(r);
    if (!P.fallback && P.retry_list && sim.status == 1) {
      if (lane == 0) P.retry_list[atomicAdd(P.retry_count, 1u)] = r;  // re-run with the safe capacity
    } else if (sim.status && lane == 0) {
      atomicOr(P.status_mask, 1u << min(sim.status, 31u));
    }
  }
  sim.flush_stash();
}

template <int POL, bool TRACE, bool RING = false, bool SEG = false, int KC = 0>
cudaError_t launch_t(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s) {
  auto k = sim_kernel<POL, TRACE, RING, SEG, KC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, block, smem, s>>>(p);
  return cudaGetLastError();
}

template <int POL, bool TRACE, bool RING = false, bool SEG = false, int KC = 0>
cudaError_t occ_t(int block, size_t smem, int* bps) {
  auto k = sim_kernel<POL, TRACE, RING, SEG, KC>;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, k);
  if (e != cudaSuccess) return e;
  if (block > fa.maxThreadsPerBlock) { *bps = 0; return cudaSuccess; }  // beyond the launch bound
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, block, smem);
}


}  // namespace
}  // namespace waitsim
