// sched_api.cpp -- the C ABI of libsched (include/sched.h): config
// validation and upload, launch sizing, sched_run / sched_run_host /
// sched_run_trace.  All simulation work runs in sim_kernel.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sched.h"
#include "setup.h"
#include "sim_internal.h"
#include "walks.h"

using namespace waitsim;

// one launch configuration (engine + capacities + grid); the handle keeps one
// for the member engine (every policy, explicit traces) and, when eligible,
// one for the class-ring engine (sched_run of fixed-length WAIT / FCFS)
struct LaunchCfg {
  bool ring = false;
  bool seg = false;                          // NESTED segment engine (fallback: the member engine's safe launch)
  uint32_t seg_cap = 0;                      // seg: resident array capacity (records)
  uint32_t Rc = 0, Rc_safe = 0;              // member: residents; ring: staging slots
  uint32_t spare = 0;                        // ring: victim slots beyond Rc (8, 32 when evictions are expected)
  uint32_t rcap[32] = {}, rcap_safe[32] = {};  // ring: per-class ring capacity
  uint32_t warp_smem = 0, fb_warp_smem = 0;
  int grid = 0, block = 0, wpb = 0, blocks_per_sm = 0;
  int fb_grid = 0, fb_block = 0, fb_wpb = 0;
  bool fallback = false;
};

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(SCHED_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x)                                      \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)
}  // namespace

struct sched_s {
  SetupInput in;
  // Nested WAIT with one class and one segment IS WAIT with one type (P10,
  // reading R7; pinned on the oracle): its sched_run calls go to this WAIT
  // handle (class-ring engine for fixed lengths; C1 Nested 60 -> 47 ms)
  sched_s* twin = nullptr;
  uint32_t tok_budget = 0, max_resident_cfg = 0, spec_resident_cfg = 0;
  uint64_t pool_entries = 1ull << 24;  // restart pool capacity (entries), shared by a launch
  int device = 0;
  int64_t d0_t = 0, d1_t = 0;
  uint32_t max_lp = 0, min_l = 0;
  DevParams base{};
  // device-side tables
  uint64_t* d_cdf_thr = nullptr;
  uint16_t* d_cdf_val = nullptr;
  uint16_t* d_cdf_guide = nullptr;
  uint8_t* d_stage_info = nullptr;
  std::vector<uint64_t> h_cdf_thr;     // uploaded lazily by prepare()
  std::vector<uint16_t> h_cdf_val, h_cdf_guide;
  std::vector<uint8_t> h_stage_info;
  std::vector<int64_t> h_rf_B, h_rf_Lam;   // time-varying rate pieces
  std::vector<double> h_rf_scale;
  int64_t* d_rf_B = nullptr;
  int64_t* d_rf_Lam = nullptr;
  double* d_rf_scale = nullptr;
  bool tv_any = false;
  // scratch
  // restart-FIFO chunk pool
  int64_t* d_pool_a = nullptr;
  int64_t* d_pool_e = nullptr;
  uint32_t* d_pool_llp = nullptr;
  uint32_t* d_pool_next = nullptr;
  unsigned long long* d_pool_free = nullptr;  // [0] free-stack head, [1] bump counter (low word)
  uint32_t pool_chunks = 0;
  uint32_t* d_counter = nullptr;
  uint32_t* d_status = nullptr;              // sticky status mask (sched_get_status)
  uint64_t* d_out = nullptr;
  size_t out_cap = 0;
  // launch: main (speculative capacity) and fallback (safe capacity) per engine
  int sm_count = 0;
  LaunchCfg mem, rng, sg;
  bool use_ring = false;                     // sched_run uses the class-ring engine
  bool use_seg = false;                      // sched_run / sched_run_trace use the segment engine
  int64_t* d_seg_a = nullptr;                // segment engine: per-warp arrival-tick arrays
  void* d_ring_g = nullptr;                  // class-ring engine: per-warp ring records (16 B)
  uint64_t ring_g_cap = 0;
  uint8_t* d_ring_log = nullptr;             // class-ring engine: per-warp admission logs (2^16 B)
  uint32_t* d_pool_stash = nullptr;          // per-slot restart-chunk stashes
  uint64_t stash_words = 0;
  uint64_t ring_log_warps = 0;
  uint32_t ring_stride = 0;
  size_t seg_a_cap = 0;
  double n_star_c[32] = {};                  // fluid prompts in service per class
  double m_star = 0;                         // fluid KV occupancy M*
  double tv_peak = 1.0;                      // max time-varying rate / lambda (speculative sizing)
  uint32_t* d_retry = nullptr;
  size_t retry_cap = 0;
  double n_star_total = 0;  // fluid equilibrium prompts in service (0 = unknown)
  bool prepared = false;
};

namespace {

bool is_fcfs(int policy) { return policy == SCHED_FCFS || policy == SCHED_FCFS_ONGOING; }

// Resident capacity: FCFS holds at most B prompts; WAIT at most n_j per stage
// (invariant P14) plus one staged batch; NESTED: non-entry stages hold at
// most n_k, entry-stage queues are bounded by memory -- take a margin.
uint32_t round32(uint64_t x) { return (uint32_t)((std::max<uint64_t>(x, 32) + 31) & ~31ull); }

// speculative (typical-case) capacity; replications that exceed it are re-run
// with the safe capacity (derive_rc) by the fallback launch
uint32_t speculative_rc(const sched_s* h, uint32_t safe) {
  if (h->spec_resident_cfg) return std::min(safe, round32(h->spec_resident_cfg));
  const auto& in = h->in;
  uint64_t rc = safe;
  if (is_fcfs(in.policy)) {
    // FCFS residents ~ fluid prompts in service n* + margin
    // (time-varying rates: the stationary fluid estimate does not hold and
    // backlogs of the peak pieces fill B -- no speculation)
    if (h->n_star_total > 0 && h->tv_peak <= 1.0) rc = (uint64_t)(1.25 * h->n_star_total) + 64;
  } else if (in.policy == SCHED_NESTED) {
    // non-entry stages hold <= n_k each; entry queues stay near n_k (Lemma,
    // PAPER.md:2345-2373) -- margin 2 n_k per boundary
    uint64_t prev = 0, base = 0;
    for (size_t k = 0; k < in.seg_end.size(); ++k) {
      base += (uint64_t)in.thresholds[k] * (in.seg_end[k] - prev + (k ? 2 : 1));
      prev = in.seg_end[k];
    }
    rc = base + 64;
  }
  if (in.policy == SCHED_NESTED) {
    // memory caps the population: a resident holds l + s - 1 KV tokens, on
    // average (time-weighted over its l' + 1 iterations) E[(l'+1)(l + l'/2)]
    // / E[l'+1] (R26), so ~ M / that residents + margin
    double num = 0, den = 0;
    for (size_t c = 0; c < in.lambda.size(); ++c) {
      double wl = 0, el = 0, wp = 0, ep1 = 0, eq = 0;
      for (auto& e : in.l[c]) { wl += (double)e.second; el += (double)e.second * e.first; }
      for (auto& e : in.lp[c]) {
        const double y = e.first;
        wp += (double)e.second;
        ep1 += (double)e.second * (y + 1);
        eq += (double)e.second * (y + 1) * y / 2;
      }
      if (wl <= 0 || wp <= 0) continue;
      el /= wl; ep1 /= wp; eq /= wp;
      num += in.lambda[c] * (ep1 * el + eq);
      den += in.lambda[c] * ep1;
    }
    // when memory binds (M^pi = sum_k n_k sum_{s in seg k} (E[l] + s) > M,
    // reading R9) LIFO eviction keeps young, small residents: wider margin
    double el = 0, lam = 0, mpi = 0;
    for (size_t c = 0; c < in.lambda.size(); ++c) {
      double w = 0, e = 0;
      for (auto& t : in.l[c]) { w += (double)t.second; e += (double)t.second * t.first; }
      if (w > 0) { el += in.lambda[c] * e / w; lam += in.lambda[c]; }
    }
    el = lam > 0 ? el / lam : 1.0;
    uint32_t prev = 0;
    for (size_t k = 0; k < in.seg_end.size() && k < in.thresholds.size(); ++k) {
      for (uint32_t st = (k ? prev + 1 : 0); st <= in.seg_end[k]; ++st) mpi += in.thresholds[k] * (el + st);
      prev = in.seg_end[k];
    }
    const double factor = mpi > (double)in.M ? 2.0 : 1.4;
    if (num > 0 && den > 0)
      rc = std::min<uint64_t>(rc, (uint64_t)(factor * (double)in.M / (num / den)) + 96);
  }
  return std::min(safe, round32(rc));
}

uint32_t derive_rc(const sched_s* h) {
  if (h->max_resident_cfg) return h->max_resident_cfg;
  uint64_t rc = 0;
  const auto& in = h->in;
  if (is_fcfs(in.policy)) {
    rc = in.B;
  } else if (in.policy == SCHED_WAIT) {
    for (size_t c = 0; c < in.thresholds.size(); ++c) {
      uint32_t mx = 0;
      for (auto& e : in.lp[c]) mx = std::max<uint32_t>(mx, e.first);
      rc += (uint64_t)in.thresholds[c] * (mx + 1);
    }
  } else {
    uint64_t prev = 0, base = 0;
    for (size_t k = 0; k < in.seg_end.size(); ++k) {
      base += (uint64_t)in.thresholds[k] * (in.seg_end[k] - prev);
      prev = in.seg_end[k];
    }
    rc = base + std::max<uint64_t>(256, base / 2) + in.thresholds[0];
    rc = std::min<uint64_t>(rc, (uint64_t)in.M / std::max<uint32_t>(1, h->min_l) + in.thresholds[0]);
  }
  rc = std::max<uint64_t>(rc, 32);
  rc = (rc + 31) & ~31ull;
  // default cap 4096 (64 KiB of shared memory per warp); larger needs an
  // explicit max_resident.  Overflow is reported per replication (status 1).
  return (uint32_t)std::min<uint64_t>(rc, 4096);
}

int prepare(sched_s* h) {
  if (h->prepared) return 0;
  if (!is_fcfs(h->in.policy) && h->in.thresholds.empty())
    return fail(SCHED_E_INVALID, "thresholds not set: pass them in sched_config or call sched_thresholds");
  CK(cudaSetDevice(h->device));
  if (!h->d_cdf_thr) {
    CK(cudaMalloc(&h->d_cdf_thr, h->h_cdf_thr.size() * 8));
    CK(cudaMalloc(&h->d_cdf_val, h->h_cdf_val.size() * 2));
    CK(cudaMemcpy(h->d_cdf_thr, h->h_cdf_thr.data(), h->h_cdf_thr.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_cdf_val, h->h_cdf_val.data(), h->h_cdf_val.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&h->d_cdf_guide, h->h_cdf_guide.size() * 2));
    CK(cudaMemcpy(h->d_cdf_guide, h->h_cdf_guide.data(), h->h_cdf_guide.size() * 2, cudaMemcpyHostToDevice));
    h->base.cdf_guide = h->d_cdf_guide;
    if (!h->h_stage_info.empty()) {
      CK(cudaMalloc(&h->d_stage_info, h->h_stage_info.size()));
      CK(cudaMemcpy(h->d_stage_info, h->h_stage_info.data(), h->h_stage_info.size(), cudaMemcpyHostToDevice));
    }
    h->base.cdf_thr = h->d_cdf_thr;
    h->base.cdf_val = h->d_cdf_val;
    h->base.stage_info = h->d_stage_info;
    h->base.tv_any = h->tv_any ? 1 : 0;
    if (h->tv_any) {
      const size_t n = h->h_rf_B.size();
      CK(cudaMalloc(&h->d_rf_B, n * 8));
      CK(cudaMalloc(&h->d_rf_Lam, n * 8));
      CK(cudaMalloc(&h->d_rf_scale, n * 8));
      CK(cudaMemcpy(h->d_rf_B, h->h_rf_B.data(), n * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->d_rf_Lam, h->h_rf_Lam.data(), n * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->d_rf_scale, h->h_rf_scale.data(), n * 8, cudaMemcpyHostToDevice));
      h->base.rf_B = h->d_rf_B;
      h->base.rf_Lam = h->d_rf_Lam;
      h->base.rf_scale = h->d_rf_scale;
    }
  }
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, h->device));
  h->sm_count = prop.multiProcessorCount;
  const int K = (int)h->in.lambda.size();
  if (h->n_star_total == 0 && h->in.policy != SCHED_NESTED) {
    sched_threshold_report rep;
    std::vector<uint32_t> ch;
    std::string err;
    try {
      if (compute_thresholds(h->in, 0, 0, 0, &rep, &ch, &err) == 0)
        for (int c = 0; c < K && c < 32; ++c) { h->n_star_total += rep.n_star[c]; h->n_star_c[c] = rep.n_star[c]; }
      h->m_star = rep.M_star;
    } catch (...) {
    }
  }
  // NESTED segment geometry (segment engine): entry stage b_k = e_{k-1}+1
  // (b_0 = 0: the FIFO), W_k = e_k - b_k non-entry stages, histogram /
  // cohort-ring offsets
  if (h->in.policy == SCHED_NESTED) {
    uint32_t ho = 0, co = 0;
    for (size_t k = 0; k < h->in.seg_end.size() && k < 32; ++k) {
      const uint32_t b = k ? h->in.seg_end[k - 1] + 1 : 0u, w = h->in.seg_end[k] - b;
      h->base.seg_b[k] = b;
      h->base.seg_w[k] = w;
      h->base.hoff[k] = ho;
      h->base.coff[k] = co;
      ho += w;
      co += w + 1;
    }
    h->base.hsize = ho;
    h->base.csize = co;
  }
  // class-ring engine: cohort-count rings, l'_c + 1 slots per class
  if (h->in.policy != SCHED_NESTED) {
    uint32_t co = 0;
    for (int c = 0; c < (int)h->in.lambda.size() && c < 32; ++c) {
      h->base.ccoff[c] = co;
      co += (uint32_t)h->in.lp[c].back().first + 1u;
    }
    h->base.ccsize = co;
  }
  // choose warps per block maximising resident warps per SM
  auto size_launch = [&](bool ring, uint32_t records, uint32_t* wsm, int* wpb_out, int* bps_out,
                         uint32_t seg_cap = 0) -> int {
    *wsm = warp_smem_bytes(records, K, h->tv_any, ring, h->in.policy == SCHED_NESTED,
                           h->in.policy == SCHED_WAIT ? (uint32_t)K : 1u, seg_cap, h->base.hsize,
                           h->base.csize, ring ? h->base.ccsize * 4u : 0u);
    int best_w = 0;
    const int cands[] = {8, 4, 2, 1};
    for (int wpb : cands) {
      if ((h->in.policy == SCHED_WAIT || ring) && wpb > 4) continue;  // kernel launch bound: 128 threads
      const size_t smem = (size_t)wpb * *wsm;
      if (smem > (size_t)prop.sharedMemPerBlockOptin) continue;
      // max blocks per SM from shared memory and registers (occupancy API)
      int bps = 0;
      const cudaError_t e = sim_occupancy(h->in.policy, 0, wpb * 32, smem, &bps, seg_cap ? 2 : ring ? 1 : 0, K);
      if (e != cudaSuccess) {  // block larger than the kernel's launch bound: not a candidate
        cudaGetLastError();
        continue;
      }
      if (bps * wpb > best_w) { best_w = bps * wpb; *wpb_out = wpb; *bps_out = bps; }
    }
    if (best_w == 0)
      return fail(SCHED_E_INVALID, "resident capacity too large for shared memory (" +
                                       std::to_string(records) + " records per replication)");
    return 0;
  };
  auto size_cfg = [&](LaunchCfg& L) -> int {
    uint32_t rec = L.Rc, rec_safe = L.Rc_safe;
    if (L.ring) {
      rec += L.spare;  // spare staging slots: eviction-round victims (the rings are in global memory)
      rec_safe += L.spare;
    }
    L.fallback = rec < rec_safe;
    for (int c = 0; L.ring && c < K; ++c) L.fallback = L.fallback || L.rcap[c] < L.rcap_safe[c];
    int wpb = 1, bps = 0;
    if (int rc = size_launch(L.ring, rec, &L.warp_smem, &wpb, &bps)) return rc;
    L.wpb = wpb;
    L.blocks_per_sm = bps;
    L.block = wpb * 32;
    L.grid = h->sm_count * bps;
    L.fb_wpb = L.wpb; L.fb_block = L.block; L.fb_grid = 0; L.fb_warp_smem = L.warp_smem;
    if (L.fallback) {
      int fw = 1, fb = 0;
      if (int rc = size_launch(L.ring, rec_safe, &L.fb_warp_smem, &fw, &fb)) return rc;
      L.fb_wpb = fw;
      L.fb_block = fw * 32;
      L.fb_grid = h->sm_count * fb;
    }
    return 0;
  };
  // member engine (every policy; explicit traces)
  h->mem = LaunchCfg{};
  h->mem.Rc_safe = derive_rc(h);
  h->mem.Rc = speculative_rc(h, h->mem.Rc_safe);
  if (int rc = size_cfg(h->mem)) return rc;
  // class-ring engine: WAIT / FCFS with fixed per-class lengths
  h->use_ring = false;
  const char* eng = getenv("WAITSIM_ENGINE");
  bool fixed = true;
  for (int c = 0; c < K; ++c) fixed = fixed && h->in.l[c].size() == 1 && h->in.lp[c].size() == 1;
  if (h->in.policy != SCHED_NESTED && fixed && !(eng && std::string(eng) == "member")) {
    LaunchCfg& L = h->rng;
    L = LaunchCfg{};
    L.ring = true;
    const auto& in = h->in;
    uint64_t safe_tot = 0;
    for (int c = 0; c < K; ++c) {
      const uint32_t l = (uint32_t)in.l[c][0].first, lp = (uint32_t)in.lp[c][0].first;
      uint64_t cs;
      if (h->max_resident_cfg) cs = h->max_resident_cfg;
      else if (in.policy == SCHED_WAIT) cs = (uint64_t)in.thresholds[c] * lp;  // P14: <= n_c per stage
      else cs = std::min<uint64_t>(in.B, (uint64_t)in.M / l);
      L.rcap_safe[c] = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(cs, 8192));
      safe_tot += L.rcap_safe[c];
    }
    if (in.policy == SCHED_WAIT) {
      uint64_t st = 0;
      for (int c = 0; c < K; ++c) st += in.thresholds[c];
      L.Rc_safe = (uint32_t)std::min<uint64_t>(st, 8192);
    } else {
      L.Rc_safe = h->max_resident_cfg ? h->max_resident_cfg : in.B;
    }
    L.Rc_safe = std::max<uint32_t>(L.Rc_safe, 1);
    // speculative capacities: FCFS residents ~ fluid prompts in service n*_c
    // + margin, staging ~ fluid admissions per batch + margin
    L.Rc = L.Rc_safe;
    for (int c = 0; c < K; ++c) L.rcap[c] = L.rcap_safe[c];
    if (h->spec_resident_cfg) {
      for (int c = 0; c < K; ++c)
        L.rcap[c] = std::max<uint32_t>(1, std::min<uint32_t>(L.rcap_safe[c],
                       (uint32_t)((uint64_t)h->spec_resident_cfg * L.rcap_safe[c] / std::max<uint64_t>(1, safe_tot))));
      L.Rc = std::min<uint32_t>(L.Rc_safe, std::max<uint32_t>(32, h->spec_resident_cfg / 4));
    } else if (is_fcfs(in.policy) && h->n_star_total > 0) {
      // FCFS residents ~ fluid prompts in service n*_c, scaled
      // by M / M* when memory binds and by B / n* when the batch cap binds
      // (WAIT needs no speculation: n_c per stage exactly, P14)
      const double fm = h->m_star > 0 ? std::min(1.0, (double)in.M / h->m_star) : 1.0;
      const double tot = std::min((double)in.B, fm * h->n_star_total * h->tv_peak);
      double adm = 0;
      for (int c = 0; c < K; ++c) {
        const double share = h->n_star_c[c] / h->n_star_total;
        // class rings live in global memory (no occupancy cost): under
        // time-varying rates the stationary estimate misses the peak-piece
        // backlog (every C3a_tv replication overflowed it), so they stay safe
        if (h->tv_peak <= 1.0) L.rcap[c] = std::min<uint32_t>(L.rcap_safe[c], (uint32_t)(1.2 * tot * share) + 48);
        adm += h->tv_peak * h->n_star_c[c] / (double)(in.lp[c][0].first + 1);
      }
      // admissions per batch ~ Poisson(adm): mean + 8 sd + 16 (tail < 1e-12)
      L.Rc = std::min<uint32_t>(L.Rc_safe, round32((uint64_t)(adm + 8.0 * std::sqrt(adm)) + 16));
    }
    L.spare = 0;  // LIFO victims are read in place (admission log): no staging slots
    // a ring footprint that does not fit in shared memory only makes the
    // ring engine ineligible (the member engine runs), unless it was forced
    const bool forced = eng && std::string(eng) == "ring";
    if (int rc = size_cfg(L)) {
      if (forced) return rc;
      L.grid = 0;
    }
    // the ring engine does O(classes + admissions) work per batch and keeps
    // only staging slots and per-clock cohort counts in shared memory (the
    // member records live in global memory, read by evictions and at the
    // end of a replication): every eligible configuration uses it
    h->use_ring = L.grid > 0;
    if (h->use_ring) {
      uint64_t stride = 0;
      for (int c = 0; c < K; ++c) stride += L.rcap_safe[c];
      const uint64_t warps = std::max<uint64_t>((uint64_t)L.grid * L.wpb, (uint64_t)L.fb_grid * L.fb_wpb);
      h->ring_stride = (uint32_t)stride;
      if (warps * stride > h->ring_g_cap) {
        cudaFree(h->d_ring_g);
        h->d_ring_g = nullptr;
        CK(cudaMalloc(&h->d_ring_g, warps * stride * 16));  // {arrival | ft, clock} per record
        h->ring_g_cap = warps * stride;
      }
      if (warps > h->ring_log_warps) {
        cudaFree(h->d_ring_log);
        h->d_ring_log = nullptr;
        CK(cudaMalloc(&h->d_ring_log, warps << 16));
        h->ring_log_warps = warps;
      }
    }
  }
  // segment engine (NESTED): O(entry-stage takes + admissions) per batch
  // instead of a pass over every resident; replications
  // that overflow its array re-run on the member engine's safe launch
  h->use_seg = false;
  // measured exceptions, where the member engine wins: a single segment
  // (C1 Nested: nothing to skip, 84 vs 89 ms) and decode-length marks with
  // M^pi > M (C5: thrashing LIFO eviction of mostly entry-stage residents,
  // tombstones of mid-segment completions: 2.46 vs 2.89 s per 1,818 s)
  bool seg_wins = true;
  if (h->in.policy == SCHED_NESTED) {
    bool marks = false;
    double el = 0, lam = 0, mpi = 0;
    for (size_t c = 0; c < h->in.lambda.size(); ++c) {
      marks = marks || h->in.lp[c].size() > 1;
      double w = 0, e = 0;
      for (auto& t : h->in.l[c]) { w += (double)t.second; e += (double)t.second * t.first; }
      if (w > 0) { el += h->in.lambda[c] * e / w; lam += h->in.lambda[c]; }
    }
    el = lam > 0 ? el / lam : 1.0;
    uint32_t prev = 0;
    for (size_t k = 0; k < h->in.seg_end.size() && k < h->in.thresholds.size(); ++k) {
      for (uint32_t st = (k ? prev + 1 : 0); st <= h->in.seg_end[k]; ++st) mpi += h->in.thresholds[k] * (el + st);
      prev = h->in.seg_end[k];
    }
    seg_wins = h->in.seg_end.size() > 1 && !(marks && mpi > (double)h->in.M);
  }
  const bool seg_forced = eng && std::string(eng) == "seg";
  if (h->in.policy == SCHED_NESTED && !(eng && std::string(eng) == "member") && (seg_wins || seg_forced)) {
    LaunchCfg& L = h->sg;
    L = LaunchCfg{};
    L.seg = true;
    L.Rc = L.Rc_safe = round32(h->in.thresholds[0]);  // staged admissions: n_1 per batch
    // array capacity = the member engine's speculative population (live
    // residents) x f + two admission batches: room for the tombstones of
    // mid-segment completions between compactions.  f in [1.2, 1.5]: the
    // largest capacity among those reaching the most resident warps per SM
    // (shared memory bounds the engine's occupancy; measured C3a 10 -> 12
    // warps 59.4 -> 54.3 ms, C3b 6 -> 8 warps 21.7 -> 17.3 ms; f = 1.0 already
    // overflows 16% of C3a's replications into the fallback launch)
    auto cap_of = [&](double f) {
      return round32((uint64_t)(f * h->mem.Rc) + 2ull * h->in.thresholds[0]);
    };
    int wpb = 1, bps = 0, best = -1;
    uint32_t wsm = 0;
    const char* fs = getenv("WAITSIM_SEG_CAP");
    const bool fixed_f = fs || h->spec_resident_cfg;  // forced, or an explicit speculative capacity: f = 1.5
    for (int step = 0; step <= (fixed_f ? 0 : 15); ++step) {
      const uint32_t cap = fs ? cap_of(std::max(0.1, atof(fs))) : cap_of(1.5 - 0.02 * step);  // step 0: f = 1.5
      int w = 1, b = 0;
      if (size_launch(false, L.Rc, &wsm, &w, &b, cap) != 0) continue;
      if (w * b > best) {
        best = w * b;
        wpb = w;
        bps = b;
        L.seg_cap = cap;
        L.warp_smem = wsm;
      }
    }
    if (best > 0) {
      L.wpb = wpb;
      L.blocks_per_sm = bps;
      L.block = wpb * 32;
      L.grid = h->sm_count * bps;
      L.fallback = true;  // the member engine's safe launch
      h->use_seg = true;
    } else if (seg_forced) {
      return SCHED_E_INVALID;
    }
    if (h->use_seg) {
      const size_t need = (size_t)L.grid * L.wpb * L.seg_cap;
      if (need > h->seg_a_cap) {
        cudaFree(h->d_seg_a);
        h->d_seg_a = nullptr;
        CK(cudaMalloc(&h->d_seg_a, need * 8));
        h->seg_a_cap = need;
      }
    }
  }
  const int n_rings = h->in.policy == SCHED_WAIT ? K : 1;
  if (!h->d_pool_a) {
    // one pool of restart-FIFO chunks for every replication of a launch:
    // memory follows the evictions that actually wait, not warps x capacity
    const uint64_t chunks = std::max<uint64_t>(1, h->pool_entries / kRestartChunk);
    if (chunks >= kNoChunk) return fail(SCHED_E_INVALID, "restart pool too large");
    h->pool_chunks = (uint32_t)chunks;
    const size_t n = (size_t)chunks * kRestartChunk;
    CK(cudaMalloc(&h->d_pool_a, n * 8));
    CK(cudaMalloc(&h->d_pool_e, n * 8));
    CK(cudaMalloc(&h->d_pool_llp, n * 4));
    CK(cudaMalloc(&h->d_pool_next, (size_t)chunks * 4));
    CK(cudaMalloc(&h->d_pool_free, 16));
    const unsigned long long init[2] = {(unsigned long long)kNoChunk, 0ull};  // empty stack, nothing handed out
    CK(cudaMemcpy(h->d_pool_free, init, 16, cudaMemcpyHostToDevice));
  }
  if (!h->d_counter) CK(cudaMalloc(&h->d_counter, 16));  // [main, fallback, retry count]
  if (!h->d_status) {
    CK(cudaMalloc(&h->d_status, 4));
    CK(cudaMemset(h->d_status, 0, 4));
  }
  DevParams& p = h->base;
  p.n_rings = n_rings;
  for (size_t i = 0; i < h->in.thresholds.size() && i < 32; ++i) p.thr[i] = h->in.thresholds[i];
  for (int c = 0; c < K; ++c)
    p.fl[c] = (uint32_t)h->in.l[c][0].first | ((uint32_t)h->in.lp[c].back().first << 16);
  p.pool_a = h->d_pool_a;
  p.pool_e = h->d_pool_e;
  p.pool_llp = h->d_pool_llp;
  p.pool_next = h->d_pool_next;
  p.pool_free = h->d_pool_free;
  p.pool_bump = (uint32_t*)(h->d_pool_free + 1);
  p.pool_chunks = h->pool_chunks;
  p.work_counter = h->d_counter;
  p.status_mask = h->d_status;
  {
    // per-slot restart-chunk stashes: slots of the widest launch of any engine
    uint64_t slots = 1;
    for (const LaunchCfg* L : {&h->mem, &h->rng, &h->sg}) {
      slots = std::max<uint64_t>(slots, (uint64_t)L->grid * L->wpb);
      slots = std::max<uint64_t>(slots, (uint64_t)L->fb_grid * L->fb_wpb);
    }
    const uint64_t words = slots * (uint64_t)n_rings * 12;
    if (words > h->stash_words) {
      // chunks held by an old stash array are not returned (bounded: 11 per slot and ring)
      cudaFree(h->d_pool_stash);
      h->d_pool_stash = nullptr;
      CK(cudaMalloc(&h->d_pool_stash, words * 4));
      CK(cudaMemset(h->d_pool_stash, 0, words * 4));
      h->stash_words = words;
    }
    p.pool_stash = h->d_pool_stash;
    // stashes hold at most half of the pool, so a small pool is not
    // exhausted by chunks parked in idle stashes (a stash below ~11 chunks
    // sends eviction-heavy FIFOs back to the contended free stack: C4
    // rho=0.95 WAIT 8.4 ms with 11, 60 ms with 7)
    const uint64_t share = (uint64_t)h->pool_chunks / (2 * slots * (uint64_t)n_rings);
    p.stash_lim = (uint32_t)std::min<uint64_t>(11, share);
    p.bump_n = std::min<uint32_t>(4, p.stash_lim + 1);
  }
  p.ring_g = h->d_ring_g;
  p.ring_log = h->d_ring_log;
  p.ring_stride = h->ring_stride;
  h->prepared = true;
  return 0;
}

void set_offsets(DevParams& p) {
  p.off_csum = layout_off_csum(p.K, p.tv_any != 0);
  p.off_rr = layout_off_rr(p.Rc, p.K, p.tv_any != 0, p.policy == SCHED_NESTED);
}

// capacities of one launch of configuration L (safe = the fallback launch)
void set_caps(DevParams& p, const LaunchCfg& L, bool safe, int K) {
  p.ring_engine = L.ring ? 1u : 0u;
  p.seg_engine = 0;
  p.spare = L.spare;
  p.Rc = safe ? L.Rc_safe : L.Rc;
  p.warp_smem = safe ? L.fb_warp_smem : L.warp_smem;
  uint32_t off = 0;
  for (int c = 0; c < K; ++c) {
    p.rcap[c] = L.ring ? (safe ? L.rcap_safe[c] : L.rcap[c]) : 0u;
    p.roff[c] = off;
    off += p.rcap[c];
  }
  set_offsets(p);
}

int launch(sched_s* h, DevParams p, cudaStream_t st, const LaunchCfg& L) {
  const int K = p.K;
  if (L.seg) {
    // segment engine; replications that overflow its array re-run on the
    // member engine with the safe capacity
    CK(cudaMemsetAsync(h->d_counter, 0, 16, st));
    if (p.n_reps > h->retry_cap) {
      cudaFree(h->d_retry);
      h->d_retry = nullptr;
      CK(cudaMalloc(&h->d_retry, (size_t)p.n_reps * 4));
      h->retry_cap = p.n_reps;
    }
    DevParams q = p;
    q.work_counter = h->d_counter;
    q.retry_count = h->d_counter + 2;
    q.retry_list = h->d_retry;
    q.fallback = 0;
    q.ring_engine = 0;
    q.seg_engine = 1;
    q.seg_cap = L.seg_cap;
    q.seg_a = h->d_seg_a;
    q.Rc = L.Rc;
    q.warp_smem = L.warp_smem;
    set_offsets(q);
    int grid = L.grid;
    if ((int64_t)p.n_reps < (int64_t)grid * L.wpb) grid = std::max<int>(1, (int)((p.n_reps + L.wpb - 1) / L.wpb));
    CK(launch_sim(q, grid, L.block, (size_t)L.wpb * L.warp_smem, st));
    const LaunchCfg& M = h->mem;
    DevParams f = p;
    f.seg_engine = 0;
    f.seg_cap = 0;
    f.fallback = 1;
    f.work_counter = h->d_counter + 1;
    f.retry_count = h->d_counter + 2;
    f.retry_list = h->d_retry;
    set_caps(f, M, M.fallback, K);
    const int fwpb = M.fallback ? M.fb_wpb : M.wpb, fblock = M.fallback ? M.fb_block : M.block;
    const int fmax = M.fallback ? M.fb_grid : M.grid;
    const int fgrid = std::min(fmax, std::max(1, (int)((p.n_reps + fwpb - 1) / fwpb)));
    CK(launch_sim(f, fgrid, fblock, (size_t)fwpb * f.warp_smem, st));
    return 0;
  }
  CK(cudaMemsetAsync(h->d_counter, 0, 16, st));
  p.work_counter = h->d_counter;
  p.retry_count = h->d_counter + 2;
  p.retry_list = nullptr;
  p.fallback = 0;
  if (L.fallback) {
    if (p.n_reps > h->retry_cap) {
      cudaFree(h->d_retry);
      h->d_retry = nullptr;
      CK(cudaMalloc(&h->d_retry, (size_t)p.n_reps * 4));
      h->retry_cap = p.n_reps;
    }
    p.retry_list = h->d_retry;
  }
  set_caps(p, L, false, K);
  const size_t smem = (size_t)L.wpb * L.warp_smem;
  int grid = L.grid;
  const int warps = grid * L.wpb;
  if ((int64_t)p.n_reps < warps) grid = std::max<int>(1, (int)((p.n_reps + L.wpb - 1) / L.wpb));
  CK(launch_sim(p, grid, L.block, smem, st));
  if (L.fallback) {
    // replications that overflowed the speculative capacity, re-run safely
    DevParams q = p;
    q.fallback = 1;
    q.work_counter = h->d_counter + 1;
    set_caps(q, L, true, K);
    const int fgrid = std::min(L.fb_grid, std::max(1, (int)((p.n_reps + L.fb_wpb - 1) / L.fb_wpb)));
    CK(launch_sim(q, fgrid, L.fb_block, (size_t)L.fb_wpb * L.fb_warp_smem, st));
  }
  return 0;
}

// the handle a sched_run of h executes on: h, or its WAIT twin (P10) with
// h's current thresholds, unless WAITSIM_ENGINE forces a Nested engine
sched_s* run_target(sched_s* h) {
  if (!h->twin) return h;
  const char* eng = getenv("WAITSIM_ENGINE");
  if (eng && (std::string(eng) == "member" || std::string(eng) == "seg")) return h;
  if (h->twin->in.thresholds != h->in.thresholds) {
    h->twin->in.thresholds = h->in.thresholds;
    h->twin->prepared = false;
  }
  return h->twin;
}

bool table_ok(const uint32_t* off, const uint64_t* w, uint32_t c) {
  if (off[c + 1] <= off[c]) return false;
  uint64_t tot = 0;
  for (uint32_t i = off[c]; i < off[c + 1]; ++i) tot |= w[i];
  return tot != 0;
}

}  // namespace

extern "C" {

const char* sched_last_error(void) { return g_err.c_str(); }

int sched_create(sched_t* out, const sched_config* cfg) {
  if (!out || !cfg) return fail(SCHED_E_INVALID, "null argument");
  *out = nullptr;
  const uint32_t K = cfg->K;
  if (K == 0 || K > 32) return fail(SCHED_E_INVALID, "K must be 1..32");
  if (!cfg->lambda || !cfg->l_off || !cfg->l_val || !cfg->l_w || !cfg->lp_off || !cfg->lp_val ||
      !cfg->lp_w)
    return fail(SCHED_E_INVALID, "null table pointer");
  if (!(cfg->d0_s > 0) || !(cfg->d1_s >= 0)) return fail(SCHED_E_INVALID, "need d0 > 0, d1 >= 0");
  if (cfg->M < 1) return fail(SCHED_E_INVALID, "M must be >= 1");
  if (cfg->tau_b0 < 0) return fail(SCHED_E_INVALID, "tau_b0 must be >= 0");
  if (cfg->policy < SCHED_WAIT || cfg->policy > SCHED_FCFS_ONGOING) return fail(SCHED_E_INVALID, "bad policy");
  sched_s* h = new sched_s();
  SetupInput& in = h->in;
  in.d0_s = cfg->d0_s; in.d1_s = cfg->d1_s; in.M = cfg->M; in.policy = cfg->policy; in.B = cfg->B;
  uint32_t max_lp = 0, min_l = 0xFFFF, max_l = 0;
  std::vector<uint64_t> thr_all;
  std::vector<uint16_t> val_all, guide_all;
  for (uint32_t c = 0; c < K; ++c) {
    if (!(cfg->lambda[c] >= 0) || std::isinf(cfg->lambda[c])) { delete h; return fail(SCHED_E_INVALID, "lambda must be finite and >= 0"); }
    if (!table_ok(cfg->l_off, cfg->l_w, c) || !table_ok(cfg->lp_off, cfg->lp_w, c)) {
      delete h;
      return fail(SCHED_E_INVALID, "empty or zero-weight length table");
    }
    in.lambda.push_back(cfg->lambda[c]);
    Table lt, lpt;
    uint32_t cmax_l = 0, cmax_lp = 0;
    for (uint32_t i = cfg->l_off[c]; i < cfg->l_off[c + 1]; ++i) {
      if (cfg->l_val[i] < 1) { delete h; return fail(SCHED_E_INVALID, "prefill length must be >= 1"); }
      lt.push_back({cfg->l_val[i], cfg->l_w[i]});
      if (cfg->l_w[i]) { cmax_l = std::max<uint32_t>(cmax_l, cfg->l_val[i]); min_l = std::min<uint32_t>(min_l, cfg->l_val[i]); }
    }
    for (uint32_t i = cfg->lp_off[c]; i < cfg->lp_off[c + 1]; ++i) {
      if (cfg->lp_val[i] < 1 || cfg->lp_val[i] > 32767) { delete h; return fail(SCHED_E_INVALID, "decode length must be 1..32767"); }
      lpt.push_back({cfg->lp_val[i], cfg->lp_w[i]});
      if (cfg->lp_w[i]) cmax_lp = std::max<uint32_t>(cmax_lp, cfg->lp_val[i]);
    }
    if (cfg->lambda[c] > 0 && (int64_t)cmax_l + cmax_lp > cfg->M) {
      delete h;
      return fail(SCHED_E_UNSATISFIABLE, "some l + l' exceeds M: that prompt can never complete");
    }
    max_lp = std::max(max_lp, cmax_lp);
    max_l = std::max(max_l, cmax_l);
    in.l.push_back(lt);
    in.lp.push_back(lpt);
    // integer CDF tables: thr_i = floor(cum_i 2^32 / W)
    for (int which = 0; which < 2; ++which) {
      const Table& t = which ? lpt : lt;
      unsigned __int128 W = 0, cum = 0;
      for (auto& e : t) W += e.second;
      ClassParam& cp = h->base.cls[c];
      (which ? cp.lp_off : cp.l_off) = (uint32_t)thr_all.size();
      (which ? cp.lp_n : cp.l_n) = (uint32_t)t.size();
      const size_t off0 = thr_all.size();
      for (size_t i = 0; i < t.size(); ++i) {
        cum += t[i].second;
        uint64_t th = (uint64_t)((cum << 32) / W);
        if (i + 1 == t.size()) th = (uint64_t)1 << 32;
        thr_all.push_back(th);
        val_all.push_back(t[i].first);
      }
      // guide table: guide[j] = min{i : j 2^(32-lg) < thr_i} (the answer for
      // the lowest x of bucket j); the device scans forward from it
      uint32_t lg = 1;
      while (lg < 12 && ((size_t)1 << lg) < t.size()) ++lg;
      (which ? cp.lp_goff : cp.l_goff) = (uint32_t)guide_all.size();
      (which ? cp.lp_n : cp.l_n) |= lg << 24;
      size_t i = 0;
      for (uint64_t j = 0; j < ((uint64_t)1 << lg); ++j) {
        const uint64_t x0 = j << (32 - lg);
        while (thr_all[off0 + i] <= x0) ++i;
        guide_all.push_back((uint16_t)i);
      }
    }
    h->base.cls[c].gap_scale = cfg->lambda[c] > 0 ? 1e12 / cfg->lambda[c] : 0.0;
    // time-varying pieces: start ticks, integrated rate (2^-32 expected
    // arrivals), inverse-rate tick scale
    std::vector<std::pair<double, double>> pieces;
    if (cfg->rf_off && cfg->rf_off[c + 1] > cfg->rf_off[c]) {
      const uint32_t a = cfg->rf_off[c], b = cfg->rf_off[c + 1];
      if (!cfg->rf_t || !cfg->rf_rate || b - a > 32 || cfg->rf_t[a] != 0.0) {
        delete h;
        return fail(SCHED_E_INVALID, "rate pieces: need rf_t/rf_rate, <= 32 pieces, first start 0");
      }
      h->base.cls[c].rf_off = (uint32_t)h->h_rf_B.size();
      h->base.cls[c].rf_n = b - a;
      int64_t Lam = 0;
      for (uint32_t i = a; i < b; ++i) {
        const double r = cfg->rf_rate[i];
        if (!(r >= 0) || std::isinf(r) || (i > a && !(cfg->rf_t[i] > cfg->rf_t[i - 1]))) {
          delete h;
          return fail(SCHED_E_INVALID, "rate pieces: rates >= 0, increasing starts");
        }
        const int64_t B = std::llround(cfg->rf_t[i] * 1e12);
        if (i > a) {
          const int64_t Bp = h->h_rf_B.back();
          const double rp = cfg->rf_rate[i - 1];
          Lam += (int64_t)(((rp * (double)(B - Bp)) * 4294967296.0) / 1e12);
        }
        h->h_rf_B.push_back(B);
        h->h_rf_Lam.push_back(Lam);
        h->h_rf_scale.push_back(r > 0 ? 1e12 / (r * 4294967296.0) : 0.0);
        pieces.push_back({cfg->rf_t[i], r});
        // peak load relative to the constant rate the fluid setup uses
        if (cfg->lambda[c] > 0) h->tv_peak = std::max(h->tv_peak, r / cfg->lambda[c]);
      }
      h->tv_any = true;
    }
    in.rf.push_back(pieces);
  }
  h->max_lp = max_lp;
  h->min_l = min_l;
  if (is_fcfs(cfg->policy)) {
    if (cfg->B < 1) { delete h; return fail(SCHED_E_INVALID, "FCFS needs B >= 1"); }
    if (cfg->tok_budget && cfg->tok_budget < max_l) { delete h; return fail(SCHED_E_INVALID, "tok_budget below the largest prefill length"); }
  }
  if (cfg->policy == SCHED_NESTED) {
    if (cfg->n_seg < 1 || cfg->n_seg > 32 || !cfg->seg_end) { delete h; return fail(SCHED_E_INVALID, "NESTED needs 1..32 segments"); }
    for (uint32_t k = 0; k < cfg->n_seg; ++k) {
      if ((k == 0 && cfg->seg_end[0] < 1) || (k > 0 && cfg->seg_end[k] <= cfg->seg_end[k - 1])) {
        delete h;
        return fail(SCHED_E_INVALID, "seg_end must be increasing and >= 1");
      }
      in.seg_end.push_back(cfg->seg_end[k]);
    }
    if (in.seg_end.back() < max_lp) { delete h; return fail(SCHED_E_INVALID, "last segment must reach max l'"); }
  }
  const uint32_t want_thr = cfg->policy == SCHED_WAIT ? K : cfg->policy == SCHED_NESTED ? cfg->n_seg : 0;
  if (cfg->n_thr && !is_fcfs(cfg->policy)) {
    if (cfg->n_thr != want_thr || !cfg->thresholds) { delete h; return fail(SCHED_E_INVALID, "threshold count mismatch"); }
    for (uint32_t i = 0; i < cfg->n_thr; ++i) {
      if (cfg->thresholds[i] < 1) { delete h; return fail(SCHED_E_INVALID, "thresholds must be >= 1"); }
      in.thresholds.push_back(cfg->thresholds[i]);
    }
  }
  h->tok_budget = cfg->tok_budget;
  h->max_resident_cfg = cfg->max_resident;
  h->spec_resident_cfg = cfg->spec_resident;
  if (cfg->restart_cap) h->pool_entries = cfg->restart_cap;
  h->device = cfg->device;
  // ticks
  h->d0_t = std::llround(cfg->d0_s * 1e12);
  h->d1_t = std::llround(cfg->d1_s * 1e12);
  DevParams& p = h->base;
  p.K = (int32_t)K;
  p.policy = cfg->policy;
  p.n_seg = (int32_t)in.seg_end.size();
  p.d0_t = h->d0_t;
  p.d1_t = h->d1_t;
  p.M = cfg->M;
  p.B = cfg->B;
  p.tok_budget = cfg->tok_budget;
  p.b0 = cfg->tau_b0;
  h->h_cdf_thr = std::move(thr_all);
  h->h_cdf_val = std::move(val_all);
  h->h_cdf_guide = std::move(guide_all);
  if (cfg->policy == SCHED_NESTED) {
    // stage -> segment index (bits 0-5, 63 = beyond the last segment) |
    // last stage of its segment << 6 | entry stage << 7 (reading R8)
    std::vector<uint8_t> info(in.seg_end.back() + 2, 0);
    for (uint32_t s = 0; s < info.size(); ++s) {
      uint32_t k = 0;
      while (k < in.seg_end.size() && s > in.seg_end[k]) ++k;
      const bool valid = k < in.seg_end.size();
      const bool entry = valid && k >= 1 && s == (uint32_t)in.seg_end[k - 1] + 1;
      const bool last = valid && s == (uint32_t)in.seg_end[k];
      info[s] = (uint8_t)((valid ? k : 0x3F) | (last ? 0x40 : 0) | (entry ? 0x80 : 0));
    }
    h->h_stage_info = std::move(info);
  }
  if (cfg->policy == SCHED_NESTED && K == 1 && cfg->n_seg == 1) {
    sched_config c2 = *cfg;
    c2.policy = SCHED_WAIT;
    c2.n_seg = 0;
    c2.seg_end = nullptr;
    c2.n_thr = cfg->n_thr ? 1u : 0u;
    sched_t tw = nullptr;
    if (sched_create(&tw, &c2) == SCHED_OK) h->twin = tw;  // else the Nested engines run it
  }
  *out = h;
  return SCHED_OK;
}

int sched_thresholds(sched_t h, int32_t mode, double delta, double budget_B,
                     sched_threshold_report* out) {
  if (!h || !out) return fail(SCHED_E_INVALID, "null argument");
  if (mode < 0 || mode > 1) return fail(SCHED_E_INVALID, "mode must be 0 or 1");
  std::vector<uint32_t> chosen;
  std::string err;
  int rc;
  try {
    rc = compute_thresholds(h->in, mode, delta, budget_B, out, &chosen, &err);
  } catch (const std::exception& ex) {
    return fail(SCHED_E_INVALID, ex.what());
  }
  if (rc == -2 && chosen.empty() && !is_fcfs(h->in.policy) && h->in.thresholds.empty())
    return fail(SCHED_E_UNSTABLE, err.empty() ? "rho >= 1" : err);
  if (rc == -3) return fail(SCHED_E_INFEASIBLE, err);
  if (rc == -1) return fail(SCHED_E_INVALID, err);
  if (h->in.thresholds.empty() && !chosen.empty()) {
    h->in.thresholds = chosen;
    h->prepared = false;
  }
  if (rc == -2) return fail(SCHED_E_UNSTABLE, "rho >= 1 (Prop. 1, PAPER.md:1290)");
  return SCHED_OK;
}

int sched_run(sched_t h, uint64_t seed, uint64_t rep_begin, uint32_t n_reps, double horizon_s,
              uint64_t* out_dev, void* cuda_stream) {
  if (!h || !out_dev) return fail(SCHED_E_INVALID, "null argument");
  if (n_reps == 0) return fail(SCHED_E_INVALID, "n_reps must be > 0");
  if (!(horizon_s > 0) || horizon_s > 1.4e5) return fail(SCHED_E_INVALID, "horizon must be in (0, 1.4e5] s");
  if (rep_begin + n_reps > (1ull << 32)) return fail(SCHED_E_INVALID, "replication index exceeds 2^32");
  if (h->twin && run_target(h) != h) {
    if (h->in.thresholds.empty()) return fail(SCHED_E_INVALID, "thresholds not set (sched_thresholds or config)");
    return sched_run(h->twin, seed, rep_begin, n_reps, horizon_s, out_dev, cuda_stream);
  }
  if (int rc = prepare(h)) return rc;
  CK(cudaSetDevice(h->device));
  DevParams p = h->base;
  p.seed = seed;
  p.rep_begin = rep_begin;
  p.n_reps = n_reps;
  p.T_t = std::llround(horizon_s * 1e12);
  p.trace_mode = 0;
  p.out = out_dev;
  return launch(h, p, (cudaStream_t)cuda_stream, h->use_seg ? h->sg : h->use_ring ? h->rng : h->mem);
}

int sched_run_host(sched_t h, uint64_t seed, uint64_t rep_begin, uint32_t n_reps,
                   double horizon_s, uint64_t* out_host, void* cuda_stream) {
  if (!h || !out_host) return fail(SCHED_E_INVALID, "null argument");
  const size_t bytes = (size_t)SCHED_NF * n_reps * 8;
  CK(cudaSetDevice(h->device));
  if (bytes > h->out_cap) {
    cudaFree(h->d_out);
    h->d_out = nullptr;
    CK(cudaMalloc(&h->d_out, bytes));
    h->out_cap = bytes;
  }
  if (int rc = sched_run(h, seed, rep_begin, n_reps, horizon_s, h->d_out, cuda_stream)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CK(cudaMemcpyAsync(out_host, h->d_out, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return SCHED_OK;
}

int sched_run_trace(sched_t h, const int64_t* t_ticks, const int32_t* cls, const int32_t* l,
                    const int32_t* lp, const int64_t* off, uint32_t n_reps, double horizon_s,
                    uint64_t* out_host, int64_t* log_host, int64_t log_cap, int64_t* n_logged) {
  if (!h || !off || !out_host || n_reps == 0) return fail(SCHED_E_INVALID, "bad argument");
  if (!(horizon_s > 0)) return fail(SCHED_E_INVALID, "horizon must be > 0");
  if (int rc = prepare(h)) return rc;
  const uint32_t K = (uint32_t)h->in.lambda.size();
  // regroup every replication's trace by class: slices [tr_off[r*K+c], tr_off[r*K+c+1])
  std::vector<int64_t> tt, troff;
  std::vector<uint16_t> tl, tlp;
  troff.push_back(0);
  for (uint32_t r = 0; r < n_reps; ++r) {
    for (uint32_t c = 0; c < K; ++c) {
      for (int64_t i = off[r]; i < off[r + 1]; ++i) {
        if (cls[i] < 0 || (uint32_t)cls[i] >= K) return fail(SCHED_E_INVALID, "trace class out of range");
        if ((uint32_t)cls[i] != c) continue;
        if (l[i] < 1 || lp[i] < 1 || lp[i] > 32767 || l[i] > 65535) return fail(SCHED_E_INVALID, "bad trace lengths");
        if (h->in.policy == SCHED_NESTED && lp[i] > (int32_t)h->in.seg_end.back()) return fail(SCHED_E_INVALID, "trace l' beyond the last segment");
        if ((int64_t)l[i] + lp[i] > h->in.M) return fail(SCHED_E_UNSATISFIABLE, "trace prompt with l + l' > M");
        if (!tt.empty() && troff.back() < (int64_t)tt.size() && t_ticks[i] < tt.back()) return fail(SCHED_E_INVALID, "trace not sorted by time");
        tt.push_back(t_ticks[i]);
        tl.push_back((uint16_t)l[i]);
        tlp.push_back((uint16_t)lp[i]);
      }
      troff.push_back((int64_t)tt.size());
    }
  }
  if (tt.empty()) { tt.push_back(0); tl.push_back(1); tlp.push_back(1); }
  CK(cudaSetDevice(h->device));
  int64_t *d_t = nullptr, *d_off = nullptr, *d_log = nullptr, *d_logn = nullptr;
  uint16_t *d_l = nullptr, *d_lp = nullptr;
  uint64_t* d_out = nullptr;
  const size_t out_bytes = (size_t)SCHED_NF * n_reps * 8;
  int rc = 0;
  cudaError_t e = cudaMalloc(&d_t, tt.size() * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_l, tl.size() * 2);
  if (e == cudaSuccess) e = cudaMalloc(&d_lp, tlp.size() * 2);
  if (e == cudaSuccess) e = cudaMalloc(&d_off, troff.size() * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, out_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&d_log, std::max<int64_t>(1, log_cap) * 7 * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_logn, 8);
  if (e == cudaSuccess) e = cudaMemcpy(d_t, tt.data(), tt.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_l, tl.data(), tl.size() * 2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_lp, tlp.data(), tlp.size() * 2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_off, troff.data(), troff.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(d_logn, 0, 8);
  if (e == cudaSuccess) {
    DevParams p = h->base;
    p.seed = 0;
    p.rep_begin = 0;
    p.n_reps = n_reps;
    p.T_t = std::llround(horizon_s * 1e12);
    p.trace_mode = 1;
    p.tr_t = d_t; p.tr_l = d_l; p.tr_lp = d_lp; p.tr_off = d_off;
    p.out = d_out;
    p.log = d_log;
    p.log_cap = log_host ? log_cap : 0;
    p.log_n = d_logn;
    rc = launch(h, p, 0, h->use_seg ? h->sg : h->mem);
    if (rc == 0) {
      e = cudaDeviceSynchronize();
      if (e == cudaSuccess) e = cudaMemcpy(out_host, d_out, out_bytes, cudaMemcpyDeviceToHost);
      int64_t nl = 0;
      if (e == cudaSuccess) e = cudaMemcpy(&nl, d_logn, 8, cudaMemcpyDeviceToHost);
      nl = std::min<int64_t>(nl, log_host ? log_cap : 0);
      if (e == cudaSuccess && log_host && nl > 0)
        e = cudaMemcpy(log_host, d_log, nl * 7 * 8, cudaMemcpyDeviceToHost);
      if (n_logged) *n_logged = nl;
    }
  }
  cudaFree(d_t); cudaFree(d_l); cudaFree(d_lp); cudaFree(d_off); cudaFree(d_out);
  cudaFree(d_log); cudaFree(d_logn);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "sched_run_trace");
  return SCHED_OK;
}

int sched_get_launch_info(sched_t h, sched_launch_info* out) {
  if (!h || !out) return fail(SCHED_E_INVALID, "null argument");
  if (h->twin && run_target(h) != h) return sched_get_launch_info(h->twin, out);
  if (int rc = prepare(h)) return rc;
  // the configuration sched_run uses (class-ring engine when eligible);
  // capacities in resident records (ring engine: rings + staging slots)
  const LaunchCfg& L = h->use_seg ? h->sg : h->use_ring ? h->rng : h->mem;
  uint32_t spec = L.seg ? L.seg_cap : L.Rc, safe = L.seg ? h->mem.Rc_safe : L.Rc_safe;
  for (int c = 0; L.ring && c < (int)h->in.lambda.size(); ++c) { spec += L.rcap_safe[c]; safe += L.rcap_safe[c]; }
  out->grid = L.grid;
  out->block = L.block;
  out->warps_per_block = L.wpb;
  out->shared_bytes = (int32_t)(L.wpb * L.warp_smem);
  out->blocks_per_sm = L.blocks_per_sm;
  out->sm_count = h->sm_count;
  out->max_resident = (int32_t)safe;
  out->restart_cap = (int32_t)std::min<uint64_t>(h->pool_entries, INT32_MAX);
  out->spec_resident = (int32_t)spec;
  out->fallback_grid = L.seg ? (h->mem.fallback ? h->mem.fb_grid : h->mem.grid) : L.fallback ? L.fb_grid : 0;
  out->fallback_warps_per_block = L.seg ? (h->mem.fallback ? h->mem.fb_wpb : h->mem.wpb) : L.fallback ? L.fb_wpb : 0;
  out->engine = L.seg ? 2 : L.ring ? 1 : 0;
  out->last_retries = 0;
  if (h->d_counter) {  // d_counter[2] = retry count of the last launch
    uint32_t r = 0;
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&r, h->d_counter + 2, 4, cudaMemcpyDeviceToHost));
    out->last_retries = (int32_t)r;
  }
  return SCHED_OK;
}

int sched_aggregate(const uint64_t* rows_dev, uint64_t ld, uint32_t n_reps, double horizon_s,
                    int64_t* out_int_dev, double* out_f64_dev, void* cuda_stream) {
  if (!rows_dev || !out_int_dev || !out_f64_dev) return fail(SCHED_E_INVALID, "null argument");
  if (n_reps == 0) return fail(SCHED_E_INVALID, "n_reps must be > 0");
  if (ld < n_reps) return fail(SCHED_E_INVALID, "row stride ld must be >= n_reps");
  if (!(horizon_s > 0)) return fail(SCHED_E_INVALID, "horizon must be > 0");
  CK(launch_aggregate(rows_dev, ld, n_reps, horizon_s, out_int_dev, out_f64_dev, (cudaStream_t)cuda_stream));
  return SCHED_OK;
}

int sched_get_status(sched_t h, uint32_t* mask) {
  if (!h || !mask) return fail(SCHED_E_INVALID, "null argument");
  *mask = 0;
  if (h->twin) {  // runs of the WAIT twin and trace runs of h itself
    uint32_t m = 0;
    if (int rc = sched_get_status(h->twin, &m)) return rc;
    *mask = m;
  }
  if (!h->d_status) return SCHED_OK;  // never launched
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(mask, h->d_status, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemset(h->d_status, 0, 4));
  return SCHED_OK;
}

int sched_restart_pool_stats(sched_t h, uint64_t* capacity_entries, uint64_t* high_water_entries) {
  if (!h || !capacity_entries || !high_water_entries) return fail(SCHED_E_INVALID, "null argument");
  if (h->twin && run_target(h) != h) return sched_restart_pool_stats(h->twin, capacity_entries, high_water_entries);
  *capacity_entries = (uint64_t)h->pool_chunks * kRestartChunk;
  *high_water_entries = 0;
  if (!h->d_pool_free) return SCHED_OK;  // never launched
  CK(cudaSetDevice(h->device));
  uint32_t bump = 0;
  CK(cudaMemcpy(&bump, h->d_pool_free + 1, 4, cudaMemcpyDeviceToHost));
  *high_water_entries = (uint64_t)std::min(bump, h->pool_chunks) * kRestartChunk;
  return SCHED_OK;
}

static int walk_params(int32_t kind, int64_t n, double mu, int64_t n_prev, double p, uint64_t seed,
                       uint64_t walk_begin, uint32_t n_walks, uint32_t B, WalkParams* w) {
  if (kind != 0 && kind != 1) return fail(SCHED_E_INVALID, "walk kind must be 0 or 1");
  if (n < 1 || n_walks == 0 || B == 0) return fail(SCHED_E_INVALID, "need n >= 1, n_walks > 0, B > 0");
  if (walk_begin + n_walks > (1ull << 32)) return fail(SCHED_E_INVALID, "walk index exceeds 2^32");
  if (kind == 0 && !(mu > 0 && mu <= 1e4)) return fail(SCHED_E_INVALID, "need 0 < mu <= 1e4");
  if (kind == 1 && (n_prev < 1 || !(p > 0 && p < 1))) return fail(SCHED_E_INVALID, "need n_prev >= 1, 0 < p < 1");
  *w = WalkParams{};
  w->kind = kind; w->n = n; w->seed = seed; w->walk_begin = walk_begin; w->n_walks = n_walks; w->B = B;
  if (kind == 0) {
    w->mu = mu;
    w->p0 = std::exp(-mu);
    w->kmax = (int64_t)(mu + 40.0 * std::sqrt(mu) + 100.0);
  } else {
    w->n_prev = n_prev;
    w->p0 = std::pow(1.0 - p, (double)n_prev);
    w->ratio = p / (1.0 - p);
  }
  return 0;
}

int sched_walks(int32_t kind, int64_t n, double mu, int64_t n_prev, double p, uint64_t seed,
                uint64_t walk_begin, uint32_t n_walks, uint32_t B, int64_t* out_dev, void* cuda_stream) {
  if (!out_dev) return fail(SCHED_E_INVALID, "null output");
  WalkParams w;
  if (int rc = walk_params(kind, n, mu, n_prev, p, seed, walk_begin, n_walks, B, &w)) return rc;
  w.out = out_dev;
  CK(launch_walks(w, (cudaStream_t)cuda_stream));
  return SCHED_OK;
}

int sched_walks_host(int32_t kind, int64_t n, double mu, int64_t n_prev, double p, uint64_t seed,
                     uint64_t walk_begin, uint32_t n_walks, uint32_t B, int64_t* out_host, int32_t device) {
  if (!out_host) return fail(SCHED_E_INVALID, "null output");
  WalkParams w;
  if (int rc = walk_params(kind, n, mu, n_prev, p, seed, walk_begin, n_walks, B, &w)) return rc;
  CK(cudaSetDevice(device));
  const size_t bytes = (size_t)kWalkFields * n_walks * 8;
  int64_t* d = nullptr;
  CK(cudaMalloc(&d, bytes));
  w.out = d;
  cudaError_t e = launch_walks(w, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out_host, d, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "sched_walks_host");
  return SCHED_OK;
}

void sched_destroy(sched_t h) {
  if (!h) return;
  sched_destroy(h->twin);
  cudaFree(h->d_cdf_thr);
  cudaFree(h->d_cdf_val);
  cudaFree(h->d_cdf_guide);
  cudaFree(h->d_stage_info);
  cudaFree(h->d_pool_a);
  cudaFree(h->d_seg_a);
  cudaFree(h->d_ring_g);
  cudaFree(h->d_ring_log);
  cudaFree(h->d_pool_stash);
  cudaFree(h->d_pool_e);
  cudaFree(h->d_pool_llp);
  cudaFree(h->d_pool_next);
  cudaFree(h->d_pool_free);
  cudaFree(h->d_counter);
  cudaFree(h->d_status);
  cudaFree(h->d_out);
  cudaFree(h->d_retry);
  cudaFree(h->d_rf_B);
  cudaFree(h->d_rf_Lam);
  cudaFree(h->d_rf_scale);
  delete h;
}

}  // extern "C"
