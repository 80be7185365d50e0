// des_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The oracle: a plain, slow, sequential CPU discrete-event simulator of the
// schedulers of arXiv 2504.11320 ("Optimizing LLM Inference: Fluid-Guided
// Online Scheduling with Memory Constraints").  It is what the CUDA path is
// checked against, element by element.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / `--impl reference` legs may load it; the
// product path (paper_2504_11320_b200/) never does and shares no code with
// it (own Philox, own logarithm, own CDF sampling, own state layout).
//
// Every step below follows the paper (PAPER.md line numbers are into
// /root/reference/PAPER.md, the authoritative version at lines 984-2609) in
// the reading fixed by DESIGN.md §4 (which restates SURVEY.md §8c):
//   * model, stages, KV footprint l+s      PAPER.md:1142-1154 (§Model)
//   * iteration time tau = d0 + d1*tokens  PAPER.md:1180-1183 (Eq. time_consump)
//   * memory constraint incl. paused KV    PAPER.md:1202-1207 (Eq. memory_constraint)
//   * LIFO eviction, restart at stage 0
//   * waiting prompts hold no GPU KV       PAPER.md:2288 (Remark), Example 1 at 1213
//   * metrics (throughput at completion,
//     latency, TTFT)
//   * WAIT (Algorithm 1)
//   * Nested WAIT (Algorithm 2)
//   * FCFS / vLLM-style baseline
// Data structures are the obvious ones (std::deque FIFOs of waiting prompts,
// a std::vector of GPU-resident prompts in admission order); nothing is
// blocked, fused or reordered.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (no fast-math):
// the exponential sampler must use only correctly-rounded IEEE operations.

#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

namespace {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- Philox
// Philox4x32-10 as defined by Salmon, Moraes, Dror, Shaw (SC'11) / Random123.
const uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
const uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

void philox(const uint32_t in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// --------------------------------------------------------- -ln(U) sampler
// DESIGN.md §4.2 (= SURVEY.md §8c.2.4): U = (2*u52+1) * 2^-53, ln U by the
// fdlibm-style reduction ln U = n*ln2 + ln f, ln f = 2*atanh(s),
// s = (f-1)/(f+1), atanh series to s^19.  Each line is one rounded IEEE op.
double exp_from_bits(uint32_t x0, uint32_t x1) {
  const uint64_t u52 = ((uint64_t)x0 << 20) | (uint64_t)(x1 >> 12);
  const uint64_t v = 2 * u52 + 1;                 // odd, < 2^53
  int e = 63 - __builtin_clzll(v);                // v in [2^e, 2^(e+1))
  double f = std::ldexp((double)v, -e);           // [1, 2), exact
  const double SQRT2 = 1.4142135623730951454746;  // 0x1.6a09e667f3bcdp+0
  if (f > SQRT2) { f = f * 0.5; e = e + 1; }
  double s = (f - 1.0) / (f + 1.0);
  double z = s * s;
  // C(2i+1) = correctly rounded 1/(2i+1)
  double P = 1.0 / 19.0;
  P = P * z + 1.0 / 17.0;
  P = P * z + 1.0 / 15.0;
  P = P * z + 1.0 / 13.0;
  P = P * z + 1.0 / 11.0;
  P = P * z + 1.0 / 9.0;
  P = P * z + 1.0 / 7.0;
  P = P * z + 1.0 / 5.0;
  P = P * z + 1.0 / 3.0;
  P = P * z + 1.0;
  double lnf = (s + s) * P;
  const int n = e - 53;
  double ln2_hi, ln2_lo;
  const uint64_t HI = 0x3fe62e42fee00000ull, LO = 0x3dea39ef35793c76ull;
  std::memcpy(&ln2_hi, &HI, 8);
  std::memcpy(&ln2_lo, &LO, 8);
  double dn = (double)n;
  double lnU = dn * ln2_hi + (dn * ln2_lo + lnf);
  return -lnU;
}

// ------------------------------------------------------ length CDF tables
// thr_i = floor(cum_i * 2^32 / W) in 128-bit arithmetic, last
// entry forced to 2^32; idx(x) = min{ i : x < thr_i }.
struct LenTable {
  std::vector<uint16_t> val;
  std::vector<uint64_t> thr;   // up to 2^32 inclusive
  void build(const uint16_t* v, const uint64_t* w, int n) {
    val.assign(v, v + n);
    thr.resize(n);
    u128 W = 0;
    for (int i = 0; i < n; ++i) W += w[i];
    u128 cum = 0;
    for (int i = 0; i < n; ++i) {
      cum += w[i];
      thr[i] = (uint64_t)((cum << 32) / W);
    }
    thr[n - 1] = (uint64_t)1 << 32;
  }
  int sample(uint32_t x) const {
    for (size_t i = 0; i < thr.size(); ++i)
      if ((uint64_t)x < thr[i]) return val[i];
    return val.back();  // unreachable: last threshold is 2^32
  }
};

// ------------------------------------------------------------ the model
struct Prompt {            // a prompt waiting in a FIFO or resident on the GPU
  int c;                   // class j (read by WAIT only)
  int64_t a;               // original arrival tick (latency/TTFT origin)
  int l, lp;               // prefill length l_j, decode length l'_j
  bool first_tok;          // first output token already emitted
  int s;                   // resident: next stage to run (1..lp); waiting: 0
};

uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27; z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// Piecewise-constant rate function of one class, generated by time change
// (DESIGN.md §4.8): operational time tau counts expected arrivals in units
// of 2^-32; arrival k sits at tau_k = sum of (int64)(E_i * 2^32); its tick
// is the inverse of the integrated rate Lambda(t), piece by piece.
struct RatePieces {
  std::vector<int64_t> B;      // piece start ticks
  std::vector<int64_t> Lam;    // integrated rate at piece starts (operational ticks)
  std::vector<double> lam;     // rate of each piece
  bool empty() const { return B.empty(); }
  void build(const double* t, const double* r, int n) {
    for (int p = 0; p < n; ++p) { B.push_back(std::llround(t[p] * 1e12)); lam.push_back(r[p]); }
    Lam.push_back(0);
    for (int p = 0; p + 1 < n; ++p)
      Lam.push_back(Lam[p] + (int64_t)(((lam[p] * (double)(B[p + 1] - B[p])) * 4294967296.0) / 1e12));
  }
  // arrival tick at operational time tau (INT64_MAX: no more arrivals)
  int64_t tick(int64_t tau) const {
    int p = 0;
    for (int q = 1; q < (int)B.size(); ++q)
      if (Lam[q] <= tau) p = q;
    if (lam[p] == 0.0) return INT64_MAX;  // only the last piece can be reached with rate 0
    const double scale = 1e12 / (lam[p] * 4294967296.0);
    int64_t t = B[p] + (int64_t)((double)(tau - Lam[p]) * scale);
    if (p + 1 < (int)B.size()) t = std::min(t, B[p + 1] - 1);
    return t;
  }
};

struct Setup {  // per-config constants, recomputed here from the raw config
  int K, policy;
  std::vector<RatePieces> rf;      // time-varying classes (empty = homogeneous)
  std::vector<double> gap_scale;   // 1e12 / lambda_c, ticks per unit exponential
  std::vector<LenTable> ltab, lptab;
  int64_t d0_t, d1_t, T_t, M, b0 = 0;
  std::vector<uint32_t> thr;
  std::vector<int> seg_end;
  uint32_t B, tok_budget;
  int max_stage = 0;               // largest decode length any table or trace can hold
  explicit Setup(const orc_config* cfg) {
    K = cfg->K; policy = cfg->policy;
    for (int c = 0; c < K; ++c) {
      gap_scale.push_back(cfg->lam[c] > 0 ? 1e12 / cfg->lam[c] : 0.0);
      LenTable a, b;
      a.build(cfg->l_val + cfg->l_off[c], cfg->l_w + cfg->l_off[c], cfg->l_off[c + 1] - cfg->l_off[c]);
      b.build(cfg->lp_val + cfg->lp_off[c], cfg->lp_w + cfg->lp_off[c], cfg->lp_off[c + 1] - cfg->lp_off[c]);
      ltab.push_back(a); lptab.push_back(b);
      for (uint16_t v : b.val) max_stage = std::max<int>(max_stage, v);
      RatePieces pc;
      if (cfg->rf_off && cfg->rf_off[c + 1] > cfg->rf_off[c])
        pc.build(cfg->rf_t + cfg->rf_off[c], cfg->rf_rate + cfg->rf_off[c], cfg->rf_off[c + 1] - cfg->rf_off[c]);
      rf.push_back(pc);
    }
    // 1 tick = 1 ps
    d0_t = std::llround(cfg->d0_s * 1e12);
    d1_t = std::llround(cfg->d1_s * 1e12);
    b0 = cfg->tau_b0;
    T_t = std::llround(cfg->horizon_s * 1e12);
    M = cfg->M;
    thr.assign(cfg->thr, cfg->thr + cfg->n_thr);
    for (int k = 0; k < cfg->n_seg; ++k) seg_end.push_back(cfg->seg_end[k]);
    B = cfg->B; tok_budget = cfg->tok_budget;
  }
};

// Poisson arrival stream of class c, replication r (type j
// arrives as a Poisson process with rate lambda_j).  Arrival k uses Philox
// counter (k, r, c, 0) and key (seed lo, seed hi) -- DESIGN.md §4.2.
struct ArrivalStream {
  const Setup* S; uint64_t seed; uint32_t r; int c;
  uint32_t k = 0; int64_t t = 0;  // next arrival: index k, tick t
  int64_t tau = 0, tau_prev = 0;  // operational time (time-varying classes)
  int l = 0, lp = 0;
  bool exhausted = false;         // lambda = 0
  // explicit-trace mode
  const int64_t* tr_t = nullptr; const int32_t* tr_l = nullptr; const int32_t* tr_lp = nullptr;
  std::vector<int64_t> tr_idx; size_t tr_pos = 0;
  int64_t t_prev = 0;

  void draw() {  // fill (t, l, lp) of arrival k
    if (tr_t) {
      if (tr_pos >= tr_idx.size()) { exhausted = true; return; }
      int64_t i = tr_idx[tr_pos];
      t = tr_t[i]; l = tr_l[i]; lp = tr_lp[i];
      return;
    }
    const bool tv = !S->rf[c].empty();
    if (!tv && S->gap_scale[c] == 0.0) { exhausted = true; return; }
    uint32_t ctr[4] = {k, r, (uint32_t)c, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    philox(ctr, key, x);
    double E = exp_from_bits(x[0], x[1]);
    if (tv) {
      // time change: tau_k = tau_{k-1} + (int64)(E * 2^32), t_k = Lambda^{-1}(tau_k)
      tau = tau_prev + (int64_t)(E * 4294967296.0);
      t = S->rf[c].tick(tau);
      if (t == INT64_MAX) { exhausted = true; return; }
    } else {
      int64_t gap = (int64_t)(E * S->gap_scale[c]);  // truncation toward zero
      t = t_prev + gap;
    }
    l = S->ltab[c].sample(x[2]);
    lp = S->lptab[c].sample(x[3]);
  }
  void advance() { t_prev = t; tau_prev = tau; ++k; ++tr_pos; draw(); }
};

struct Plan {
  std::vector<char> res_in;       // per resident: batched this iteration
  std::vector<int> new_fifo;      // FIFO index each new admission comes from
  std::vector<int> new_pos;       // position within that FIFO (front = 0)
};

struct Sim {
  const Setup& S;
  uint64_t seed; uint32_t r;
  std::vector<ArrivalStream> streams;
  std::vector<std::deque<Prompt>> fifo;   // WAIT: one per class; else one
  std::vector<Prompt> res;                // GPU-resident, admission order
  // per (row, stage) prompt counters of the decision step, row = class
  // (WAIT) or 0 (NESTED: the stage fixes the segment); zeroed after use
  std::vector<uint64_t> qcnt;
  size_t qw = 0;
  int64_t now = 0, KV = 0;                // KV = sum over residents of (l+s-1)
  // metrics
  uint64_t arrivals = 0, admitted = 0, completed = 0, completed_after_T = 0,
           completed_tokens = 0, first_tokens = 0, batches = 0, request_steps = 0,
           prefill_steps = 0, evictions = 0, cbi = 0, sum_waiting = 0;
  int64_t busy = 0, idle = 0, max_kv = 0;
  u128 sum_lat = 0, sum_ttft = 0, sum_arr_all = 0, sum_arr_done = 0;
  uint64_t h;
  int status = 0;
  int64_t* log = nullptr; int64_t log_cap = 0, log_n = 0;

  Sim(const Setup& s, uint64_t seed_, uint32_t r_) : S(s), seed(seed_), r(r_) {
    fifo.resize(S.policy == ORC_WAIT ? S.K : 1);
    qw = (size_t)std::max(S.max_stage, S.seg_end.empty() ? 0 : S.seg_end.back()) + 2;
    qcnt.assign((S.policy == ORC_WAIT ? S.K : 1) * qw, 0);
    h = mix64(seed ^ ((uint64_t)r * 0x9E3779B97F4A7C15ull));
  }
  int fifo_of(int c) const { return S.policy == ORC_WAIT ? c : 0; }

  // INGEST (DESIGN.md §4.4 step 1): every arrival with t <= now and t < T
  // joins its FIFO, in (t, class, k) order across classes.
  void ingest() {
    for (;;) {
      int best = -1;
      for (int c = 0; c < S.K; ++c) {
        const ArrivalStream& st = streams[c];
        if (st.exhausted || st.t > now || st.t >= S.T_t) continue;
        if (best < 0 || st.t < streams[best].t) best = c;  // ties: lower class
      }
      if (best < 0) return;
      ArrivalStream& st = streams[best];
      fifo[fifo_of(best)].push_back(Prompt{best, st.t, st.l, st.lp, false, 0});
      ++arrivals;
      sum_arr_all += (u128)st.t;
      st.advance();
    }
  }

  bool next_arrival(int64_t* t) const {
    bool any = false;
    for (int c = 0; c < S.K; ++c) {
      const ArrivalStream& st = streams[c];
      if (st.exhausted || st.t >= S.T_t) continue;
      if (!any || st.t < *t) { *t = st.t; any = true; }
    }
    return any;
  }

  // segment index (0-based) of stage s under Nested WAIT: segment k covers
  // stages e_{k-1}+1 .. e_k, segment 0 covers 0..e_0 (reading R8).
  int segment_of(int s) const {
    for (size_t k = 0; k < S.seg_end.size(); ++k)
      if (s <= S.seg_end[k]) return (int)k;
    return (int)S.seg_end.size();  // beyond the last segment (invalid config)
  }

  // Invariant P14 (follows by induction from Alg. 1
  // / Alg. 2 "Advance min{n_k, Q_{k,s}}"): WAIT stage counts Q_{j,s} <= n_j
  // for s >= 1; Nested non-entry stages Q_{k,s} <= n_k.  Checked at every
  // decision epoch; a violation marks the row with status 3 (never set by
  // a correct simulator: the tests require status 0).
  uint64_t& q_at(const Prompt& p) { return qcnt[(S.policy == ORC_WAIT ? p.c : 0) * qw + p.s]; }
  void clear_q() { for (const Prompt& p : res) q_at(p) = 0; }
  //
  // Nested also checks the ordering property the CUDA segment engine relies
  // on (derived from the same two rules: every non-entry
  // stage of an active segment advances, an entry stage takes its oldest
  // n_k first): residents in admission order have
  // non-increasing stages.  A violation is status 3 as well.
  void check_p14() {
    int prev_s = INT32_MAX;
    for (const Prompt& p : res) {
      if (S.policy == ORC_WAIT) {
        if (++q_at(p) > S.thr[p.c]) status = 3;
      } else if (S.policy == ORC_NESTED) {
        const int k = segment_of(p.s);
        const bool entry = k >= 1 && p.s == S.seg_end[k - 1] + 1;
        if (!entry && ++q_at(p) > S.thr[k]) status = 3;
        if (p.s > prev_s) status = 3;
        prev_s = p.s;
      }
    }
    clear_q();
  }

  // DECIDE.  Returns false for "no batch: wait".
  bool decide(Plan& P) {
    P.res_in.assign(res.size(), 0);
    P.new_fifo.clear(); P.new_pos.clear();
    if (S.policy == ORC_WAIT) {
      check_p14();
      // Algorithm 1 line "Check if n_j0 >= n_j": Q = classes
      // whose waiting inventory reached the threshold.
      std::vector<char> inQ(S.K, 0);
      bool any = false;
      for (int c = 0; c < S.K; ++c)
        if (fifo[c].size() >= S.thr[c]) { inQ[c] = 1; any = true; }
      if (!any) return false;
      // "selecting min{n_j, n_js} prompts of type j at each
      // stage s for all j meeting the condition" -- the oldest (admission
      // order) first at every stage s >= 1 (reading R6) ...
      for (size_t i = 0; i < res.size(); ++i) {
        const Prompt& p = res[i];
        if (!inQ[p.c]) continue;  // line 1491: other types wait, KV kept
        uint64_t& taken = q_at(p);  // selected so far at (type, stage)
        if (taken < S.thr[p.c]) { P.res_in[i] = 1; ++taken; }
      }
      clear_q();
      // ... and at stage 0 the first n_j waiting prompts, class-major (R28)
      for (int c = 0; c < S.K; ++c)
        if (inQ[c])
          for (uint32_t j = 0; j < S.thr[c]; ++j) { P.new_fifo.push_back(c); P.new_pos.push_back((int)j); }
      return true;
    }
    if (S.policy == ORC_NESTED) {
      check_p14();
      // Algorithm 2 line "Find largest k such that Q_{k', entry} >= n_k' for
      // all k' <= k".  Segment 1's entry stage is stage 0
      // (the FIFO); segment k>=2 enters at stage e_{k-1}+1 (reading R8).
      const int L = (int)S.seg_end.size();
      if (fifo[0].size() < S.thr[0]) return false;
      int kstar = 0;  // 0-based index of the last active segment
      for (int k = 1; k < L; ++k) {
        const int entry = S.seg_end[k - 1] + 1;
        uint64_t cnt = 0;
        for (const Prompt& p : res) cnt += (p.s == entry);
        if (cnt >= S.thr[k]) kstar = k; else break;
      }
      // "Form batch from segments 1, ..., k: select
      // min{n_k', Q_{k',s}} prompts per stage", the oldest (admission order)
      // first at every stage (reading R6); prompts of later segments wait
      // with their KV (line 1643).
      for (size_t i = 0; i < res.size(); ++i) {
        const int k = segment_of(res[i].s);
        if (k > kstar) continue;
        uint64_t& taken = q_at(res[i]);  // selected so far at this stage
        if (taken < S.thr[k]) { P.res_in[i] = 1; ++taken; }
      }
      clear_q();
      // stage 0 of segment 1: the first n_1 prompts of the FIFO
      for (uint32_t j = 0; j < S.thr[0]; ++j) { P.new_fifo.push_back(0); P.new_pos.push_back((int)j); }
      return true;
    }
    // FCFS, vLLM-style "new arrivals first" (DESIGN.md
    // reading R15): every resident decodes, then admit the FIFO head in
    // order while the batch-size limit, the current-KV check and the prefill
    // token budget all hold; stop at the first candidate that fails.
    // Sarathi-style "ongoing first" (reading R29) differs in
    // one term: the KV check also reserves the residents' growth of one
    // token each, so only what fits after the ongoing prompts is admitted.
    for (size_t i = 0; i < res.size(); ++i) P.res_in[i] = 1;
    const int64_t reserve = S.policy == ORC_FCFS_ONGOING ? (int64_t)res.size() : 0;
    int64_t new_l = 0;
    uint64_t n_new = 0;
    for (size_t j = 0; j < fifo[0].size(); ++j) {
      const Prompt& p = fifo[0][j];
      if ((uint64_t)res.size() + n_new >= S.B) break;
      if (KV + reserve + new_l + p.l > S.M) break;
      if (S.tok_budget != 0 && (uint64_t)(new_l + p.l) > S.tok_budget) break;
      new_l += p.l; ++n_new;
      P.new_fifo.push_back(0); P.new_pos.push_back((int)j);
    }
    if (res.empty() && n_new == 0) return false;
    return true;
  }

  void hash_batch(int64_t t_start, uint64_t plan_size, int64_t tokens,
                  uint64_t n_complete, uint64_t n_evict, uint64_t n_new) {
    h = mix64(h ^ (uint64_t)t_start);
    h = mix64(h ^ (plan_size | ((uint64_t)tokens << 32)));
    h = mix64(h ^ (n_complete | (n_evict << 20) | (n_new << 40)));
  }

  void run() {
    for (;;) {
      ingest();                                   // step 1
      if (now >= S.T_t) break;                    // step 2
      Plan P;
      bool go = decide(P);                        // step 3
      uint64_t n_evict = 0;
      int64_t peak = 0;
      // waiting inventory the decision reads (n_j0 of Alg. 1 line 1488 /
      // Q_{1,0} of Alg. 2): after ingest, before admission and
      // before this epoch's evictions (reading R32; summed over executed
      // batches, it is the pre-service queue of the Kingman bounds, P17)
      uint64_t waiting = 0;
      for (auto& q : fifo) waiting += q.size();
      if (go) {
        // step 4, MEMORY: the KV held after this iteration must fit in M
        // (Eq. memory_constraint; paused prompts keep their
        // KV, waiting prompts hold none).  Post-iteration size of a batched
        // resident is l+s, of a paused one l+s-1, of a new admission l.
        peak = KV;
        for (size_t i = 0; i < res.size(); ++i) peak += P.res_in[i];
        for (size_t j = 0; j < P.new_fifo.size(); ++j)
          peak += fifo[P.new_fifo[j]][P.new_pos[j]].l;
        // LIFO eviction: the most recently admitted
        // resident loses its KV and re-enters its FIFO at stage 0.
        while (peak > S.M && !res.empty()) {
          Prompt v = res.back();
          const int in_plan = P.res_in.back();
          res.pop_back(); P.res_in.pop_back();
          peak -= (v.l + v.s - 1) + in_plan;
          KV -= v.l + v.s - 1;
          v.s = 0;
          fifo[fifo_of(v.c)].push_back(v);
          ++evictions; ++n_evict;
        }
        // still infeasible: drop the most recent new admissions (they stay
        // in their FIFO, in place).
        while (peak > S.M && !P.new_fifo.empty()) {
          peak -= fifo[P.new_fifo.back()][P.new_pos.back()].l;
          P.new_fifo.pop_back(); P.new_pos.pop_back();
        }
        uint64_t n_res_plan = 0;
        for (char x : P.res_in) n_res_plan += x;
        if (n_res_plan + P.new_fifo.size() == 0) go = false;  // empty batch = wait
        else if (peak > max_kv) max_kv = peak;
      }
      if (!go) {
        int64_t t;
        if (!next_arrival(&t)) break;
        idle += t - now;
        now = t;
        continue;
      }
      // step 5, EXECUTE.  tau = d0 + d1 * (sum_prefill l + sum_decode (l+s))
      // (Eq. time_consump).
      sum_waiting += waiting;
      int64_t tokens = 0;
      uint64_t n_res_plan = 0;
      for (size_t i = 0; i < res.size(); ++i)
        if (P.res_in[i]) { tokens += res[i].l + res[i].s; ++n_res_plan; }
      std::vector<Prompt> fresh;
      {
        // pop the admitted prompts from their FIFO fronts, in plan order
        // (each FIFO contributes a contiguous prefix)
        std::vector<uint64_t> popped(fifo.size(), 0);
        for (size_t j = 0; j < P.new_fifo.size(); ++j) {
          fresh.push_back(fifo[P.new_fifo[j]][P.new_pos[j]]);
          ++popped[P.new_fifo[j]];
        }
        for (size_t q = 0; q < fifo.size(); ++q)
          for (uint64_t x = 0; x < popped[q]; ++x) fifo[q].pop_front();
      }
      for (const Prompt& p : fresh) tokens += p.l;
      // ... piecewise linear beyond b0 tokens (b0 = 0: Eq. time_consump)
      const int64_t tau = S.d0_t + S.d1_t * std::max<int64_t>(0, tokens - S.b0);
      const int64_t t_end = now + tau;
      uint64_t n_complete = 0;
      std::vector<Prompt> kept;
      kept.reserve(res.size() + fresh.size());
      for (size_t i = 0; i < res.size(); ++i) {
        Prompt p = res[i];
        if (P.res_in[i]) {
          // TTFT: the first output token is produced by the stage-1
          // iteration.
          if (p.s == 1 && !p.first_tok) {
            p.first_tok = true;
            if (t_end <= S.T_t) { sum_ttft += (u128)(t_end - p.a); ++first_tokens; }
          }
          if (p.s == p.lp) {
            // the stage-l' iteration completes the prompt; its KV is cleared
            // (PAPER.md:1284, 1486); throughput is credited at completion
            // (PAPER.md:1239).
            KV -= p.l + p.lp - 1;
            ++n_complete;
            if (t_end <= S.T_t) {
              ++completed; completed_tokens += (uint64_t)p.lp;
              sum_lat += (u128)(t_end - p.a); sum_arr_done += (u128)p.a;
              cbi += batches;
            } else {
              ++completed_after_T;
            }
            continue;
          }
          p.s += 1;
          KV += 1;
        }
        kept.push_back(p);
      }
      for (Prompt p : fresh) {  // prefill: stage 0 -> next stage 1, KV l
        p.s = 1;
        KV += p.l;
        ++admitted;
        kept.push_back(p);
      }
      res.swap(kept);
      const uint64_t plan_size = n_res_plan + fresh.size();
      if (log && log_n < log_cap) {
        int64_t* e = log + 7 * log_n;
        e[0] = now; e[1] = (int64_t)plan_size; e[2] = tokens; e[3] = (int64_t)n_complete;
        e[4] = (int64_t)n_evict; e[5] = (int64_t)fresh.size(); e[6] = peak;
        ++log_n;
      }
      hash_batch(now, plan_size, tokens, n_complete, n_evict, fresh.size());
      request_steps += plan_size;
      prefill_steps += fresh.size();
      busy += tau;
      ++batches;
      now = t_end;
    }
  }
  void write(uint64_t* out, int64_t n_reps, int64_t i) const {
    auto put = [&](int f, uint64_t v) { out[(int64_t)f * n_reps + i] = v; };
    uint64_t waiting = 0;
    for (auto& q : fifo) waiting += q.size();
    // sojourn truncated at T: completed-by-T prompts contribute c-a, all
    // other arrivals T-a (Little's-law check)
    u128 soj = sum_lat + (u128)(arrivals - completed) * (u128)S.T_t - (sum_arr_all - sum_arr_done);
    put(ORC_F_ARRIVALS, arrivals); put(ORC_F_ADMITTED, admitted);
    put(ORC_F_COMPLETED, completed); put(ORC_F_COMPLETED_AFTER_T, completed_after_T);
    put(ORC_F_COMPLETED_TOKENS, completed_tokens); put(ORC_F_FIRST_TOKENS, first_tokens);
    put(ORC_F_BATCHES, batches); put(ORC_F_REQUEST_STEPS, request_steps);
    put(ORC_F_PREFILL_STEPS, prefill_steps); put(ORC_F_EVICTIONS, evictions);
    put(ORC_F_BUSY_TICKS, (uint64_t)busy); put(ORC_F_IDLE_TICKS, (uint64_t)idle);
    put(ORC_F_LAT_LO, (uint64_t)sum_lat); put(ORC_F_LAT_HI, (uint64_t)(sum_lat >> 64));
    put(ORC_F_TTFT_LO, (uint64_t)sum_ttft); put(ORC_F_TTFT_HI, (uint64_t)(sum_ttft >> 64));
    put(ORC_F_SOJ_LO, (uint64_t)soj); put(ORC_F_SOJ_HI, (uint64_t)(soj >> 64));
    put(ORC_F_COMPLETION_BATCH_IDX, cbi); put(ORC_F_MAX_KV_PEAK, (uint64_t)max_kv);
    put(ORC_F_FINAL_WAITING, waiting); put(ORC_F_FINAL_RESIDENT, res.size());
    put(ORC_F_TRAJ_HASH, h); put(ORC_F_STATUS, (uint64_t)(int64_t)status);
    put(ORC_F_NOW_STOP, (uint64_t)now); put(ORC_F_SUM_WAITING, sum_waiting);
  }
};

}  // namespace

extern "C" {

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox(ctr, key, out);
}

double orc_exp_from_bits(uint32_t x0, uint32_t x1) { return exp_from_bits(x0, x1); }

int orc_gen_arrivals(const orc_config* cfg, uint64_t seed, uint32_t r, int32_t c,
                     int64_t n, int64_t* t, int32_t* l, int32_t* lp) {
  Setup S(cfg);
  ArrivalStream st;
  st.S = &S; st.seed = seed; st.r = r; st.c = c;
  st.draw();
  for (int64_t i = 0; i < n; ++i) {
    if (st.exhausted) return -1;
    t[i] = st.t; l[i] = st.l; lp[i] = st.lp;
    st.advance();
  }
  return 0;
}

static void run_one(const Setup& S, uint64_t seed, uint32_t r, uint64_t* out,
                    int64_t n_reps, int64_t i) {
  Sim sim(S, seed, r);
  sim.streams.resize(S.K);
  for (int c = 0; c < S.K; ++c) {
    ArrivalStream& st = sim.streams[c];
    st.S = &S; st.seed = seed; st.r = r; st.c = c;
    st.draw();
  }
  sim.run();
  sim.write(out, n_reps, i);
}

int orc_run(const orc_config* cfg, uint64_t seed, uint64_t rep_begin, int64_t n_reps,
            uint64_t* out, int32_t n_threads) {
  Setup S(cfg);
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < n_threads; ++w)
    th.emplace_back([&, w] {
      for (int64_t i = w; i < n_reps; i += n_threads)
        run_one(S, seed, (uint32_t)(rep_begin + (uint64_t)i), out, n_reps, i);
    });
  for (auto& x : th) x.join();
  return 0;
}

int64_t orc_run_trace(const orc_config* cfg, const int64_t* t, const int32_t* cls,
                      const int32_t* l, const int32_t* lp, const int64_t* off,
                      int64_t n_reps, uint64_t* out, int64_t* log, int64_t log_cap) {
  Setup S(cfg);
  for (int64_t a = 0; a < off[n_reps]; ++a) S.max_stage = std::max<int>(S.max_stage, lp[a]);
  int64_t logged = 0;
  for (int64_t i = 0; i < n_reps; ++i) {
    Sim sim(S, 0, (uint32_t)i);
    sim.streams.resize(S.K);
    for (int c = 0; c < S.K; ++c) {
      ArrivalStream& st = sim.streams[c];
      st.S = &S; st.c = c; st.tr_t = t; st.tr_l = l; st.tr_lp = lp;
      for (int64_t a = off[i]; a < off[i + 1]; ++a)
        if (cls[a] == c) st.tr_idx.push_back(a);
      st.draw();
    }
    if (i == 0) { sim.log = log; sim.log_cap = log_cap; }
    sim.run();
    if (i == 0) logged = sim.log_n;
    sim.write(out, n_reps, i);
  }
  return logged;
}

}  // extern "C"
