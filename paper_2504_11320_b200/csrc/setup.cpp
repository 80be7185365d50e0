// setup.cpp -- host-side setup of libsched (sched_thresholds): the fluid
// equilibrium, integer thresholds, theta_k and the Thm-2 memory budget of
// arXiv 2504.11320.  Integer decisions use exact rational arithmetic on
// arbitrary-precision integers (every double input converts exactly), so
// boundary cases such as 7 * (12/14) = 6 in C3a cannot be flipped by
// rounding; reported reals are plain doubles.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "setup.h"

namespace waitsim {
namespace {

// ---------------------------------------------------- unsigned big integer
struct Big {
  std::vector<uint32_t> d;  // little-endian limbs, no leading zero limbs
  Big() {}
  explicit Big(uint64_t v) {
    while (v) { d.push_back((uint32_t)v); v >>= 32; }
  }
  bool zero() const { return d.empty(); }
  void trim() { while (!d.empty() && d.back() == 0) d.pop_back(); }
  static int cmp(const Big& a, const Big& b) {
    if (a.d.size() != b.d.size()) return a.d.size() < b.d.size() ? -1 : 1;
    for (size_t i = a.d.size(); i-- > 0;)
      if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
    return 0;
  }
  friend Big operator+(const Big& a, const Big& b) {
    Big r;
    const size_t n = std::max(a.d.size(), b.d.size());
    r.d.resize(n + 1);
    uint64_t c = 0;
    for (size_t i = 0; i < n; ++i) {
      c += (uint64_t)(i < a.d.size() ? a.d[i] : 0) + (i < b.d.size() ? b.d[i] : 0);
      r.d[i] = (uint32_t)c;
      c >>= 32;
    }
    r.d[n] = (uint32_t)c;
    r.trim();
    return r;
  }
  friend Big operator-(const Big& a, const Big& b) {  // requires a >= b
    Big r;
    r.d.resize(a.d.size());
    int64_t br = 0;
    for (size_t i = 0; i < a.d.size(); ++i) {
      int64_t x = (int64_t)a.d[i] - (i < b.d.size() ? b.d[i] : 0) - br;
      br = x < 0;
      if (x < 0) x += (int64_t)1 << 32;
      r.d[i] = (uint32_t)x;
    }
    r.trim();
    return r;
  }
  friend Big operator*(const Big& a, const Big& b) {
    Big r;
    if (a.zero() || b.zero()) return r;
    r.d.assign(a.d.size() + b.d.size(), 0);
    for (size_t i = 0; i < a.d.size(); ++i) {
      uint64_t c = 0;
      for (size_t j = 0; j < b.d.size(); ++j) {
        c += (uint64_t)a.d[i] * b.d[j] + r.d[i + j];
        r.d[i + j] = (uint32_t)c;
        c >>= 32;
      }
      r.d[i + b.d.size()] += (uint32_t)c;
    }
    r.trim();
    return r;
  }
  Big shl(int k) const {
    Big r;
    if (zero()) return r;
    const int w = k / 32, b = k % 32;
    r.d.assign(d.size() + w + 1, 0);
    for (size_t i = 0; i < d.size(); ++i) {
      r.d[i + w] |= d[i] << b;
      if (b) r.d[i + w + 1] |= d[i] >> (32 - b);
    }
    r.trim();
    return r;
  }
  Big shr(int k) const {
    Big r;
    const int w = k / 32, b = k % 32;
    if (w >= (int)d.size()) return r;
    r.d.assign(d.size() - w, 0);
    for (size_t i = w; i < d.size(); ++i) {
      r.d[i - w] = d[i] >> b;
      if (b && i + 1 < d.size()) r.d[i - w] |= d[i + 1] << (32 - b);
    }
    r.trim();
    return r;
  }
  int bits() const {
    if (zero()) return 0;
    return 32 * (int)(d.size() - 1) + (32 - __builtin_clz(d.back()));
  }
  bool bit(int i) const { return (i / 32 < (int)d.size()) && ((d[i / 32] >> (i % 32)) & 1); }
  // floor(a / b) by shift-subtract long division
  static Big div(const Big& a, const Big& b) {
    if (b.zero()) throw std::runtime_error("division by zero");
    Big q, r;
    for (int i = a.bits() - 1; i >= 0; --i) {
      r = r.shl(1);
      if (a.bit(i)) r = r + Big(1);
      if (cmp(r, b) >= 0) {
        r = r - b;
        q = q + Big(1).shl(i);
      }
    }
    return q;
  }
  double to_double() const {
    double x = 0;
    for (size_t i = d.size(); i-- > 0;) x = x * 4294967296.0 + d[i];
    return x;
  }
  uint64_t to_u64() const {
    if (d.size() > 2) throw std::runtime_error("integer overflow");
    uint64_t v = 0;
    for (size_t i = d.size(); i-- > 0;) v = (v << 32) | d[i];
    return v;
  }
};

// non-negative rational n/d (not reduced; compared by cross-multiplication)
struct Rat {
  Big n, d;
  Rat() : n(), d(1) {}
  Rat(uint64_t a, uint64_t b = 1) : n(a), d(b) {}
  Rat(Big a, Big b) : n(std::move(a)), d(std::move(b)) {}
  static Rat of_double(double x) {  // exact: x = m * 2^e
    if (!(x >= 0) || std::isinf(x)) throw std::runtime_error("bad real");
    if (x == 0) return Rat(0, 1);
    int e;
    const double fr = std::frexp(x, &e);              // x = fr * 2^e, fr in [0.5, 1)
    const uint64_t m = (uint64_t)std::ldexp(fr, 53);  // exact 53-bit integer
    e -= 53;
    if (e >= 0) return Rat(Big(m).shl(e), Big(1));
    return Rat(Big(m), Big(1).shl(-e));
  }
  friend Rat operator+(const Rat& a, const Rat& b) { return Rat(a.n * b.d + b.n * a.d, a.d * b.d); }
  friend Rat operator*(const Rat& a, const Rat& b) { return Rat(a.n * b.n, a.d * b.d); }
  friend Rat operator/(const Rat& a, const Rat& b) { return Rat(a.n * b.d, a.d * b.n); }
  friend int cmp(const Rat& a, const Rat& b) { return Big::cmp(a.n * b.d, b.n * a.d); }
  Big floor() const { return Big::div(n, d); }
  Big ceil() const {
    Big q = Big::div(n, d);
    return Big::cmp(q * d, n) == 0 ? q : q + Big(1);
  }
  double to_double() const {  // for reporting: scale both into double range
    const int sh = std::max(0, std::max(n.bits(), d.bits()) - 900);
    return n.shr(sh).to_double() / d.shr(sh).to_double();
  }
};

// E[f(v)] of an integer-weight table as a rational
template <class F>
Rat expect(const Table& t, F f) {
  Big num, W;
  for (auto& e : t) {
    num = num + Big(e.second) * Big((uint64_t)f(e.first));
    W = W + Big(e.second);
  }
  return Rat(num, W);
}

// E[(l'+1)(l + l'/2)] = E[l'+1] E[l] + E[l'(l'+1)/2]  (l, l' independent;
// PAPER.md:1290-1297 / 1302-1309; reading R26)
Rat class_cost(const Table& lt, const Table& lpt) {
  const Rat El = expect(lt, [](uint64_t v) { return v; });
  const Rat Elp1 = expect(lpt, [](uint64_t v) { return v + 1; });
  const Rat tri = expect(lpt, [](uint64_t v) { return v * (v + 1); }) * Rat(1, 2);
  return Elp1 * El + tri;
}

double expect_d(const Table& t, double (*f)(double)) {
  double num = 0, W = 0;
  for (auto& e : t) { num += (double)e.second * f(e.first); W += (double)e.second; }
  return num / W;
}

}  // namespace

int compute_thresholds(const SetupInput& in, int mode, double delta, double budget_B,
                       sched_threshold_report* out, std::vector<uint32_t>* chosen,
                       std::string* err) {
  std::memset(out, 0, sizeof(*out));
  const int K = (int)in.lambda.size();
  // ---- fluid benchmark, reported in double
  double A = 0, thr = 0, lam_tot = 0;
  std::vector<double> cost_d(K), Elp1_d(K);
  for (int c = 0; c < K; ++c) {
    const double El = expect_d(in.l[c], [](double v) { return v; });
    const double Elp = expect_d(in.lp[c], [](double v) { return v; });
    Elp1_d[c] = expect_d(in.lp[c], [](double v) { return v + 1; });
    cost_d[c] = Elp1_d[c] * El + expect_d(in.lp[c], [](double v) { return v * (v + 1) / 2; });
    A += in.lambda[c] * cost_d[c];
    thr += in.lambda[c] * Elp;
    lam_tot += in.lambda[c];
  }
  out->rho = in.d1_s * A;
  out->thr_star = thr;
  const bool stable = out->rho < 1.0;
  if (stable) {
    out->dT_star = in.d0_s / (1.0 - out->rho);
    out->M_star = out->dT_star * A;
    for (int c = 0; c < K && c < 32; ++c) out->n_star[c] = out->dT_star * in.lambda[c] * Elp1_d[c];
  }

  const Rat d0 = Rat::of_double(in.d0_s), d1 = Rat::of_double(in.d1_s);
  std::vector<Rat> lam(K);
  for (int c = 0; c < K; ++c) lam[c] = Rat::of_double(in.lambda[c]);
  std::vector<uint32_t> n;

  if (in.policy == 0 /* WAIT */) {
    std::vector<Rat> cost(K);
    for (int c = 0; c < K; ++c) cost[c] = class_cost(in.l[c], in.lp[c]);
    auto mem = [&](const std::vector<uint32_t>& nn) {
      Rat m(0, 1);
      for (int c = 0; c < K; ++c) m = m + Rat(nn[c]) * cost[c];
      return m;
    };
    // Eq. wait_thresholds: d0 + d1 M^pi <= n_j / lambda_j
    auto feasible = [&](const std::vector<uint32_t>& nn) {
      const Rat dT = d0 + d1 * mem(nn);
      for (int c = 0; c < K; ++c)
        if (!lam[c].n.zero() && cmp(dT, Rat(nn[c]) / lam[c]) > 0) return false;
      return true;
    };
    if (!in.thresholds.empty()) {
      n = in.thresholds;
    } else if (mode == 1) {
      // heuristic n_j = B rho_j / (l'_j + 1), rho_j = lambda_j / sum lambda
      // (PAPER.md:1754), rounded half up, >= 1 (reading R13)
      Rat tot(0, 1);
      for (int c = 0; c < K; ++c) tot = tot + lam[c];
      for (int c = 0; c < K; ++c) {
        const Rat x = Rat(in.B) * lam[c] / tot / expect(in.lp[c], [](uint64_t v) { return v + 1; });
        const Rat xh = x + Rat(1, 2);
        n.push_back((uint32_t)std::max<uint64_t>(1, xh.floor().to_u64()));
      }
    } else {
      if (!stable) { *err = "rho >= 1: no stable WAIT thresholds (Prop. 1)"; return -2; }
      // smallest K on the candidate set {k / lambda_c}, n_c = max(1, ceil(lambda_c K))
      // (reading R24)
      std::vector<uint64_t> ks(K, 1);
      for (int it = 0; it < 10000000; ++it) {
        int cbest = -1;
        Rat Kb;
        for (int c = 0; c < K; ++c) {
          if (lam[c].n.zero()) continue;
          const Rat cand = Rat(ks[c]) / lam[c];
          if (cbest < 0 || cmp(cand, Kb) < 0) { Kb = cand; cbest = c; }
        }
        if (cbest < 0) { *err = "all rates are zero"; return -1; }
        std::vector<uint32_t> nn(K);
        for (int c = 0; c < K; ++c)
          nn[c] = lam[c].n.zero() ? 1u : (uint32_t)std::max<uint64_t>(1, (lam[c] * Kb).ceil().to_u64());
        if (feasible(nn)) { n = nn; break; }
        for (int c = 0; c < K; ++c)
          if (!lam[c].n.zero() && cmp(Rat(ks[c]) / lam[c], Kb) == 0) ++ks[c];
      }
      if (n.empty()) { *err = "no feasible WAIT thresholds"; return -3; }
    }
    const Rat M = mem(n);
    out->M_pi = M.to_double();
    out->dT_n = (d0 + d1 * M).to_double();
    out->feasible = feasible(n);
    out->mem_exceeds_M = cmp(M, Rat((uint64_t)in.M)) > 0;
  } else if (in.policy == 1 /* NESTED */) {
    const int L = (int)in.seg_end.size();
    // tail_k: rate of prompts with l' > e_{k-1} (reading R8)
    std::vector<Rat> tail(L);
    Rat Lam(0, 1), El_num(0, 1);
    for (int c = 0; c < K; ++c) {
      Lam = Lam + lam[c];
      El_num = El_num + lam[c] * expect(in.l[c], [](uint64_t v) { return v; });
    }
    const Rat El = El_num / Lam;
    for (int k = 0; k < L; ++k) {
      const uint64_t lo = k == 0 ? 0 : in.seg_end[k - 1];
      Rat t(0, 1);
      for (int c = 0; c < K; ++c)
        t = t + lam[c] * expect(in.lp[c], [lo](uint64_t v) { return (uint64_t)(v > lo); });
      tail[k] = t;
    }
    // exact per-stage memory sum_k n_k sum_{s in seg k} (E[l] + s) (reading R9)
    auto mem = [&](const std::vector<uint32_t>& nn) {
      Rat m(0, 1);
      for (int k = 0; k < L; ++k) {
        const uint64_t lo = k == 0 ? 0 : (uint64_t)in.seg_end[k - 1] + 1, hi = in.seg_end[k];
        const uint64_t cntk = hi - lo + 1, ssum = (lo + hi) * cntk / 2;
        m = m + Rat(nn[k]) * (Rat(cntk) * El + Rat(ssum));
      }
      return m;
    };
    // Eq. nested_wait_thresholds: dT(n) < n_1 / sum lambda
    auto dT_ok = [&](const std::vector<uint32_t>& nn) {
      return cmp(d0 + d1 * mem(nn), Rat(nn[0]) / Lam) < 0;
    };
    auto from_n1 = [&](uint32_t n1) {
      std::vector<uint32_t> nn{n1};
      for (int k = 1; k < L; ++k) {
        uint32_t next = 1;
        if (!tail[k - 1].n.zero()) {
          // smallest integer > n_{k} p_k, capped at n_k (reading R25)
          const Rat x = Rat(nn.back()) * tail[k] / tail[k - 1];
          next = (uint32_t)x.floor().to_u64() + 1;
        }
        nn.push_back(std::min(nn.back(), next));
      }
      return nn;
    };
    if (!in.thresholds.empty()) {
      n = in.thresholds;
    } else {
      for (uint32_t n1 = 1; n1 < 1000000; ++n1) {
        std::vector<uint32_t> nn = from_n1(n1);
        if (dT_ok(nn)) { n = nn; break; }
      }
      if (n.empty()) { *err = "no feasible nested thresholds"; return -3; }
    }
    const Rat M = mem(n);
    out->M_pi = M.to_double();
    out->dT_n = (d0 + d1 * M).to_double();
    bool ratio_ok = true;
    for (int k = 0; k + 1 < L; ++k)  // n_{k+1}/n_k > p_k
      if (cmp(Rat(n[k + 1]) * tail[k], Rat(n[k]) * tail[k + 1]) <= 0) ratio_ok = false;
    out->feasible = dT_ok(n) && ratio_ok;
    out->mem_exceeds_M = cmp(M, Rat((uint64_t)in.M)) > 0;
    // printed formula sum_k n_k (l + L'_k/2) dl'_k, L'_k cumulative
    double Mp = 0, Lc = 0, prev = 0;
    const double Eld = El.to_double();
    for (int k = 0; k < L; ++k) {
      Lc += in.seg_end[k];
      Mp += n[k] * (Eld + Lc / 2) * (in.seg_end[k] - prev);
      prev = in.seg_end[k];
    }
    out->M_pi_paper = Mp;
    // theta_k (Lemma) and the Thm-2 budget (PAPER.md:1692-1712,
    // union bound 2375-2407, reading R12)
    out->budget_base = out->M_pi;
    for (int k = 1; k < L; ++k) {
      const double foot = Eld + in.seg_end[k - 1];
      out->budget_queue += foot * n[k];
      if (tail[k - 1].n.zero()) continue;
      const double p = (tail[k] / tail[k - 1]).to_double();
      out->p[k] = p;
      const double np = n[k - 1], nk = n[k];
      if (!(np > nk && nk > np * p && p > 0 && p < 1)) continue;  // theta = inf or n/a
      auto g = [&](double x) { return -x * nk + np * std::log(1 - p + p * std::exp(x)); };
      double hi = 1.0;
      while (g(hi) < 0) hi *= 2;
      double lo = 0.0;
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (g(mid) < 0) lo = mid; else hi = mid;
      }
      const double th = 0.5 * (lo + hi);
      out->theta[k] = th;
      out->theta_lb[k] = 8 * (nk - np * p) / np;  // reading R10: / n_{k-1}
      if (delta > 0 && budget_B > 0 && L > 1)
        out->budget_hp += foot * std::log((L - 1) * budget_B / delta) / th;
    }
    out->budget_total = out->budget_base + out->budget_queue + out->budget_hp;
  } else {
    n.clear();  // FCFS has no thresholds
  }
  // time-varying check, NESTED only.  For piecewise-
  // constant rates the accumulated arrivals over [t, t+dT] are piecewise
  // linear in t, so the supremum is attained at t = b_p or t = b_p - dT;
  // p_k over any window is a mediant of per-piece ratios, so its supremum
  // is the largest per-piece ratio.
  out->tv_feasible = -1;
  bool any_tv = false;
  for (auto& r : in.rf) any_tv = any_tv || !r.empty();
  if (any_tv && in.policy == 1 && !n.empty()) {
    const double dT = out->dT_n;
    auto rate_at = [&](int c, double t) {  // lambda_c(t)
      if (in.rf[c].empty()) return in.lambda[c];
      double r = 0;
      for (auto& pc : in.rf[c]) if (pc.first <= t) r = pc.second;
      return r;
    };
    auto integral = [&](int c, double t0, double t1) {  // int_t0^t1 lambda_c
      if (in.rf[c].empty()) return in.lambda[c] * (t1 - t0);
      double acc = 0;
      const auto& P = in.rf[c];
      for (size_t p = 0; p < P.size(); ++p) {
        const double a = std::max(t0, P[p].first);
        const double b = std::min(t1, p + 1 < P.size() ? P[p + 1].first : 1e300);
        if (b > a) acc += P[p].second * (b - a);
      }
      return acc;
    };
    std::vector<double> cand{0.0};
    for (auto& r : in.rf)
      for (auto& pc : r) { cand.push_back(pc.first); cand.push_back(std::max(0.0, pc.first - dT)); }
    double sup = 0;
    for (double t : cand) {
      double a = 0;
      for (int c = 0; c < K; ++c) a += integral(c, t, t + dT);
      sup = std::max(sup, a);
    }
    out->tv_Lambda_pi = sup;
    bool ok = sup < (double)n[0];
    const int L = (int)in.seg_end.size();
    for (int k = 0; k + 1 < L; ++k) {
      // per-piece tail rates of segments k and k+1
      double pmax = 0;
      for (double t : cand) {
        double tk = 0, tk1 = 0;
        const uint64_t lo = k == 0 ? 0 : in.seg_end[k - 1], lo1 = in.seg_end[k];
        for (int c = 0; c < K; ++c) {
          double W = 0, w0 = 0, w1 = 0;
          for (auto& e : in.lp[c]) {
            W += (double)e.second;
            if (e.first > lo) w0 += (double)e.second;
            if (e.first > lo1) w1 += (double)e.second;
          }
          const double r = rate_at(c, t);
          tk += r * w0 / W;
          tk1 += r * w1 / W;
        }
        if (tk > 0) pmax = std::max(pmax, tk1 / tk);
      }
      if (k + 1 < 32) out->tv_p_star[k + 1] = pmax;
      if (!((double)n[k + 1] > (double)n[k] * pmax)) ok = false;
    }
    out->tv_feasible = ok;
  }
  out->n_thr = (uint32_t)std::min<size_t>(n.size(), 32);
  for (size_t i = 0; i < n.size() && i < 32; ++i) out->thresholds[i] = n[i];
  if (chosen) *chosen = n;
  return stable ? 0 : -2;
}

}  // namespace waitsim
