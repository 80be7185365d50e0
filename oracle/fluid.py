"""Host-side setup math of the paper in exact rational arithmetic -- TEST INFRASTRUCTURE.

Independent of the product's C++ `sched_thresholds` (csrc/setup.cpp): plain
Python `fractions.Fraction` (every float input is converted exactly), a
scan for the smallest feasible threshold vector, and float bisection for
theta.  Each function cites the passage it follows.

Length tables are integer-weight distributions; for the paper's fixed-length
types the expectations below reduce to the printed formulas (DESIGN.md
reading R26: with length tables, replace (l'+1)(l+l'/2) by its
expectation E[(l'+1)(l+l'/2)], l and l' independent).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction as Fr
from typing import List, Optional, Sequence


def _E(tab, f=lambda v: v) -> Fr:
    W = sum(w for _, w in tab)
    return sum(Fr(w) * Fr(f(v)) for v, w in tab) / W


def class_cost(l_tab, lp_tab) -> Fr:
    """E[(l'+1)(l+l'/2)]: KV-token iterations one prompt needs over its
    l'+1 stages (Prop. 1; 1302-1309)."""
    El = _E(l_tab)
    return _E(lp_tab, lambda v: v + 1) * El + _E(lp_tab, lambda v: Fr(v * (v + 1), 2))


@dataclass
class Fluid:
    rho: Fr
    dT: Optional[Fr]
    n_star: List[Fr]
    M_star: Optional[Fr]
    thr_star: Fr
    stable: bool


def fluid(wl) -> Fluid:
    """Multi-type fluid equilibrium (Eqs. memory_multi1/2,
    time_fluid, throughput_fluid_multiple): rho = d1 sum_j lambda_j c_j,
    dT* = d0/(1-rho), n*_j = dT* lambda_j (l'_j+1), M* = dT* sum lambda_j c_j,
    Throughput* = sum_j lambda_j l'_j.  Unstable iff rho >= 1 (Prop. 1,
    PAPER.md:1290)."""
    d0, d1 = Fr(wl.d0_s), Fr(wl.d1_s)
    lam = [Fr(x) for x in wl.lam]
    cost = [class_cost(a, b) for a, b in zip(wl.l_tab, wl.lp_tab)]
    A = sum(l * c for l, c in zip(lam, cost))
    rho = d1 * A
    thr = sum(l * _E(tab) for l, tab in zip(lam, wl.lp_tab))
    if rho >= 1:
        return Fluid(rho, None, [], None, thr, False)
    dT = d0 / (1 - rho)
    n_star = [dT * l * _E(tab, lambda v: v + 1) for l, tab in zip(lam, wl.lp_tab)]
    return Fluid(rho, dT, n_star, dT * A, thr, True)


def single_type(l: int, lp: int, lam: float, d0: float, d1: float):
    """Single-type closed forms: n*, M*, Throughput*."""
    l, lp, lam, d0, d1 = Fr(l), Fr(lp), Fr(lam), Fr(d0), Fr(d1)
    n = d0 * lam * (lp + 1) / (1 - d1 * lam * (lp + 1) * (l + lp / 2))
    return n, n * (l + lp / 2), lam * lp


# ----------------------------------------------------------------- WAIT
def wait_memory(wl, n: Sequence[int]) -> Fr:
    """M^pi = sum_j n_j (l'_j+1)(l_j+l'_j/2) (Eq. wait_thresholds)."""
    return sum(Fr(nj) * class_cost(a, b) for nj, a, b in zip(n, wl.l_tab, wl.lp_tab))


def wait_feasible(wl, n: Sequence[int]) -> bool:
    """d0 + d1 M^pi <= n_j / lambda_j for all j (Eq. wait_thresholds)."""
    dT = Fr(wl.d0_s) + Fr(wl.d1_s) * wait_memory(wl, n)
    return all(lam == 0 or dT <= Fr(nj) / Fr(lam) for nj, lam in zip(n, wl.lam))


def wait_fluid_integer(wl, max_k: int = 1_000_000) -> List[int]:
    """Smallest integer thresholds on the fluid ray (reading R24):
    scan K over {k/lambda_c} increasing, n_c = max(1, ceil(lambda_c K)),
    accept the first K with wait_feasible."""
    lam = [Fr(x) for x in wl.lam]
    # walk candidates lazily in increasing order (merge of K arithmetic sequences)
    ks = [1] * len(lam)
    while True:
        K = min(Fr(ks[c]) / lam[c] for c in range(len(lam)) if lam[c] > 0)
        n = [max(1, math.ceil(l * K)) if l > 0 else 1 for l in lam]
        if wait_feasible(wl, n):
            return n
        for c in range(len(lam)):
            if lam[c] > 0 and Fr(ks[c]) / lam[c] == K:
                ks[c] += 1
        if min(ks) > max_k:
            raise ValueError("no feasible WAIT thresholds")


def wait_heuristic(wl, B: int) -> List[int]:
    """n_j = B rho_j / (l'_j+1), rho_j = lambda_j / sum lambda,
    rounded half up, at least 1 (reading R13)."""
    tot = sum(Fr(x) for x in wl.lam)
    out = []
    for lam, tab in zip(wl.lam, wl.lp_tab):
        x = Fr(B) * Fr(lam) / tot / _E(tab, lambda v: v + 1)
        out.append(max(1, math.floor(x + Fr(1, 2))))
    return out


# --------------------------------------------------------------- NESTED
def nested_tails(wl, seg_end: Sequence[int]) -> List[Fr]:
    """tail_k = arrival rate of prompts that reach segment k, i.e. whose l'
    exceeds e_{k-1} (e_0 = 0): sum_{j>=k} lambda_j for the m-type model
    (PAPER.md:1680)."""
    out = []
    for k in range(len(seg_end)):
        lo = 0 if k == 0 else seg_end[k - 1]
        tot = Fr(0)
        for lam, tab in zip(wl.lam, wl.lp_tab):
            W = sum(w for _, w in tab)
            tot += Fr(lam) * Fr(sum(w for v, w in tab if v > lo), W)
        out.append(tot)
    return out


def nested_memory_exact(wl, seg_end: Sequence[int], n: Sequence[int]) -> Fr:
    """Memory with exactly n_k prompts at every stage of segment k:
    sum_k n_k sum_{s in seg k} (E[l]+s); segment 1 = stages 0..e_1, segment
    k>=2 = e_{k-1}+1..e_k.  This is the exact per-stage sum behind the garbled
    Eq. nested_wait_memory (old draft 287, 380-392;
    DESIGN.md reading R9)."""
    lam = [Fr(x) for x in wl.lam]
    El = sum(l * _E(t) for l, t in zip(lam, wl.l_tab)) / sum(lam)
    tot = Fr(0)
    for k, e in enumerate(seg_end):
        lo = 0 if k == 0 else seg_end[k - 1] + 1
        tot += Fr(n[k]) * sum(El + s for s in range(lo, e + 1))
    return tot


def nested_memory_paper(wl, seg_end, n) -> Fr:
    """The printed formula sum_k n_k (l + L'_k/2) dl'_k with cumulative
    L'_k = sum_{r<=k} l'_r -- reported, not used."""
    lam = [Fr(x) for x in wl.lam]
    El = sum(l * _E(t) for l, t in zip(lam, wl.l_tab)) / sum(lam)
    tot, L, prev = Fr(0), 0, 0
    for k, e in enumerate(seg_end):
        L += e
        tot += Fr(n[k]) * (El + Fr(L, 2)) * (e - prev)
        prev = e
    return tot


def nested_dT_ok(wl, seg_end, n) -> bool:
    """dT_[1..m](n) < n_1 / sum_j lambda_j (Eq. nested_wait_thresholds)."""
    lam = sum(Fr(x) for x in wl.lam)
    dT = Fr(wl.d0_s) + Fr(wl.d1_s) * nested_memory_exact(wl, seg_end, n)
    return dT < Fr(n[0]) / lam


def nested_from_n1(wl, seg_end, n1: int) -> List[int]:
    """n_{k+1} = min(n_k, floor(n_k p_k) + 1): the smallest integer with
    n_{k+1}/n_k > p_k, capped at n_k (Lemma hypothesis
    n_{k-1} > n_k; reading R25)."""
    tails = nested_tails(wl, seg_end)
    n = [n1]
    for k in range(1, len(seg_end)):
        p = tails[k] / tails[k - 1] if tails[k - 1] > 0 else Fr(0)
        n.append(min(n[-1], math.floor(n[-1] * p) + 1))
    return n


def nested_strict(wl, seg_end, max_n1: int = 100_000) -> List[int]:
    for n1 in range(1, max_n1):
        n = nested_from_n1(wl, seg_end, n1)
        if nested_dT_ok(wl, seg_end, n):
            return n
    raise ValueError("no feasible nested thresholds")


def nested_paper(wl, seg_end, ratio: Sequence[int]) -> List[int]:
    """Thresholds proportional to tail rates,
    smallest integer multiple meeting the dT condition."""
    for s in range(1, 100_000):
        n = [s * r for r in ratio]
        if nested_dT_ok(wl, seg_end, n):
            return n
    raise ValueError


def theta(n_prev: int, n_k: int, p: float, iters: int = 200) -> float:
    """Unique theta > 0 with e^{-theta n_k} (1-p+p e^theta)^{n_{k-1}} = 1
    (Lemma): bracket by doubling, then bisection on
    g(theta) = -theta n_k + n_{k-1} ln(1-p+p e^theta)."""
    if not (n_prev > n_k > n_prev * p and 0 < p < 1):
        raise ValueError("need n_{k-1} > n_k > n_{k-1} p_k")

    def g(x):
        return -x * n_k + n_prev * math.log(1 - p + p * math.exp(x))

    hi = 1.0
    while g(hi) < 0:
        hi *= 2
    lo = 0.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if g(mid) < 0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def thm2_budget(wl, seg_end, n, B: float, delta: float):
    """M^pi + sum_{k>=2} (l + e_{k-1}) (n_k + ln((L-1) B / delta) / theta_k)
    (Thm 2; union-bound form 2375-2407; R12).
    Returns (base, queue, hp, total) as floats; theta = inf (n_k = n_{k-1})
    drops the high-probability term."""
    lam = [Fr(x) for x in wl.lam]
    El = float(sum(l * _E(t) for l, t in zip(lam, wl.l_tab)) / sum(lam))
    tails = nested_tails(wl, seg_end)
    L = len(seg_end)
    base = float(nested_memory_exact(wl, seg_end, n))
    queue = hp = 0.0
    for k in range(1, L):
        foot = El + seg_end[k - 1]
        queue += foot * n[k]
        if n[k] < n[k - 1]:
            p = float(tails[k] / tails[k - 1])
            th = theta(n[k - 1], n[k], p)
            hp += foot * math.log((L - 1) * B / delta) / th
    return base, queue, hp, base + queue + hp


# ------------------------------------------------------- time-varying rates
def accumulated(rate_pieces, lam_const, t0: Fr, t1: Fr) -> Fr:
    """lambda_j[t0, t1] = int_{t0}^{t1} lambda_j(s) ds for a piecewise-constant
    rate ("accumulated arrivals of type j")."""
    if not rate_pieces:
        return Fr(lam_const) * (t1 - t0)
    acc = Fr(0)
    for p, (b, r) in enumerate(rate_pieces):
        lo = max(t0, Fr(b))
        hi = t1 if p + 1 == len(rate_pieces) else min(t1, Fr(rate_pieces[p + 1][0]))
        if hi > lo:
            acc += Fr(r) * (hi - lo)
    return acc


def validate_time_varying(wl, seg_end, n, dT):
    """Eq. nested_wait_thresholds_time_varying for
    piecewise-constant rates: Lambda^pi = sup_t sum_j lambda_j[t, t+dT] must
    be < n_1 and n_{k+1}/n_k > sup_{t,dt} p_k[t, t+dt].  The window integral
    is piecewise linear in t (sup at t = b or b - dT); p_k over a window is a
    mediant of instantaneous ratios, so its sup is the largest per-piece
    ratio.  Returns (Lambda_pi, [p*_k for k>=1], feasible)."""
    dT = Fr(dT)
    rfs = wl.rate_fn or [None] * wl.K
    cand = {Fr(0)}
    for pieces in rfs:
        for b, _ in (pieces or []):
            cand.add(Fr(b))
            cand.add(max(Fr(0), Fr(b) - dT))
    sup = max(sum(accumulated(rfs[c], wl.lam[c], t, t + dT) for c in range(wl.K)) for t in cand)
    pstar = [Fr(0)]
    for k in range(1, len(seg_end)):
        lo, lo1 = (0 if k == 1 else seg_end[k - 2]), seg_end[k - 1]
        best = Fr(0)
        for t in cand:
            tk = tk1 = Fr(0)
            for c in range(wl.K):
                pieces = rfs[c]
                r = Fr(wl.lam[c]) if not pieces else Fr([rr for b, rr in pieces if Fr(b) <= t][-1])
                W = sum(w for _, w in wl.lp_tab[c])
                tk += r * Fr(sum(w for v, w in wl.lp_tab[c] if v > lo), W)
                tk1 += r * Fr(sum(w for v, w in wl.lp_tab[c] if v > lo1), W)
            if tk > 0:
                best = max(best, tk1 / tk)
        pstar.append(best)
    ok = sup < n[0] and all(Fr(n[k]) > Fr(n[k - 1]) * pstar[k] for k in range(1, len(seg_end)))
    return sup, pstar, ok
