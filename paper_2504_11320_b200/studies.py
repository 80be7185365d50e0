"""Segment-wise design study (NEXT(3); §Extensions "Segment Design").

For m decode-length types grouped into L segments of m/L types, the paper
bounds the Nested-WAIT memory by three terms (Eq. nested_wait_memory_L,
PAPER.md:1952-1962; plotted at 1978-2010):

  1. M^pi            peak batch memory with n_k prompts at every stage
  2. sum_{k>=2} n_k (l + l'_{k-1})            deterministic entry-queue bound
  3. sum_{k>=2} theta_k^-1 (l + l'_{k-1}) ln((L-1)(T+1)/delta)   high-probability term

and claims a U-shape in L with the minimum near L = 5-10.
This module computes the three terms with the product's host setup
(`sched_thresholds`: strict thresholds, exact stage-sum M^pi, theta_k by
bisection) and checks them against simulated peaks (`sched_run` with an
unconstrained KV limit): the fraction of replications whose peak KV
exceeds the bound must stay below delta (Thm 4).

Workload (the figure data are not printed): m = 500 single-token-spaced
decode types, prefill l = 62, rates proportional to the paper's LMSYS bin
masses 23:11:8:7:6:4:3:2:1:1 spread uniformly inside each 50-token bin
 -- one class with a decode-length table, which is the
same Poisson superposition the m-type model describes.
"""
from __future__ import annotations

import json
import math
import sys
from typing import Dict, List, Sequence

BIN_MASS = [23, 11, 8, 7, 6, 4, 3, 2, 1, 1]


def study_workload(total_rate: float, T: float, m: int = 500, l: int = 62, M: int = 1 << 40,
                   d1_s: float = None):
    import workloads as W
    lp = [(y, BIN_MASS[min(9, (y - 1) * 10 // m)]) for y in range(1, m + 1)]
    return W.Workload(f"segstudy_{total_rate:g}", [total_rate], [W.fixed(l)], [lp], M=M,
                      horizon_s=T, seed=W.seed_for(10), d1_s=W.D1_S if d1_s is None else d1_s)


def segment_terms(total_rate: float, T: float, delta: float, L: int, m: int = 500,
                  d1_s: float = None) -> Dict:
    """The three bound terms for L segments (host setup only)."""
    import workloads as W
    from . import SchedError, Scheduler
    wl = study_workload(total_rate, T, m, d1_s=d1_s)
    seg = [m * (k + 1) // L for k in range(L)]
    s = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg))
    # budget_B = T + 1 reproduces the figure's ln((L-1)(T+1)/delta)
    try:
        r = s.thresholds(mode=0, delta=delta, budget_B=T + 1)
    except SchedError as e:  # no integer thresholds meet Eq. nested_wait_thresholds_L
        return dict(L=L, seg_end=seg, thresholds=None, feasible=False, reason=str(e))
    base, queue, hp, total = r["budget"]
    return dict(L=L, seg_end=seg, thresholds=r["thresholds"], term1=base, term2=queue, term3=hp,
                total=total, dT=r["dT_n"], feasible=r["feasible"], theta=r["theta"])


def simulate_peaks(total_rate: float, T: float, L: int, thresholds: Sequence[int], reps: int,
                   m: int = 500, device: int = 0, d1_s: float = None):
    """Per-replication peak KV of Nested WAIT with these thresholds and no
    memory limit (so the bound's 'no overflow' event is observable)."""
    import numpy as np
    import workloads as W
    from . import F, Scheduler
    wl = study_workload(total_rate, T, m, d1_s=d1_s)
    seg = [m * (k + 1) // L for k in range(L)]
    # capacity: n_k per non-entry stage plus entry-queue margin (cf. derive_rc)
    cap = sum(n * (e - (seg[k - 1] if k else 0) + 4) for k, (n, e) in enumerate(zip(thresholds, seg)))
    cap = min(13_000, max(1024, int(cap * 1.25) + 256))
    s = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg), list(thresholds), device=device,
                  max_resident=cap)
    rows = s.run_host(wl.seed, 0, reps, T)
    if (rows[F["status"]] != 0).any():
        raise RuntimeError("capacity overflow in the segment study")
    return rows[F["max_kv_peak"]].astype(np.int64), rows


def segment_study(total_rate: float = 50.0, T: float = 200.0, delta: float = 0.1,
                  Ls: Sequence[int] = (1, 2, 4, 5, 10, 20, 25), reps: int = 2048,
                  simulate: bool = True, d1_s: float = None) -> List[Dict]:
    out = []
    for L in Ls:
        row = segment_terms(total_rate, T, delta, L, d1_s=d1_s)
        if simulate and row["thresholds"]:
            import numpy as np
            peaks, rows = simulate_peaks(total_rate, T, L, row["thresholds"], reps, d1_s=d1_s)
            row.update(peak_mean=float(peaks.mean()), peak_p99=float(np.percentile(peaks, 99)),
                       peak_max=int(peaks.max()),
                       frac_over_bound=float((peaks > row["total"]).mean()),
                       frac_over_mpi=float((peaks > row["term1"]).mean()), reps=reps)
        out.append(row)
    return out


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--rate", type=float, default=50.0)
    ap.add_argument("--T", type=float, default=200.0)
    ap.add_argument("--delta", type=float, default=0.1)
    ap.add_argument("--reps", type=int, default=2048)
    ap.add_argument("--d1", type=float, default=None, help="seconds per KV token (default 0.35e-6)")
    ap.add_argument("--no-sim", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    res = segment_study(a.rate, a.T, a.delta, reps=a.reps, simulate=not a.no_sim, d1_s=a.d1)
    txt = json.dumps(dict(rate=a.rate, T=a.T, delta=a.delta, d1=a.d1, rows=res))
    if a.out:
        open(a.out, "w").write(txt + "\n")
    for r in res:
        if not r["thresholds"]:
            print(f"L={r['L']:3d} infeasible")
            continue
        print(f"L={r['L']:3d} n={r['thresholds']} term1={r['term1']:.0f} term2={r['term2']:.0f} "
              f"term3={r['term3']:.0f} total={r['total']:.0f}"
              + (f" peak_p99={r['peak_p99']:.0f} over_bound={r['frac_over_bound']:.4f}" if 'peak_p99' in r else ""))


if __name__ == "__main__":
    main(sys.argv[1:])


# --------------------------------------------------- Thm 1 zeta-sweep (NEXT(4))
def zeta_sweep(zetas=(1, 2, 4, 8, 16), reps: int = 4096, slack: bool = True, device: int = 0):
    """Asymptotic regime of Thm 1: scale arrival rates
    by zeta and the batch-time coefficients by 1/zeta (C fixed).  WAIT with
    the fluid-integer thresholds of the zeta = 1 system.  Reports per zeta the
    throughput gap Throughput* - E[Throughput] (in tokens per unscaled second,
    i.e. divided by zeta) and mean latency / TTFT (times zeta): Thm 1 gives a
    gap O((zeta T)^-1) and O(1) latency under strict slack (dT < n_j/lambda_j),
    O((zeta T)^-1/2) and O((zeta T)^1/2) at equality."""
    import numpy as np
    import workloads as W
    from . import F, Scheduler, u128
    base = W.C1P if slack else W.Workload("C1eq", [74.0], [W.fixed(8)], [W.fixed(16)], M=272,
                                          horizon_s=W.C1P.horizon_s, seed=W.seed_for(11),
                                          d0_s=1.0 / 74.0 - W.D1_S * 272)
    out = []
    # at equality the recipe would round to n = 2 (M^pi > M); Thm 1's
    # equality case is n = 1 with dT(n) = n / lambda
    thr = None if slack else [1]
    for z in zetas:
        wl = W.Workload(f"{base.name}_z{z}", [x * z for x in base.lam], base.l_tab, base.lp_tab,
                        M=base.M, horizon_s=base.horizon_s, seed=base.seed,
                        d0_s=base.d0_s / z, d1_s=base.d1_s / z)
        s = Scheduler(wl, W.Policy(W.WAIT), thr, device=device)
        rep = s.thresholds()
        if thr is None:
            thr = rep["thresholds"]
        rows = s.run_host(wl.seed, 0, reps, wl.horizon_s)
        T = wl.horizon_s
        thr_tok = rows[F["completed_tokens"]].astype(float) / T
        lat = np.array(u128(rows, "lat"), float) / 1e12 / np.maximum(rows[F["completed"]], 1)
        ttft = np.array(u128(rows, "ttft"), float) / 1e12 / np.maximum(rows[F["first_tokens"]], 1)
        gap = (rep["thr_star"] - thr_tok) / z
        out.append(dict(zeta=z, thresholds=thr, dT_n=rep["dT_n"], slack=1.0 / 74.0 - rep["dT_n"] * z,
                        gap=float(gap.mean()), gap_se=float(gap.std(ddof=1) / np.sqrt(reps)),
                        latency=float((lat * z).mean()), ttft=float((ttft * z).mean()),
                        evictions=int(rows[F["evictions"]].sum())))
    return out
