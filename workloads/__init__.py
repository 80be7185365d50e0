"""Seeded synthetic workloads shared by the oracle tests and the product path.

This module is INPUT DEFINITION ONLY: prompt classes (rate lambda_j, prefill
length table l_j, decode length table l'_j), the linear batch-time
coefficients (d0, d1), the KV limit M, batch-size limits, horizons and master
seeds.  It holds none of the method's arithmetic (no fluid solve, no
thresholds, no simulation) -- the oracle (`oracle/`) and the CUDA path
(`paper_2504_11320_b200/`) each derive everything else from these numbers on
their own.  The recipe behind every number is in DESIGN.md §3 ("input
recipe"); the shapes follow the paper's experiments:

* C2  -- PAPER.md:1750 (§Numerical Experiments, "Low demand": m=2,
         l=(10,10), l'=(10,20), lambda=(1000,1000)).
* C3a -- PAPER.md:1791 (Nested WAIT synthetic: m=4, l=10,
         l'=(20,40,80,160), rates 20:40:80:160).
* C4  -- PAPER.md:1752 ("High demand": m=3, l=20, l'=(100,200,300),
         rates 6000:4000:2000 used as a 3:2:1 ratio, rates swept).
* C5  -- PAPER.md:1793-1797 (LMSYS-shaped: decode 1..500 in 10 bins of 50
         with bin masses 23:11:8:7:6:4:3:2:1:1, mean prefill ~60, QPS 55).
* EX2 -- PAPER.md:1435-1446 (Example 2, l=l'=1, C=12, lambda=4).
* GOLDEN -- PAPER.md:2100-2104 (Prop. 3 instance (1,1,1),(1,2,1)).

A length table is a list of (value, integer weight) pairs; a 1-entry table is
a fixed length.  Rates are in 1/s, times in seconds, lengths/M in tokens.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

Table = List[Tuple[int, int]]  # [(value u16, weight u64)]

D0_S = 0.012        # 12 ms fixed iteration overhead (SURVEY A21 reading)
D1_S = 0.35e-6      # 0.35 us per KV token (SURVEY A21 reading)
M_7B = 131_072      # tokens: 64 GiB / 512 KiB per token of fp16 Llama-2-7B KV

WAIT, NESTED, FCFS, FCFS_ONGOING = 0, 1, 2, 3
POLICY_NAMES = {WAIT: "wait", NESTED: "nested", FCFS: "fcfs", FCFS_ONGOING: "fcfs_ongoing"}


def fixed(v: int) -> Table:
    return [(int(v), 1)]


@dataclass
class Workload:
    """One simulated system + arrival process (the method's input)."""
    name: str
    lam: List[float]            # per-class Poisson rate [1/s]
    l_tab: List[Table]          # per-class prefill length table
    lp_tab: List[Table]         # per-class decode length table
    M: int                      # KV-cache capacity [tokens]
    horizon_s: float            # simulated horizon T [s]
    seed: int                   # 64-bit master seed
    d0_s: float = D0_S
    d1_s: float = D1_S
    reps: int = 1               # replications the config is quoted on
    note: str = ""
    # optional time-varying rates: per class a list of
    # (start second, rate) pieces, first start 0; None / [] = constant lam
    rate_fn: Optional[List[Optional[List[Tuple[float, float]]]]] = None
    # piecewise-linear iteration time tau = d0 + d1 max(0, tokens - tau_b0)
    # (reading R31); 0 = the linear model
    tau_b0: int = 0

    @property
    def K(self) -> int:
        return len(self.lam)


@dataclass
class Policy:
    """Scheduler choice; thresholds None = let the setup recipe choose."""
    kind: int
    thresholds: Optional[List[int]] = None
    seg_end: Optional[List[int]] = None     # NESTED: last stage of each segment
    B: int = 0                               # FCFS: max resident prompts
    tok_budget: int = 0                      # FCFS: prefill tokens / iter (0 = inf)


def seed_for(k: int) -> int:
    return (0x25041132 << 32) | k


# --------------------------------------------------------------------------
# C1 / C1': single type l=8, l'=16, lambda=74/s, ~2000 arrivals.
C1 = Workload("C1", [74.0], [fixed(8)], [fixed(16)], M=256,
              horizon_s=2000.0 / 74.0, seed=seed_for(1), reps=1,
              note="WAIT n=1 is in the LIFO-eviction regime (M^pi=272>256)")
C1P = Workload("C1p", [74.0], [fixed(8)], [fixed(16)], M=272,
               horizon_s=2000.0 / 74.0, seed=seed_for(1), reps=1)

# C2: PAPER.md:1750 low-demand two-type workload, 7B KV budget.
C2 = Workload("C2", [1000.0, 1000.0], [fixed(10), fixed(10)],
              [fixed(10), fixed(20)], M=M_7B, horizon_s=10.0,
              seed=seed_for(2), reps=10_000)

# C3a: PAPER.md:1791 nested synthetic; kappa chosen for rho ~ 0.5.
_KAPPA = 10.582
C3A = Workload("C3a", [_KAPPA * r for r in (1, 2, 4, 8)], [fixed(10)] * 4,
               [fixed(20), fixed(40), fixed(80), fixed(160)], M=M_7B,
               horizon_s=60.0, seed=seed_for(3), reps=100_000)


def _geom_table(lo: int, hi: int, q: float, scale: float) -> Table:
    """Truncated geometric weights floor(scale * q^(y-lo)) on [lo, hi]."""
    return [(y, int(math.floor(scale * q ** (y - lo)))) for y in range(lo, hi + 1)]


# C3b: one class with geometric decode marks on [1,500] (E[l'] = 96.69).
C3B = Workload("C3b", [58.30], [fixed(60)], [_geom_table(1, 500, 0.99, 2.0 ** 40)],
               M=524_288, horizon_s=60.0, seed=seed_for(4), reps=100_000)

# C4: PAPER.md:1752 high demand, lambda split 3:2:1, total rate per rho grid.
C4_RHO = [0.5, 0.7, 0.8, 0.9, 0.95]
C4_LAMBDA_TOTAL = [71.06, 99.49, 113.70, 127.91, 135.02]


def c4(i: int) -> Workload:
    tot = C4_LAMBDA_TOTAL[i]
    return Workload(f"C4_rho{C4_RHO[i]}", [tot * 3 / 6, tot * 2 / 6, tot * 1 / 6],
                    [fixed(20)] * 3, [fixed(100), fixed(200), fixed(300)],
                    M=M_7B, horizon_s=20.0, seed=seed_for(5), reps=100_000)


# C5: chat-shaped marks (bin masses at 2675).
C5_BIN_MASS = [23, 11, 8, 7, 6, 4, 3, 2, 1, 1]


def _c5_lp_table() -> Table:
    # uniform inside each 50-token bin: every length in bin k gets weight b_k
    return [(y, C5_BIN_MASS[(y - 1) // 50]) for y in range(1, 501)]


def c5(qps: float = 55.0, arrivals: int = 1_000_000) -> Workload:
    return Workload(f"C5_qps{qps:g}", [qps],
                    [_geom_table(1, 1000, 1.0 - 1.0 / 60.0, 2.0 ** 40)],
                    [_c5_lp_table()], M=M_7B, horizon_s=arrivals / qps,
                    seed=seed_for(6), reps=16_384)


# Example 2 and the Prop.3 golden instance (2100-2104).
EX2 = Workload("EX2", [4.0], [fixed(1)], [fixed(1)], M=12, horizon_s=100.0,
               seed=seed_for(7), d0_s=0.5, d1_s=1.0 / 24.0)
GOLDEN = Workload("GOLDEN", [1.0, 1.0], [fixed(1), fixed(1)], [fixed(1), fixed(2)],
                  M=9, horizon_s=100.0, seed=seed_for(8), d0_s=0.5, d1_s=1.0 / 18.0)

# policies quoted with each workload (thresholds None = setup recipe)
POLICIES = {
    "C1": [Policy(WAIT), Policy(FCFS, B=32), Policy(NESTED, seg_end=[16])],
    "C2": [Policy(WAIT), Policy(FCFS, B=1024)],
    "C3a": [Policy(NESTED, seg_end=[20, 40, 80, 160]), Policy(FCFS, B=1024)],
    "C3b": [Policy(NESTED, seg_end=[50 * k for k in range(1, 11)]), Policy(FCFS, B=2048)],
    "C4": [Policy(WAIT), Policy(NESTED, seg_end=[100, 200, 300]), Policy(FCFS, B=1024)],
    "C5": [Policy(NESTED, seg_end=[50 * k for k in range(1, 11)]), Policy(FCFS, B=1024)],
}

# paper-given nested threshold ratios
PAPER_NESTED_RATIO_C3A = [15, 14, 12, 8]
PAPER_NESTED_RATIO_C5 = [66, 43, 32, 24, 17, 11, 7, 4, 2, 1]


# --------------------------------------------------------------------------
# Seeded random workloads for property / parity sweeps (tests only).
def random_small(rng, K: Optional[int] = None, max_len: int = 6,
                 horizon_s: float = 2.0) -> Workload:
    """A small random workload: a few classes, short lengths, tight M."""
    K = K or int(rng.integers(1, 4))
    lam, lt, lpt = [], [], []
    for _ in range(K):
        lam.append(float(rng.choice([5.0, 20.0, 50.0, 120.0])))
        if rng.random() < 0.5:
            lt.append(fixed(int(rng.integers(1, max_len + 1))))
        else:
            n = int(rng.integers(2, 5))
            lt.append([(int(v), int(rng.integers(1, 10))) for v in
                       sorted(rng.choice(range(1, max_len + 1), n, replace=False))])
        if rng.random() < 0.5:
            lpt.append(fixed(int(rng.integers(1, max_len + 1))))
        else:
            n = int(rng.integers(2, 5))
            lpt.append([(int(v), int(rng.integers(1, 10))) for v in
                        sorted(rng.choice(range(1, max_len + 1), n, replace=False))])
    maxfoot = max(max(v for v, _ in a) + max(v for v, _ in b) for a, b in zip(lt, lpt))
    M = int(rng.integers(maxfoot, maxfoot * 8 + 1))
    return Workload("rand", lam, lt, lpt, M=M, horizon_s=horizon_s,
                    seed=int(rng.integers(0, 2 ** 63)),
                    d0_s=float(rng.choice([0.002, 0.005, 0.01])),
                    d1_s=float(rng.choice([1e-5, 1e-4, 5e-4])))


def trace_arrays(arrivals: Sequence[Tuple[float, int, int, int]], tick_s: float = 1e-12):
    """Explicit trace [(t_seconds, class, l, l')] -> integer-tick tuples."""
    out = []
    for t, c, l, lp in arrivals:
        out.append((int(round(t / tick_s)), int(c), int(l), int(lp)))
    out.sort(key=lambda x: (x[0], x[1]))
    return out


# Time-varying variant of C3a (NEXT(2)): the same four
# types with a day-like profile -- rates scaled by 0.5x, 1.0x, 1.5x, 1.0x over
# four 15-second periods (peak = 1.5x the C3a rates).
def c3a_time_varying(profile=(0.5, 1.0, 1.5, 1.0), period_s: float = 15.0) -> Workload:
    wl = Workload("C3a_tv", list(C3A.lam), list(C3A.l_tab), list(C3A.lp_tab), M=C3A.M,
                  horizon_s=period_s * len(profile), seed=seed_for(9), reps=100_000)
    wl.rate_fn = [[(i * period_s, lam * f) for i, f in enumerate(profile)] for lam in C3A.lam]
    return wl
