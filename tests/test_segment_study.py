"""NEXT(3) segment-wise design study: the product's
bound terms agree with the oracle's exact-rational setup, show the paper's
U-shape in L, and (GPU) simulated peaks respect the Thm-4 bound."""
import math

import numpy as np
import pytest

import workloads as W
from oracle import fluid as fl
from paper_2504_11320_b200 import studies


@pytest.mark.parametrize("L", [4, 5, 10, 20])
def test_terms_match_oracle(L):
    r = studies.segment_terms(50.0, 200.0, 0.1, L)
    wl = studies.study_workload(50.0, 200.0)
    seg = r["seg_end"]
    n = fl.nested_strict(wl, seg, max_n1=2000)
    assert r["thresholds"] == n
    base, queue, hp, tot = fl.thm2_budget(wl, seg, n, 201.0, 0.1)
    assert (r["term1"], r["term2"], r["term3"], r["total"]) == pytest.approx((base, queue, hp, tot), rel=1e-9)


def test_u_shape_minimum_between_5_and_10():
    """'The minimum occurs around L = 5-10' and term 1
    dominates terms 2 and 3 (PAPER.md:1989 (i))."""
    for rate, d1 in [(50.0, None), (500.0, 3.5e-8)]:
        rows = [studies.segment_terms(rate, 200.0, 0.1, L, d1_s=d1) for L in (1, 2, 4, 5, 10, 20, 25)]
        ok = [r for r in rows if r["thresholds"]]
        best = min(ok, key=lambda r: r["total"])
        assert best["L"] in (5, 10)
        assert ok[-1]["total"] > best["total"] and ok[0]["total"] > best["total"]
        for r in ok:
            assert r["term1"] > r["term2"] and r["term1"] > r["term3"]
    # term 3 grows as delta shrinks and T grows (log dependence)
    a = studies.segment_terms(50.0, 200.0, 0.1, 10)["term3"]
    b = studies.segment_terms(50.0, 200.0, 1e-5, 10)["term3"]
    c = studies.segment_terms(50.0, 2000.0, 0.1, 10)["term3"]
    assert b > a and c > a


@pytest.mark.gpu
@pytest.mark.parametrize("L", [5, 10])
def test_simulated_peaks_respect_bound(L):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = studies.segment_terms(50.0, 200.0, 0.1, L)
    peaks, rows = studies.simulate_peaks(50.0, 200.0, L, r["thresholds"], 512)
    frac = float((peaks > r["total"]).mean())
    assert frac <= 0.1 + 3 * math.sqrt(0.1 * 0.9 / 512)


@pytest.mark.gpu
def test_thm1_zeta_sweep_strict_slack():
    """Thm 1 under strict slack: the zeta-normalised
    throughput gap shrinks ~ 1/zeta (faster than zeta^-1/2) and the
    zeta-normalised latency stays O(1)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rows = studies.zeta_sweep(zetas=(1, 4, 16), reps=2048)
    g1, g4, g16 = (r["gap"] for r in rows)
    assert g16 < g1 / 4 ** 0.5 * 0.5          # much faster than the zeta^-1/2 rate
    lat = [r["latency"] for r in rows]
    assert max(lat) < 1.5 * min(lat)
    assert all(r["evictions"] == 0 for r in rows)


@pytest.mark.gpu
def test_thm1_zeta_sweep_equality():
    """Thm 1 at equality dT(n) = n/lambda: gap O((zeta T)^-1/2), latency
    O((zeta T)^1/2) -- the gap falls roughly like zeta^-1/2 and latency grows."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rows = studies.zeta_sweep(zetas=(1, 16), reps=2048, slack=False)
    ratio = rows[1]["gap"] / rows[0]["gap"]
    assert 1 / 16 < ratio < 1 / 2          # between the 1/zeta and flat rates; ~ zeta^-1/2 = 1/4
    assert rows[1]["latency"] > 1.5 * rows[0]["latency"]
