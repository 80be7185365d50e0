"""NEXT(4): the appendix's random-walk chains (App. B-C).

Oracle pins (-m "not gpu"): pathwise identities the Lemmas rest on (stuck
time, coupled dominance, Lindley representation), the arrival laws, and the
theory's expectations / tails (Spitzer-Strait identity, throughput-gap
bound, Kingman, Doob) computed independently from exact pmfs.  GPU parity
(-m gpu): the kernel's per-walk outputs equal the oracle's bit for bit.
"""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
from oracle import WF
from oracle import fluid as fl


def _pathwise(r, n, B, kind):
    c0 = 2 * n if kind == 0 else n
    # W^B = sum X - n (B - B_stuck): every non-stuck step removes a batch of n
    assert np.array_equal(r[WF["W_B"]], r[WF["sumX"]] - n * (B - r[WF["stuck"]]))
    # coupled process dominates at every step (Lemmas)
    assert (r[WF["viol"]] == 0).all()
    # Lindley: W~^B = c0 + S^B - min_{i<=B} S^i
    assert np.array_equal(r[WF["Wt_B"]] - c0, r[WF["S_B"]] - r[WF["minS"]])
    assert np.array_equal(r[WF["S_B"]], r[WF["sumX"]] - n * B)


@pytest.mark.parametrize("n,mu", [(8, 8.0), (4, 3.3), (20, 21.5)])
def test_wait_chain_pathwise_and_law(n, mu):
    B, N = 500, 2000
    r = oracle.walks(0, n, B, N, seed=11, mu=mu)
    _pathwise(r, n, B, 0)
    x = r[WF["sumX"]].astype(float)
    assert abs(x.mean() / B - mu) < 4 * math.sqrt(mu / (B * N))          # Poisson mean
    assert abs(x.var(ddof=1) / (B * mu) - 1) < 0.15                      # Poisson variance


def test_stuck_time_identity_and_gap_bound():
    """Lemma 'Queue Length and Stuck Time': at critical load
    E[W^B] = lambda E[B_stuck]; Lemma 'Throughput Gap Bound':
    E[W^B] - lambda <= sqrt(lambda) sum_k k^{-1/2}."""
    n, B, N = 8, 400, 4000
    r = oracle.walks(0, n, B, N, seed=3, mu=float(n))
    d = r[WF["W_B"]] - n * r[WF["stuck"]]
    assert abs(d.mean()) < 4 * d.std(ddof=1) / math.sqrt(N)
    bound = n + math.sqrt(n) * sum(k ** -0.5 for k in range(1, B + 1))
    assert r[WF["W_B"]].mean() <= bound


def test_spitzer_strait_identity():
    """E[max_{k<=B} S_k^+] = sum_k E[S_k^+]/k (Lemma 'Random Walk Maximum',
    PAPER.md:2187), with S_k = Poisson(k mu) - k n evaluated from the exact
    pmf."""
    n, mu, B, N = 6, 5.4, 60, 20000
    r = oracle.walks(0, n, B, N, seed=9, mu=mu)
    rhs = 0.0
    for k in range(1, B + 1):
        lo = k * n
        m = k * mu
        ks = np.arange(lo + 1, int(m + 20 * math.sqrt(m) + 50))
        rhs += float(np.sum((ks - lo) * stats.poisson.pmf(ks, m))) / k
    mx = r[WF["maxS"]].astype(float)
    assert abs(mx.mean() - rhs) < 4 * mx.std(ddof=1) / math.sqrt(N)


@pytest.mark.parametrize("n_prev,n,p", [(10, 6, 0.5), (7, 5, 2.0 / 3.0), (12, 10, 0.75)])
def test_nested_chain_kingman_and_doob(n_prev, n, p):
    """Segment-k chain with Binomial(n_{k-1}, p_k) thinning:
    Kingman E[W] <= n_k + n_{k-1} p(1-p) / (2 (n_k - n_{k-1} p)) (2324) and
    Doob P(max_i S^i >= c) <= exp(-theta_k c) (2360-2367)."""
    B, N = 400, 4000
    r = oracle.walks(1, n, B, N, seed=5, n_prev=n_prev, p=p)
    _pathwise(r, n, B, 1)
    x = r[WF["sumX"]].astype(float)
    assert abs(x.mean() / B - n_prev * p) < 4 * math.sqrt(n_prev * p * (1 - p) / (B * N))
    tavg = r[WF["sumW"]].astype(float) / B
    kingman = n + n_prev * p * (1 - p) / (2 * (n - n_prev * p))
    assert tavg.mean() <= kingman + 3 * tavg.std(ddof=1) / math.sqrt(N)
    th = fl.theta(n_prev, n, p)
    for c in range(1, 12):
        frac = float((r[WF["maxS"]] >= c).mean())
        bound = math.exp(-th * c)
        assert frac <= bound + 3 * math.sqrt(max(bound * (1 - bound), 1e-4) / N)


def test_walk_sharding_invariance():
    a = oracle.walks(1, 5, 100, 64, seed=1, n_prev=7, p=0.6)
    b = oracle.walks(1, 5, 100, 32, seed=1, walk_begin=32, n_prev=7, p=0.6)
    assert np.array_equal(a[:, 32:], b)


# ------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,mu,n_prev,p,B", [
    (0, 8, 8.0, 0, 0.0, 300), (0, 3, 2.2, 0, 0.0, 500), (0, 40, 39.0, 0, 0.0, 200),
    (1, 6, 0.0, 10, 0.5, 300), (1, 5, 0.0, 7, 2.0 / 3.0, 400), (1, 1, 0.0, 2, 0.3, 300)])
def test_gpu_walks_parity(kind, n, mu, n_prev, p, B):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_11320_b200._lib import walks
    N = 3000
    got = walks(kind, n, B, N, seed=123, walk_begin=77, mu=mu, n_prev=n_prev, p=p)
    ref = oracle.walks(kind, n, B, N, seed=123, walk_begin=77, mu=mu, n_prev=n_prev, p=p)
    assert np.array_equal(got, ref)
