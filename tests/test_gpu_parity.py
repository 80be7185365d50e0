"""Parity of the CUDA path (through the C ABI) with the CPU oracle (-m gpu).

Bar: every integer field of every per-replication row is
bit-exact (counts, KV peaks, 128-bit tick sums, completion batch indices,
the trajectory hash); batch logs of explicit traces are identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import workloads as W
from oracle import fluid as fl

pytestmark = pytest.mark.gpu

SEG3A = [20, 40, 80, 160]
SEG10 = [50 * k for k in range(1, 11)]
SEG4 = [100, 200, 300]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2504_11320_b200 import lib
    lib()


def gpu_rows(wl, pol, thr, n, horizon_s=None, rep_begin=0, seed=None, **kw):
    from paper_2504_11320_b200 import Scheduler
    s = Scheduler(wl, pol, thr, **kw)
    out = s.run_host(wl.seed if seed is None else seed, rep_begin, n,
                     wl.horizon_s if horizon_s is None else horizon_s)
    s.close()
    return out


def assert_rows_equal(got, ref, what=""):
    assert got.shape == ref.shape
    if not np.array_equal(got, ref):
        bad = {oracle.FIELDS[f]: int(np.sum(got[f] != ref[f])) for f in range(ref.shape[0])
               if not np.array_equal(got[f], ref[f])}
        reps = sorted(set(np.nonzero((got != ref).any(axis=0))[0].tolist()))[:5]
        st = got[oracle.F["status"], reps].tolist()
        raise AssertionError(f"{what}: mismatching fields {bad}, first reps {reps}, gpu status {st}")


def check(wl, pol, thr, n, horizon_s=None, **kw):
    ref = oracle.run(wl, pol, thr, n_reps=n, n_threads=8, horizon_s=horizon_s)
    got = gpu_rows(wl, pol, thr, n, horizon_s, **kw)
    assert_rows_equal(got, ref, f"{wl.name}/{W.POLICY_NAMES[pol.kind]}")
    assert (got[oracle.F["status"]] == 0).all()
    return got


# ----------------------------------------------------------- configs
def test_c1_all_policies():
    check(W.C1, W.Policy(W.WAIT), [1], 64)          # LIFO-eviction regime (M < M^pi)
    check(W.C1P, W.Policy(W.WAIT), [1], 64)         # eviction-free
    check(W.C1, W.Policy(W.FCFS, B=32), [0], 64)
    check(W.C1, W.Policy(W.FCFS_ONGOING, B=32), [0], 64)
    check(W.C1, W.Policy(W.NESTED, seg_end=[16]), [1], 64)
    check(W.C1, W.Policy(W.WAIT), [3], 32)


def test_c2_wait_fluid_heuristic_fcfs():
    check(W.C2, W.Policy(W.WAIT), fl.wait_fluid_integer(W.C2), 48, horizon_s=2.0)
    check(W.C2, W.Policy(W.WAIT), fl.wait_heuristic(W.C2, 1024), 48, horizon_s=2.0)
    check(W.C2, W.Policy(W.FCFS, B=1024), [0], 48, horizon_s=2.0)
    check(W.C2, W.Policy(W.FCFS_ONGOING, B=1024), [0], 48, horizon_s=2.0)


def test_c2_full_horizon_sample():
    check(W.C2, W.Policy(W.WAIT), [16, 16], 16)
    check(W.C2, W.Policy(W.FCFS, B=1024), [0], 16)


def test_c3a_nested_strict_and_paper():
    check(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), fl.nested_strict(W.C3A, SEG3A), 24, horizon_s=20.0)
    check(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), W.PAPER_NESTED_RATIO_C3A, 24, horizon_s=20.0)
    check(W.C3A, W.Policy(W.FCFS, B=1024), [0], 24, horizon_s=20.0)


def test_c3b_geometric_marks():
    check(W.C3B, W.Policy(W.NESTED, seg_end=SEG10), fl.nested_strict(W.C3B, SEG10), 16, horizon_s=20.0)
    check(W.C3B, W.Policy(W.FCFS, B=2048), [0], 16, horizon_s=20.0)


@pytest.mark.parametrize("i", range(5))
def test_c4_rate_sweep(i):
    wl = W.c4(i)
    check(wl, W.Policy(W.WAIT), fl.wait_fluid_integer(wl), 12, horizon_s=8.0)
    check(wl, W.Policy(W.NESTED, seg_end=SEG4), fl.nested_strict(wl, SEG4), 12, horizon_s=8.0)
    check(wl, W.Policy(W.FCFS, B=1024), [0], 12, horizon_s=8.0)
    check(wl, W.Policy(W.FCFS_ONGOING, B=1024), [0], 12, horizon_s=8.0)


@pytest.mark.parametrize("qps", [55.0, 110.0])
def test_c5_chat_shaped(qps):
    wl = W.c5(qps)
    kw = dict(max_resident=4096, restart_cap=1 << 20)
    check(wl, W.Policy(W.NESTED, seg_end=SEG10), W.PAPER_NESTED_RATIO_C5, 8, horizon_s=120.0, **kw)
    check(wl, W.Policy(W.FCFS, B=1024), [0], 8, horizon_s=120.0, **kw)
    check(wl, W.Policy(W.FCFS_ONGOING, B=1024), [0], 8, horizon_s=120.0, **kw)


# ------------------------------------------------ time-varying rates (NEXT 2)
def test_c3a_time_varying_all_policies():
    wl = W.c3a_time_varying()
    check(wl, W.Policy(W.NESTED, seg_end=SEG3A), [11, 11, 10, 7], 16)
    check(wl, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5], 16)
    check(wl, W.Policy(W.FCFS, B=1024), [0], 16)
    check(wl, W.Policy(W.WAIT), [3, 5, 9, 17], 16)


@pytest.mark.parametrize("seed", range(12))
def test_random_time_varying(seed):
    rng = np.random.default_rng(500 + seed)
    wl = W.random_small(rng, horizon_s=1.5)
    rf = []
    for c in range(wl.K):
        if rng.random() < 0.3:
            rf.append(None)
            continue
        npieces = int(rng.integers(1, 5))
        starts = [0.0] + sorted(float(x) for x in rng.uniform(0.05, 1.4, npieces - 1))
        rf.append([(t0, float(rng.choice([0.0, 10.0, 40.0, 150.0]))) for t0 in starts])
    wl.rate_fn = rf
    maxlp = max(v for t in wl.lp_tab for v, _ in t)
    check(wl, W.Policy(W.WAIT), [int(rng.integers(1, 5)) for _ in range(wl.K)], 16)
    check(wl, W.Policy(W.FCFS, B=int(rng.integers(1, 40))), [0], 16)
    check(wl, W.Policy(W.NESTED, seg_end=[maxlp]), [int(rng.integers(1, 4))], 16)


# ------------------------------------------------- random small systems
@pytest.mark.parametrize("seed", range(40))
def test_random_small_workloads(seed):
    rng = np.random.default_rng(1000 + seed)
    wl = W.random_small(rng, horizon_s=1.5)
    maxlp = max(v for t in wl.lp_tab for v, _ in t)
    seg = sorted({int(x) for x in rng.integers(1, maxlp + 1, 2)} | {maxlp})
    check(wl, W.Policy(W.WAIT), [int(rng.integers(1, 5)) for _ in range(wl.K)], 16)
    for fk in (W.FCFS, W.FCFS_ONGOING):
        check(wl, W.Policy(fk, B=int(rng.integers(1, 40)),
                           tok_budget=int(rng.choice([0, 0, 12]))), [0], 16)
    check(wl, W.Policy(W.NESTED, seg_end=seg),
          sorted([int(x) for x in rng.integers(1, 5, len(seg))], reverse=True), 16)


# --------------------------------------------------------- explicit traces
@pytest.mark.parametrize("kind", [W.FCFS, W.FCFS_ONGOING])
def test_example2_trace_log(kind):
    from paper_2504_11320_b200 import Scheduler
    from test_oracle import _ex2_trace
    tr, t_end = _ex2_trace()
    pol = W.Policy(kind, B=1000)
    ref_rows, ref_log = oracle.run_trace(W.EX2, pol, [0], [tr], log_cap=32, horizon_s=t_end / 1e12)
    s = Scheduler(W.EX2, pol)
    rows, log = s.run_trace([tr], t_end / 1e12, log_cap=32)
    assert np.array_equal(log, ref_log)
    assert_rows_equal(rows, ref_rows, "EX2")


def test_bruteforce_tiny_traces():
    """P20(a): every multiset of <= 5 arrivals on a 5-point grid, M in 3..8,
    l, l' in {1,2}, three policies: GPU rows == oracle rows."""
    import itertools
    from paper_2504_11320_b200 import Scheduler
    unit = 4 * 10 ** 9
    for l, lp in [(1, 1), (1, 2), (2, 1), (2, 2)]:
        traces = []
        for k in range(6):
            for combo in itertools.combinations_with_replacement(range(5), k):
                traces.append([(x * unit, 0, l, lp) for x in combo])
        for M in range(l + lp, 9):
            wl = W.Workload("bf", [1.0], [W.fixed(l)], [W.fixed(lp)], M=M, horizon_s=0.1,
                            seed=0, d0_s=0.005, d1_s=0.001)
            for pol, thr in [(W.Policy(W.FCFS, B=3), [0]), (W.Policy(W.FCFS_ONGOING, B=3), [0]),
                             (W.Policy(W.WAIT), [1]), (W.Policy(W.WAIT), [2]),
                             (W.Policy(W.NESTED, seg_end=[lp]), [2])]:
                ref, _ = oracle.run_trace(wl, pol, thr, traces)
                s = Scheduler(wl, pol, thr)
                got, _ = s.run_trace(traces, 0.1)
                s.close()
                assert_rows_equal(got, ref, f"bf l={l} lp={lp} M={M} pol={pol.kind}")


def test_multiclass_traces_with_ties():
    """Same-tick arrivals across classes, restarts and tiny M on 2-3 classes."""
    from paper_2504_11320_b200 import Scheduler
    rng = np.random.default_rng(7)
    for trial in range(30):
        K = int(rng.integers(2, 4))
        l = [int(rng.integers(1, 4)) for _ in range(K)]
        lp = [int(rng.integers(1, 5)) for _ in range(K)]
        M = max(a + b for a, b in zip(l, lp)) + int(rng.integers(0, 8))
        wl = W.Workload("mc", [1.0] * K, [W.fixed(x) for x in l], [W.fixed(x) for x in lp],
                        M=M, horizon_s=0.2, seed=0, d0_s=0.003, d1_s=0.0005)
        traces = []
        for _ in range(8):
            n = int(rng.integers(0, 25))
            ts = sorted(int(x) * 2 * 10 ** 9 for x in rng.integers(0, 40, n))
            cl = [int(x) for x in rng.integers(0, K, n)]
            tr = sorted(zip(ts, cl), key=lambda x: (x[0], x[1]))
            traces.append([(t, c, l[c], lp[c]) for t, c in tr])
        maxlp = max(lp)
        for pol, thr in [(W.Policy(W.FCFS, B=int(rng.integers(1, 10))), [0]),
                         (W.Policy(W.FCFS_ONGOING, B=int(rng.integers(1, 10))), [0]),
                         (W.Policy(W.WAIT), [int(rng.integers(1, 4)) for _ in range(K)]),
                         (W.Policy(W.NESTED, seg_end=sorted({1, maxlp})), None)]:
            if thr is None:
                thr = sorted([int(x) for x in rng.integers(1, 4, len(pol.seg_end))], reverse=True)
            ref, _ = oracle.run_trace(wl, pol, thr, traces)
            s = Scheduler(wl, pol, thr)
            got, _ = s.run_trace(traces, 0.2)
            s.close()
            assert_rows_equal(got, ref, f"trial {trial} pol {pol.kind}")


# ---------------------------------------------- sharding / determinism / errors
def test_sharding_invariance_and_determinism():
    pol, thr = W.Policy(W.WAIT), [16, 16]
    full = gpu_rows(W.C2, pol, thr, 64, horizon_s=1.0)
    again = gpu_rows(W.C2, pol, thr, 64, horizon_s=1.0)
    assert np.array_equal(full, again)
    for g in (2, 4, 8):
        parts = [gpu_rows(W.C2, pol, thr, 64 // g, horizon_s=1.0, rep_begin=i * 64 // g) for i in range(g)]
        assert np.array_equal(np.concatenate(parts, axis=1), full)


@pytest.mark.parametrize("engine", ["member", "seg"])
@pytest.mark.parametrize("spec", [32, 64, 256])
def test_speculative_capacity_fallback(spec, engine, monkeypatch):
    """Replications overflowing the speculative capacity are re-run by the
    fallback launch with the safe capacity: rows stay bit-exact.  (Segment
    engine: its array is 1.5x the member engine's speculative population plus
    two admission batches; overflow re-runs on the member engine.)"""
    from paper_2504_11320_b200 import Scheduler
    monkeypatch.setenv("WAITSIM_ENGINE", engine)
    s = Scheduler(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5], spec_resident=spec)
    li = s.launch_info()
    want = spec if engine == "member" else ((int(1.5 * spec) + 14 + 31) // 32) * 32
    assert li["spec_resident"] == want and li["fallback_grid"] > 0
    got = s.run_host(W.C3A.seed, 0, 24, 20.0)
    ref = oracle.run(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5], n_reps=24, n_threads=8,
                     horizon_s=20.0)
    assert_rows_equal(got, ref, f"spec={spec}")
    s2 = Scheduler(W.C2, W.Policy(W.FCFS, B=1024), spec_resident=spec)
    got = s2.run_host(W.C2.seed, 0, 16, 2.0)
    ref = oracle.run(W.C2, W.Policy(W.FCFS, B=1024), [0], n_reps=16, n_threads=8, horizon_s=2.0)
    assert_rows_equal(got, ref, f"fcfs spec={spec}")


def test_capacity_overflow_is_reported():
    """A safe capacity below the population: status 1 in every row and in the
    handle's sticky status mask (sched_get_status), which a read clears."""
    from paper_2504_11320_b200 import Scheduler
    s = Scheduler(W.C2, W.Policy(W.FCFS, B=1024), max_resident=64)
    assert s.status_mask() == 0
    rows = s.run_host(W.C2.seed, 0, 4, 1.0)
    assert (rows[oracle.F["status"]] == 1).all()
    assert s.status_mask() == 1 << 1
    assert s.status_mask() == 0
    s.run_host(W.C2.seed, 0, 4, 0.001)  # too short to overflow
    assert s.status_mask() == 0
    s.close()


def test_full_size_bench_config_sampled():
    """C2 at the bench launch configuration (10^4 replications, both
    policies), sampled replications checked against the oracle one by one."""
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200.sim import run_rows
    idx = [0, 1, 777, 4095, 5000, 9998, 9999]
    for pol, thr in [(W.Policy(W.WAIT), [16, 16]), (W.Policy(W.FCFS, B=1024), [0])]:
        s = Scheduler(W.C2, pol, None if pol.kind == W.FCFS else thr)
        rows = run_rows(s, W.C2.seed, 0, 10_000, W.C2.horizon_s)
        torch.cuda.synchronize()
        got = rows.cpu().numpy().view(np.uint64)
        assert (got[oracle.F["status"]] == 0).all()
        for i in idx:
            ref = oracle.run(W.C2, pol, thr, n_reps=1, rep_begin=i)
            assert_rows_equal(got[:, i:i + 1], ref, f"C2 rep {i}")
        # properties at any size: conservation, memory bound
        f = lambda k: got[oracle.F[k]].astype(object)
        assert (f("arrivals") == f("completed") + f("completed_after_T") + f("final_waiting")
                + f("final_resident")).all()
        assert (got[oracle.F["max_kv_peak"]] <= W.C2.M).all()
        s.close()


# ------------------------------------------------------------- edge cases
def test_many_classes_and_zero_rates():
    """K = 12 classes (some with rate 0), variable length tables."""
    rng = np.random.default_rng(42)
    lam, lt, lpt = [], [], []
    for c in range(12):
        lam.append(0.0 if c % 5 == 3 else float(rng.choice([10.0, 40.0, 90.0])))
        lt.append(W.fixed(int(rng.integers(1, 6))) if c % 2 else [(2, 3), (4, 1), (7, 2)])
        lpt.append(W.fixed(int(rng.integers(1, 8))) if c % 3 else [(1, 5), (3, 2), (9, 1)])
    wl = W.Workload("k12", lam, lt, lpt, M=120, horizon_s=1.0, seed=77, d0_s=0.004, d1_s=2e-4)
    check(wl, W.Policy(W.WAIT), [int(x) for x in rng.integers(1, 4, 12)], 16)
    check(wl, W.Policy(W.FCFS, B=40), [0], 16)
    check(wl, W.Policy(W.FCFS_ONGOING, B=40, tok_budget=20), [0], 16)
    check(wl, W.Policy(W.NESTED, seg_end=[2, 5, 9]), [4, 3, 2], 16)


def test_degenerate_horizons_and_capacity():
    """No arrival before T; M = l + l' exactly (one prompt fits); all rates 0."""
    tiny = W.Workload("tiny", [0.5], [W.fixed(3)], [W.fixed(4)], M=7, horizon_s=0.01, seed=5)
    for pol, thr in [(W.Policy(W.WAIT), [1]), (W.Policy(W.FCFS, B=4), [0]),
                     (W.Policy(W.NESTED, seg_end=[4]), [1])]:
        check(tiny, pol, thr, 8)
        check(W.Workload("m", [50.0], [W.fixed(3)], [W.fixed(4)], M=7, horizon_s=1.0, seed=6),
              pol, thr, 8)
    zero = W.Workload("zero", [0.0, 0.0], [W.fixed(1)] * 2, [W.fixed(1)] * 2, M=10,
                      horizon_s=1.0, seed=1)
    rows = check(zero, W.Policy(W.FCFS, B=2), [0], 4)
    assert (rows[oracle.F["arrivals"]] == 0).all()


# ------------------------------------------- both engines, every eligible case
@pytest.mark.parametrize("engine", ["member", "ring"])
@pytest.mark.parametrize("case", ["c2_wait", "c2_fcfs", "c2_ongoing", "c4_wait_evict", "c4_fcfs_evict",
                                  "c1_wait_evict", "random_wait", "random_fcfs", "fcfs_evict_2cls",
                                  "ongoing_evict_2cls"])
def test_engines_bit_exact(engine, case, monkeypatch):
    """The member engine and the class-ring engine are two
    layouts of one semantics: forced either way, every row matches the
    oracle, including the LIFO-eviction regime (batched ring eviction) and
    pending first tokens of evicted prompts."""
    from paper_2504_11320_b200 import Scheduler
    monkeypatch.setenv("WAITSIM_ENGINE", engine)
    rng = np.random.default_rng(77)
    if case.startswith("c2"):
        kind = {"c2_wait": W.WAIT, "c2_fcfs": W.FCFS, "c2_ongoing": W.FCFS_ONGOING}[case]
        wl, pol, thr, n, T = W.C2, W.Policy(kind, B=1024), ([16, 16] if kind == W.WAIT else [0]), 24, 2.0
    elif case == "c4_wait_evict":
        wl, pol, thr, n, T = W.c4(3), W.Policy(W.WAIT), [9, 6, 3], 12, 8.0
    elif case == "c4_fcfs_evict":
        wl, pol, thr, n, T = W.c4(4), W.Policy(W.FCFS, B=1024), [0], 12, 8.0
    elif case in ("fcfs_evict_2cls", "ongoing_evict_2cls"):
        # two fixed-length classes, tight M: FCFS evicts (LIFO) across classes,
        # restarts must re-enter their own class ring
        wl = W.Workload("ev2", [30.0, 40.0], [W.fixed(2), W.fixed(1)], [W.fixed(3), W.fixed(5)], M=20,
                        horizon_s=3.0, seed=3, d0_s=0.02, d1_s=0.002)
        kind = W.FCFS if case == "fcfs_evict_2cls" else W.FCFS_ONGOING
        pol, thr, n, T = W.Policy(kind, B=1000), [0], 32, 3.0
    elif case == "c1_wait_evict":
        wl, pol, thr, n, T = W.C1, W.Policy(W.WAIT), [1], 32, W.C1.horizon_s
    else:
        wl = W.random_small(rng, horizon_s=2.0)
        while any(len(x) > 1 for x in wl.l_tab + wl.lp_tab):  # fixed lengths: ring-eligible
            wl = W.random_small(rng, horizon_s=2.0)
        kind = W.WAIT if case == "random_wait" else W.FCFS
        pol = W.Policy(kind, B=64)
        thr = [int(x) for x in rng.integers(1, 4, size=wl.K)] if kind == W.WAIT else [0]
        n, T = 32, 2.0
    s = Scheduler(wl, pol, None if pol.kind in (W.FCFS, W.FCFS_ONGOING) else thr)
    assert s.launch_info()["engine"] == (1 if engine == "ring" else 0)
    got = s.run_host(wl.seed, 0, n, T)
    s.close()
    ref = oracle.run(wl, pol, thr, n_reps=n, n_threads=8, horizon_s=T)
    assert_rows_equal(got, ref, f"{case}/{engine}")
    assert (got[oracle.F["status"]] == 0).all()


# ------------------------------- piecewise-linear iteration time
@pytest.mark.parametrize("engine", ["member", "ring"])
def test_piecewise_linear_tau(engine, monkeypatch):
    """tau = d0 + d1 max(0, tokens - b0) (reading R31), both engines, C2 with
    b0 inside the batch-token range, and random small systems."""
    import dataclasses
    monkeypatch.setenv("WAITSIM_ENGINE", engine)
    for b0 in [3000, 8000]:
        wl = dataclasses.replace(W.C2, tau_b0=b0)
        check(wl, W.Policy(W.WAIT), [16, 16], 16, horizon_s=2.0)
        check(wl, W.Policy(W.FCFS, B=1024), [0], 16, horizon_s=2.0)
    rng = np.random.default_rng(4242)
    for _ in range(6):
        wl = dataclasses.replace(W.random_small(rng, horizon_s=1.5), tau_b0=int(rng.integers(0, 40)))
        seg = [max(max(v for v, _ in t) for t in wl.lp_tab)]
        check(wl, W.Policy(W.NESTED, seg_end=seg), [2], 16)
        check(wl, W.Policy(W.FCFS, B=64), [0], 16)


def test_idle_skip_partial_jumps():
    """Idle skip: thresholds above the 32-arrival window force
    jumps to the window bound (partial), multi-class merges and ties at the
    horizon; rows stay bit-exact."""
    wl = W.Workload("skip", [40.0, 25.0, 90.0], [W.fixed(3), W.fixed(5), W.fixed(2)],
                    [W.fixed(4), W.fixed(9), W.fixed(2)], M=4000, horizon_s=6.0, seed=99)
    check(wl, W.Policy(W.WAIT), [40, 33, 70], 16)
    check(wl, W.Policy(W.WAIT), [1, 2, 3], 16)
    check(wl, W.Policy(W.NESTED, seg_end=[2, 9]), [45, 20], 16)
    check(wl, W.Policy(W.NESTED, seg_end=[2, 9]), [3, 2], 16)


def test_engine_selection_rule(monkeypatch):
    """the class-ring engine for every fixed-length WAIT /
    FCFS configuration (and one-class one-segment Nested, P10) (its member records live in global memory, so its
    footprint no longer depends on the population), the segment engine for
    Nested except one segment or decode-length marks with M^pi > M (member
    engine, measured faster there), the member engine for length marks under
    WAIT / FCFS."""
    from paper_2504_11320_b200 import Scheduler
    monkeypatch.delenv("WAITSIM_ENGINE", raising=False)
    eng = lambda wl, pol, thr=None: Scheduler(wl, pol, thr).launch_info()["engine"]
    assert eng(W.C2, W.Policy(W.WAIT), [16, 16]) == 1
    assert eng(W.C2, W.Policy(W.FCFS, B=1024)) == 1
    assert eng(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5]) == 2
    assert eng(W.C3B, W.Policy(W.NESTED, seg_end=SEG10), fl.nested_strict(W.C3B, SEG10)) == 2
    assert eng(W.c4(4), W.Policy(W.NESTED, seg_end=SEG4), [46, 23, 8]) == 2
    # one class, one segment: Nested IS WAIT with one type (P10, pinned on the
    # oracle) -> its runs go to a WAIT twin handle on the class-ring engine
    assert eng(W.C1, W.Policy(W.NESTED, seg_end=[16]), [1]) == 1
    assert eng(W.c5(55.0), W.Policy(W.NESTED, seg_end=SEG10), [11, 8, 6, 5, 4, 3, 2, 2, 2, 2]) == 0  # marks, M^pi > M
    monkeypatch.setenv("WAITSIM_ENGINE", "member")
    assert eng(W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5]) == 0
    assert eng(W.C2, W.Policy(W.FCFS, B=1024)) == 0
    monkeypatch.delenv("WAITSIM_ENGINE")
    assert eng(W.C3B, W.Policy(W.FCFS, B=2048)) == 0                 # marks
    assert eng(W.c4(1), W.Policy(W.FCFS, B=1024)) == 1               # long decodes
    assert eng(W.c4(4), W.Policy(W.WAIT), [18, 12, 6]) == 1
    assert eng(W.c4(2), W.Policy(W.WAIT), [6, 4, 2]) == 1


@pytest.mark.parametrize("name", ["C3a", "C3b", "C4", "C5"])
def test_full_size_bench_workloads_sampled(name):
    """Every bench workload at its bench launch configuration (bench.py's
    registry: replication counts, horizons, thresholds from sched_thresholds,
    handle options), sampled replications checked against the oracle one by
    one, conservation and the memory bound checked on every row."""
    import importlib.util
    import os
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200.sim import run_rows
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    pols, reps, _ = bench.expand(name)
    if name == "C4":
        pols = [p for p in pols if p[0].endswith("@0.5") or p[0].endswith("@0.9")]
    kw = bench.SCHED_KW.get(name, {})
    n_check = 2 if name == "C5" else 4
    for label, pol, thr, wl in pols:
        s = Scheduler(wl, pol, thr, **kw)
        if thr is None and pol.kind in (W.WAIT, W.NESTED):
            thr = s.thresholds()["thresholds"]
        rows = run_rows(s, wl.seed, 0, reps, wl.horizon_s)
        torch.cuda.synchronize()
        got = rows.cpu().numpy().view(np.uint64)
        s.close()
        assert (got[oracle.F["status"]] == 0).all(), label
        for i in np.linspace(0, reps - 1, n_check).astype(int).tolist():
            ref = oracle.run(wl, pol, thr if thr is not None else [0], n_reps=1, rep_begin=i)
            assert_rows_equal(got[:, i:i + 1], ref, f"{name}/{label} rep {i}")
        f = lambda k: got[oracle.F[k]].astype(object)
        assert (f("arrivals") == f("completed") + f("completed_after_T") + f("final_waiting")
                + f("final_resident")).all()
        assert (got[oracle.F["max_kv_peak"]] <= wl.M).all()


def test_r28_trace_log():
    """Reading R28 (class-major simultaneous WAIT admissions decide the LIFO
    victim), the hand-traced CPU pin's trace through sched_run_trace."""
    from paper_2504_11320_b200 import Scheduler
    from test_oracle import _r28_trace
    wl, tr = _r28_trace()
    ref_rows, ref_log = oracle.run_trace(wl, W.Policy(W.WAIT), [1, 1], [tr], log_cap=8)
    s = Scheduler(wl, W.Policy(W.WAIT), [1, 1])
    rows, log = s.run_trace([tr], wl.horizon_s, log_cap=8)
    assert np.array_equal(log, ref_log)
    assert_rows_equal(rows, ref_rows, "R28")
    assert (int(log[1][2]), int(log[1][4])) == (5, 1)  # tokens, evictions of batch 2


# ---------------------------------------------- hand traces (tests/hand_traces.py)
@pytest.mark.parametrize("case", ["nested_A", "nested_B", "fcfs_budget"])
def test_hand_traces_replayed(case):
    """The hand-derived batch logs and rows of the multi-segment Nested WAIT
    traces (Alg. 2: k* prefix, >= at equality,
    oldest-first entry stage, paused KV, LIFO cascade) and the FCFS token
    budget, replayed through sched_run_trace: equal to the hand values and
    to the oracle, element by element."""
    import hand_traces as H
    from paper_2504_11320_b200 import Scheduler
    if case == "fcfs_budget":
        wl, pol, thr, T, log_exp, row_exp = (H.fcfs_workload(), H.FCFS_POLICY, [0], 10.0, H.FCFS_LOG,
                                             H.FCFS_ROW)
        tr = H.FCFS_TRACE
    else:
        M, log_exp, row_exp = ((H.NESTED_A_M, H.NESTED_A_LOG, H.NESTED_A_ROW) if case == "nested_A"
                               else (H.NESTED_B_M, H.NESTED_B_LOG, H.NESTED_B_ROW))
        wl, pol, thr, T, tr = H.nested_workload(M), H.NESTED_POLICY, H.NESTED_THR, H.NESTED_T_S, H.NESTED_TRACE
    s = Scheduler(wl, pol, thr if pol.kind != W.FCFS else None)
    rows, log = s.run_trace([tr], T, log_cap=64)
    s.close()
    assert [tuple(int(x) for x in r) for r in log] == log_exp
    assert H.row_matches(rows, 0, row_exp, oracle.F, oracle.u128) == {}
    ref_rows, ref_log = oracle.run_trace(wl, pol, thr, [tr], log_cap=64, horizon_s=T)
    assert np.array_equal(log, ref_log)
    assert_rows_equal(rows, ref_rows, case)


# ------------------------------------------------ restart pool
def test_restart_pool_chunks_are_reused():
    """C1 WAIT evicts ~280 prompts per replication; 16,384 replications push
    ~4.6M restart entries through a pool of 2^19 (8,192 chunks, more than
    the ~4,700 warps in flight each hold while a restart waits): chunks are
    returned and reused, every row has status 0, sampled rows equal the
    oracle and the high-water mark stays within the pool."""
    from paper_2504_11320_b200 import Scheduler
    s = Scheduler(W.C1, W.Policy(W.WAIT), [1], restart_cap=1 << 19)
    rows = s.run_host(W.C1.seed, 0, 16384, W.C1.horizon_s)
    pool = s.restart_pool()
    s.close()
    assert (rows[oracle.F["status"]] == 0).all()
    assert int(rows[oracle.F["evictions"]].astype(np.int64).sum()) > 4 * pool["capacity_entries"]
    assert 0 < pool["high_water_entries"] <= pool["capacity_entries"]
    for i in [0, 1, 5000, 16383]:
        ref = oracle.run(W.C1, W.Policy(W.WAIT), [1], n_reps=1, rep_begin=i)
        assert_rows_equal(rows[:, i:i + 1], ref, f"C1 rep {i}")


def test_restart_pool_exhaustion_is_reported():
    """A pool of one chunk cannot hold the concurrent restarts of 256 C1
    replications: some rows report status 2, the others stay bit-exact."""
    from paper_2504_11320_b200 import Scheduler
    s = Scheduler(W.C1, W.Policy(W.WAIT), [1], restart_cap=64)
    rows = s.run_host(W.C1.seed, 0, 256, W.C1.horizon_s)
    assert s.status_mask() == 1 << 2
    s.close()
    st = rows[oracle.F["status"]]
    assert (st == 2).any() and set(st.tolist()) <= {0, 2}
    ok = np.nonzero(st == 0)[0][:4].tolist()
    for i in ok:
        ref = oracle.run(W.C1, W.Policy(W.WAIT), [1], n_reps=1, rep_begin=i)
        assert_rows_equal(rows[:, i:i + 1], ref, f"C1 rep {i}")


# ------------------------------- Nested: segment engine vs member engine
@pytest.mark.parametrize("engine", ["member", "seg"])
@pytest.mark.parametrize("case", ["c1", "c3a", "c3b", "c4_evict", "c5_thrash", "k12", "random", "tight_cap",
                                  "one_stage_segments"])
def test_nested_engines_bit_exact(engine, case, monkeypatch):
    """The member engine and the segment engine (residents in
    admission order = stage order, completion histograms per segment,
    cohorts leaving as blocks, tombstones and compaction) are two layouts of
    Algorithm 2's semantics: forced either way, every
    row matches the oracle -- LIFO eviction into entry-stage queues, late
    last batches, completions at entry stages (one-stage segments) and
    compaction under a tight array (tight_cap) included."""
    from paper_2504_11320_b200 import Scheduler
    monkeypatch.setenv("WAITSIM_ENGINE", engine)
    kw, T = {}, None
    if case == "c1":
        wl, seg, thr, n = W.C1, [16], [1], 64
    elif case == "c3a":
        wl, seg, thr, n, T = W.C3A, SEG3A, W.PAPER_NESTED_RATIO_C3A, 24, 20.0
    elif case == "c3b":
        wl, seg, n, T = W.C3B, SEG10, 16, 20.0
        thr = fl.nested_strict(wl, seg)
    elif case == "c4_evict":
        wl, seg, n, T = W.c4(3), SEG4, 12, 8.0
        thr = fl.nested_strict(wl, seg)
    elif case == "c5_thrash":
        wl, seg, n, T = W.c5(55.0), SEG10, 8, 200.0
        thr = fl.nested_strict(wl, seg)
    elif case == "k12":
        wl = W.Workload("k12", [10.0, 40, 0, 90] * 3, [W.fixed(2)] * 12, [[(1, 5), (3, 2), (9, 1)]] * 12,
                        M=120, horizon_s=1.0, seed=77, d0_s=0.004, d1_s=2e-4)
        seg, thr, n = [2, 5, 9], [4, 3, 2], 16
    elif case == "random":
        rng = np.random.default_rng(7)
        for _ in range(8):
            wl = W.random_small(rng, horizon_s=1.5)
            maxlp = max(v for t in wl.lp_tab for v, _ in t)
            seg = sorted({int(x) for x in rng.integers(1, maxlp + 1, 3)} | {maxlp})
            thr = sorted([int(x) for x in rng.integers(1, 6, len(seg))], reverse=True)
            check(wl, W.Policy(W.NESTED, seg_end=seg), thr, 16)
        return
    elif case == "tight_cap":
        monkeypatch.setenv("WAITSIM_SEG_CAP", "0.5")
        wl, seg, thr, n, T = W.C3A, SEG3A, [7, 7, 7, 5], 32, 6.0
    else:  # segments of one stage: entry stage = last stage (W_k = 0)
        wl = W.Workload("w0", [30.0, 20.0], [W.fixed(3), [(1, 2), (6, 1)]], [[(2, 1), (3, 1), (4, 2)], W.fixed(5)],
                        M=90, horizon_s=3.0, seed=123, d0_s=0.01, d1_s=1e-4)
        seg, thr, n = [2, 3, 4, 5], [3, 3, 2, 2], 24
    got = check(wl, W.Policy(W.NESTED, seg_end=seg), thr, n, horizon_s=T, **kw)
    s = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg), thr)
    assert s.launch_info()["engine"] == (2 if engine == "seg" else 0)
    s.close()
    f = lambda k: got[oracle.F[k]].astype(object)
    assert (f("arrivals") == f("completed") + f("completed_after_T") + f("final_waiting")
            + f("final_resident")).all()


@pytest.mark.parametrize("name", ["C2", "C3a", "C3a_tv", "C3b", "C4"])
def test_speculative_capacity_rarely_falls_back(name):
    """Cost guard on the speculative capacities: at every
    bench workload's launch configuration at most 1% of the replications
    overflow the main launch and re-run in the fallback launch
    (`launch_info()["last_retries"]`).  Rows are bit-exact either way; a
    systematic overflow doubles the cost (C3a_tv FCFS once re-ran all 10^4:
    117 vs 47 ms)."""
    import importlib.util
    import os
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200.sim import run_rows
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    pols, reps, _ = bench.expand(name)
    for label, pol, thr, wl in pols:
        s = Scheduler(wl, pol, thr, **bench.SCHED_KW.get(name, {}))
        if thr is None and pol.kind in (W.WAIT, W.NESTED):
            s.thresholds()
        rows = run_rows(s, wl.seed, 0, reps, wl.horizon_s)
        torch.cuda.synchronize()
        li = s.launch_info()
        s.close()
        assert int((rows[oracle.F["status"]] != 0).sum().item()) == 0, label
        assert li["last_retries"] <= reps // 100, f"{name}/{label}: {li['last_retries']} of {reps} re-ran"


def test_one_segment_nested_runs_as_wait(monkeypatch):
    """P10 routing: a one-class one-segment Nested handle runs on its WAIT twin
    (class-ring engine); rows are bit-identical to the oracle's Nested rows and
    to the same handle forced onto the Nested member engine, with thresholds
    installed by sched_thresholds after creation."""
    from paper_2504_11320_b200 import Scheduler
    monkeypatch.delenv("WAITSIM_ENGINE", raising=False)
    pol = W.Policy(W.NESTED, seg_end=[16])
    for thr in ([1], [2], None):
        s = Scheduler(W.C1, pol, thr)
        th = thr if thr is not None else s.thresholds()["thresholds"]
        assert s.launch_info()["engine"] == 1
        got = s.run_host(W.C1.seed, 5, 64, 8.0)
        assert s.status_mask() == 0
        s.close()
        ref = oracle.run(W.C1, pol, th, n_reps=64, rep_begin=5, n_threads=8, horizon_s=8.0)
        assert_rows_equal(got, ref, f"nested one segment thr={th}")
        monkeypatch.setenv("WAITSIM_ENGINE", "member")
        s = Scheduler(W.C1, pol, th)
        assert s.launch_info()["engine"] == 0
        assert_rows_equal(s.run_host(W.C1.seed, 5, 64, 8.0), ref, "member engine")
        s.close()
        monkeypatch.delenv("WAITSIM_ENGINE")
