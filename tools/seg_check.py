"""Quick Nested parity + timing under each engine (development check, -m gpu
covers the same through pytest).  env: ENGINES=seg,member"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import workloads as W
from oracle import fluid as fl
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

SEG3A = [20, 40, 80, 160]
SEG10 = [50 * k for k in range(1, 11)]
SEG4 = [100, 200, 300]


def cases():
    yield "C1", W.C1, W.Policy(W.NESTED, seg_end=[16]), [1], 64, None, {}
    yield "C3a", W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), fl.nested_strict(W.C3A, SEG3A), 24, 20.0, {}
    yield "C3a_paper", W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), W.PAPER_NESTED_RATIO_C3A, 24, 20.0, {}
    yield "C3b", W.C3B, W.Policy(W.NESTED, seg_end=SEG10), fl.nested_strict(W.C3B, SEG10), 16, 20.0, {}
    for i in range(5):
        wl = W.c4(i)
        yield f"C4_{i}", wl, W.Policy(W.NESTED, seg_end=SEG4), fl.nested_strict(wl, SEG4), 12, 8.0, {}
    for q in (55.0, 110.0):
        yield f"C5_{q}", W.c5(q), W.Policy(W.NESTED, seg_end=SEG10), W.PAPER_NESTED_RATIO_C5, 8, 120.0, dict(
            max_resident=4096, restart_cap=1 << 20)
    yield "C3a_tv", W.c3a_time_varying(), W.Policy(W.NESTED, seg_end=SEG3A), [11, 11, 10, 7], 16, None, {}
    wl = W.Workload("k12", [10.0, 40, 0, 90, 10, 40, 0, 90, 10, 40, 0, 90], [W.fixed(2)] * 12,
                    [[(1, 5), (3, 2), (9, 1)]] * 12, M=120, horizon_s=1.0, seed=77, d0_s=0.004, d1_s=2e-4)
    yield "k12", wl, W.Policy(W.NESTED, seg_end=[2, 5, 9]), [4, 3, 2], 16, None, {}
    wl = W.Workload("skip", [40.0, 25.0, 90.0], [W.fixed(3), W.fixed(5), W.fixed(2)],
                    [W.fixed(4), W.fixed(9), W.fixed(2)], M=4000, horizon_s=6.0, seed=99)
    yield "skip1", wl, W.Policy(W.NESTED, seg_end=[2, 9]), [45, 20], 16, None, {}
    yield "skip2", wl, W.Policy(W.NESTED, seg_end=[2, 9]), [3, 2], 16, None, {}
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        wl = W.random_small(rng, horizon_s=1.5)
        maxlp = max(v for t in wl.lp_tab for v, _ in t)
        seg = sorted({int(x) for x in rng.integers(1, maxlp + 1, 2)} | {maxlp})
        [int(rng.integers(1, 5)) for _ in range(wl.K)]
        for _ in (0, 1):
            int(rng.integers(1, 40)); int(rng.choice([0, 0, 12]))
        thr = sorted([int(x) for x in rng.integers(1, 5, len(seg))], reverse=True)
        yield f"rand{seed}", wl, W.Policy(W.NESTED, seg_end=seg), thr, 16, None, {}
    for spec in (32, 64, 256):
        yield f"spec{spec}", W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), [7, 7, 7, 5], 24, 5.0, dict(spec_resident=spec)


def run_case(name, wl, pol, thr, n, T, kw):
    ref = oracle.run(wl, pol, thr, n_reps=n, n_threads=8, horizon_s=T)
    s = Scheduler(wl, pol, thr, **kw)
    got = s.run_host(wl.seed, 0, n, wl.horizon_s if T is None else T)
    eng = s.launch_info()["engine"]
    s.close()
    if np.array_equal(got, ref):
        return f"ok  eng={eng}"
    bad = {oracle.FIELDS[f]: int(np.sum(got[f] != ref[f])) for f in range(ref.shape[0])
           if not np.array_equal(got[f], ref[f])}
    reps = sorted(set(np.nonzero((got != ref).any(axis=0))[0].tolist()))[:4]
    return f"BAD eng={eng} {bad} reps {reps} status {got[oracle.F['status'], reps].tolist()}"


def traces():
    import hand_traces as H
    out = []
    for case in ("nested_A", "nested_B"):
        M, log_exp, row_exp = ((H.NESTED_A_M, H.NESTED_A_LOG, H.NESTED_A_ROW) if case == "nested_A"
                               else (H.NESTED_B_M, H.NESTED_B_LOG, H.NESTED_B_ROW))
        wl, pol, thr, T, tr = H.nested_workload(M), H.NESTED_POLICY, H.NESTED_THR, H.NESTED_T_S, H.NESTED_TRACE
        s = Scheduler(wl, pol, thr)
        rows, log = s.run_trace([tr], T, log_cap=64)
        s.close()
        ok = [tuple(int(x) for x in r) for r in log] == log_exp and H.row_matches(rows, 0, row_exp, oracle.F, oracle.u128) == {}
        out.append(f"{case}: {'ok' if ok else 'BAD'}")
    return out


def timing(wl, pol, thr, R, T):
    s = Scheduler(wl, pol, thr)
    if thr is None:
        s.thresholds()
    out = torch.empty((26, R), dtype=torch.int64, device="cuda")
    run_rows(s, wl.seed, 10 ** 6, R, T, out)
    torch.cuda.synchronize()
    ts = []
    for k in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_rows(s, wl.seed, k * R, R, T, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    st = int((out[23] != 0).sum())
    info = s.launch_info()
    s.close()
    return min(ts), info, st


for eng in os.environ.get("ENGINES", "seg,member").split(","):
    os.environ["WAITSIM_ENGINE"] = eng
    print(f"===== engine {eng}", flush=True)
    if os.environ.get("PARITY", "1") == "1":
        for c in cases():
            t0 = time.time()
            try:
                r = run_case(*c)
            except Exception as ex:  # noqa
                r = f"EXC {ex}"
            print(f"{c[0]:12s} {r}  ({time.time() - t0:.1f}s)", flush=True)
        for line in traces():
            print(line, flush=True)
    for name, wl, pol, R, T in [("C3a", W.C3A, W.Policy(W.NESTED, seg_end=SEG3A), 10000, None),
                                ("C4_2", W.c4(2), W.Policy(W.NESTED, seg_end=SEG4), 2000, None),
                                ("C3b", W.C3B, W.Policy(W.NESTED, seg_end=SEG10), 10000, None),
                                ("C5_55", W.c5(55.0), W.Policy(W.NESTED, seg_end=SEG10, thresholds=W.PAPER_NESTED_RATIO_C5), 2048, 1500.0)]:
        ms, info, st = timing(wl, pol, pol.thresholds, R, wl.horizon_s if T is None else T)
        print(f"TIME {name:6s} {ms:9.2f} ms  status!=0: {st}  {info}", flush=True)
