import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle, workloads as W
from paper_2504_11320_b200 import Scheduler
SEG10 = [50 * k for k in range(1, 11)]
wl = W.c5(55.0)
pol = W.Policy(W.NESTED, seg_end=SEG10)
thr = W.PAPER_NESTED_RATIO_C5
for eng, capf, T, n in [("seg", "1.5", 300.0, 4), ("seg", "3", 300.0, 4), ("member", "1.5", 300.0, 4), ("seg", "1.5", 1500.0, 2), ("seg", "3", 1500.0, 64)]:
    os.environ["WAITSIM_ENGINE"] = eng; os.environ["WAITSIM_SEG_CAP"] = capf
    s = Scheduler(wl, pol, thr)
    t0 = time.time(); got = s.run_host(wl.seed, 0, n, T); dt = time.time() - t0
    info = s.launch_info(); s.close()
    ref = oracle.run(wl, pol, thr, n_reps=min(n, 4), n_threads=8, horizon_s=T)
    ok = np.array_equal(got[:, :min(n, 4)], ref)
    bad = {oracle.FIELDS[f]: int(np.sum(got[f, :min(n,4)] != ref[f])) for f in range(ref.shape[0]) if not np.array_equal(got[f, :min(n,4)], ref[f])}
    print(eng, capf, T, n, f"{dt:.2f}s", "ok" if ok else bad, "status", got[oracle.F["status"]].tolist()[:8], "evict", got[oracle.F["evictions"]].tolist()[:4], "res", got[oracle.F["final_resident"]].tolist()[:4], info["spec_resident"], flush=True)
