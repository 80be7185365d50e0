import sys, numpy as np
sys.path.insert(0, '.')
import workloads as W, oracle
from paper_2504_11320_b200 import Scheduler
wl = W.c3a_time_varying()
for pol, thr in [(W.Policy(W.FCFS, B=1024), None), (W.Policy(W.WAIT), [3, 5, 9, 17])]:
    s = Scheduler(wl, pol, thr)
    print(pol.kind, s.launch_info(), flush=True)
    got = s.run_host(wl.seed, 0, 16, wl.horizon_s)
    ref = oracle.run(wl, pol, thr or [0], n_reps=16, n_threads=8)
    print("equal", np.array_equal(got, ref), flush=True)
