import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from paper_2504_11320_b200 import Scheduler, F
seg10 = [50 * k for k in range(1, 11)]
for qps in (55.0, 110.0):
    wl = W.c5(qps)
    for thr in ([11, 8, 6, 5, 4, 3, 2, 2, 2, 2], [33, 22, 16, 12, 9, 6, 4, 2, 1, 1]):
        s = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg10), thr, max_resident=4096, restart_cap=1 << 18)
        t = time.time()
        r = s.run_host(wl.seed, 0, 16, wl.horizon_s)
        print(qps, thr, "%.1fs" % (time.time() - t), "status", r[F["status"]].tolist()[:4],
              "res", r[F["final_resident"]].tolist()[:4], "wait", r[F["final_waiting"]].tolist()[:4],
              "evict", r[F["evictions"]].tolist()[:4], "maxkv", r[F["max_kv_peak"]].tolist()[:4],
              "rs", int(r[F["request_steps"]].sum()), flush=True)
