"""One launch per policy of a workload for ncu (default: C2 WAIT + FCFS, 10^4 replications).
env: WL=C2|C4_<i>|C3a|C3b|C5_55, POLS=comma list of policy names, REPS, HORIZON"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

wl_name = os.environ.get("WL", "C2")
seg10 = [50 * k for k in range(1, 11)]
if wl_name == "C2":
    wl, pols = W.C2, [W.Policy(W.WAIT), W.Policy(W.FCFS, B=1024)]
elif wl_name.startswith("C4_"):
    wl = W.c4(int(wl_name[3:]))
    pols = [W.Policy(W.WAIT), W.Policy(W.NESTED, seg_end=[100, 200, 300]), W.Policy(W.FCFS, B=1024)]
elif wl_name == "C3a":
    wl, pols = W.C3A, [W.Policy(W.NESTED, seg_end=[20, 40, 80, 160]), W.Policy(W.FCFS, B=1024)]
elif wl_name == "C3a_tv":
    wl, pols = W.c3a_time_varying(), [W.Policy(W.NESTED, seg_end=[20, 40, 80, 160], thresholds=[11, 11, 10, 7]),
                                      W.Policy(W.FCFS, B=1024)]
elif wl_name == "C3b":
    wl, pols = W.C3B, [W.Policy(W.NESTED, seg_end=seg10), W.Policy(W.FCFS, B=2048)]
else:
    wl, pols = W.c5(55.0), [W.Policy(W.NESTED, seg_end=seg10), W.Policy(W.FCFS, B=1024)]  # bench.py's C5
if os.environ.get("POLS"):
    keep = os.environ["POLS"].split(",")
    pols = [p for p in pols if W.POLICY_NAMES[p.kind] in keep]
R = int(os.environ.get("REPS", "10000"))
T = float(os.environ.get("HORIZON", str(wl.horizon_s)))
for pol in pols:
    kw = dict(max_resident=4096, restart_cap=2_000_000_000) if wl_name.startswith("C5") else {}
    s = Scheduler(wl, pol, pol.thresholds, **kw)
    if pol.kind != W.FCFS and not pol.thresholds:
        s.thresholds()
    rows = run_rows(s, wl.seed, 0, R, T)
    torch.cuda.synchronize()
    print(W.POLICY_NAMES[pol.kind], s.launch_info(), int(rows[7].sum()))
