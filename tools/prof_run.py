"""One step of the bench workload (C2, WAIT then FCFS, 10^4 replications) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

R = int(os.environ.get("REPS", "10000"))
T = float(os.environ.get("HORIZON", "10.0"))
for pol in [W.Policy(W.WAIT), W.Policy(W.FCFS, B=1024)]:
    s = Scheduler(W.C2, pol)
    if pol.kind != W.FCFS:
        s.thresholds()
    rows = run_rows(s, W.C2.seed, 0, R, T)
    torch.cuda.synchronize()
    print(pol.kind, s.launch_info(), int(rows[7].sum()))
