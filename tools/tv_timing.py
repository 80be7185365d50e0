import sys, os
sys.path.insert(0, '.')
import torch, workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows
import paper_2504_11320_b200._lib as L
wl = W.c3a_time_varying()
for kw in [{}, {"spec_resident": 1024}]:
    s = Scheduler(wl, W.Policy(W.FCFS, B=1024), None, **kw)
    out = torch.empty((L.NF, 10000), dtype=torch.int64, device="cuda")
    for rb in [0, 20_000_000, 0]:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run_rows(s, wl.seed, rb, 10000, wl.horizon_s, out); b.record(); torch.cuda.synchronize()
        print(kw, rb, round(a.elapsed_time(b), 1), s.launch_info()["spec_resident"], s.launch_info()["fallback_grid"])
