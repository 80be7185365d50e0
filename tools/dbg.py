import faulthandler, os, sys
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows
print("create", flush=True)
s = Scheduler(W.C2, W.Policy(W.WAIT))
print("thr", s.thresholds()["thresholds"], flush=True)
print("li", s.launch_info(), flush=True)
out = run_rows(s, 1, 0, 100, 1.0)
torch.cuda.synchronize()
print("ran", int(out[7].sum()), flush=True)
s2 = Scheduler(W.C3A, W.Policy(W.NESTED, seg_end=[20, 40, 80, 160]), [7, 7, 7, 5], spec_resident=32)
print("li2", s2.launch_info(), flush=True)
r = s2.run_host(1, 0, 8, 5.0)
print("ran2", r[7].sum(), flush=True)
