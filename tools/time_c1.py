"""C1 timing of all three policies (CUDA events, best of 3); runs against the package in cwd."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows
R = 16384
for name, pol, thr in [("wait", W.Policy(W.WAIT), [1]), ("fcfs", W.Policy(W.FCFS, B=32), None),
                       ("nested", W.Policy(W.NESTED, seg_end=[16]), [1])]:
    s = Scheduler(W.C1, pol, thr)
    out = torch.empty((26, R), dtype=torch.int64, device="cuda")
    run_rows(s, W.C1.seed, 10 ** 6, R, W.C1.horizon_s, out)
    torch.cuda.synchronize()
    ts = []
    for k in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_rows(s, W.C1.seed, k * R, R, W.C1.horizon_s, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    li = s.launch_info()
    print(f"C1 {name:6s} {min(ts):8.2f} ms eng={li.get('engine')} warps/SM={li['blocks_per_sm'] * li['warps_per_block']} smem={li['shared_bytes']}", flush=True)
