"""C2 WAIT + FCFS: serial vs concurrent streams (launch order), CUDA-event timed, for the tail experiment
(measured r2: serial 30.5 ms, concurrent 31.4 ms, a fused two-policy persistent launch with one work queue
31.8-32.2 ms -- removed again).
env: WL (C2), REPS (10000), WAITSIM_CARVEOUT"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
import paper_2504_11320_b200._lib as L
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

wl = W.C2
R = int(os.environ.get("REPS", "10000"))
hs = {"wait": Scheduler(wl, W.Policy(W.WAIT), None), "fcfs": Scheduler(wl, W.Policy(W.FCFS, B=1024), None)}
hs["wait"].thresholds()
out = {k: torch.empty((L.NF, R), dtype=torch.int64, device="cuda") for k in hs}
st = {k: torch.cuda.Stream() for k in hs}
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")


def go(order, conc, k):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for name in order:
        s = st[name] if conc else cur
        s.wait_event(a)
        run_rows(hs[name], wl.seed, k * R, R, wl.horizon_s, out[name], s)
        e = torch.cuda.Event()
        e.record(s)
        cur.wait_event(e)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for order, conc in [(("wait", "fcfs"), False), (("fcfs", "wait"), False), (("wait", "fcfs"), "concurrent"),
                    (("fcfs", "wait"), "concurrent")]:
    go(order, conc, 100)
    ts = [go(order, conc, k) for k in range(5)]
    rs = sum(int(out[n][L.F["request_steps"]].sum()) for n in hs)
    print(f"carveout={os.environ.get('WAITSIM_CARVEOUT', '-')} {'->'.join(order)} {conc or 'serial'}"
          f" ms={min(ts):.3f} med={sorted(ts)[2]:.3f} rs/s={rs / min(ts) * 1e3:.3e}")
