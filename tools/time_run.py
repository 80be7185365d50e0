"""Quick timing of one config/policy set (CUDA events), for A/B experiments.
env: WL=C2|C3a|C4_<i>|C5_55 ; REPS ; HORIZON ; LIB=path to alternate libsched.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
import paper_2504_11320_b200._lib as L
if os.environ.get("LIB"):
    L.LIB_PATH = os.environ["LIB"]
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

wl_name = os.environ.get("WL", "C2")
seg10 = [50 * k for k in range(1, 11)]
if wl_name == "C2":
    wl, pols = W.C2, [W.Policy(W.WAIT), W.Policy(W.FCFS, B=1024)]
elif wl_name == "C1":
    wl, pols = W.C1, [W.Policy(W.WAIT), W.Policy(W.FCFS, B=32), W.Policy(W.NESTED, seg_end=[16], thresholds=[1])]
elif wl_name == "C3a":
    wl, pols = W.C3A, [W.Policy(W.NESTED, seg_end=[20, 40, 80, 160]), W.Policy(W.FCFS, B=1024)]
elif wl_name == "C3a_tv":
    wl, pols = W.c3a_time_varying(), [W.Policy(W.NESTED, seg_end=[20, 40, 80, 160], thresholds=[11, 11, 10, 7]),
                                      W.Policy(W.FCFS, B=1024)]
elif wl_name.startswith("C4_"):
    wl = W.c4(int(wl_name[3:]))
    pols = [W.Policy(W.WAIT), W.Policy(W.NESTED, seg_end=[100, 200, 300]), W.Policy(W.FCFS, B=1024)]
elif wl_name == "C3b":
    wl, pols = W.C3B, [W.Policy(W.NESTED, seg_end=seg10), W.Policy(W.FCFS, B=2048)]
else:
    wl, pols = W.c5(55.0), [W.Policy(W.NESTED, seg_end=seg10), W.Policy(W.FCFS, B=1024)]
R = int(os.environ.get("REPS", "10000"))
T = float(os.environ.get("HORIZON", str(wl.horizon_s)))
for pol in pols:
    kw = dict(max_resident=4096, restart_cap=2_000_000_000) if wl_name.startswith("C5") else {}  # as bench.py
    if os.environ.get("POLS") and W.POLICY_NAMES[pol.kind] not in os.environ["POLS"].split(","):
        continue
    if os.environ.get("RCAP"):
        kw["restart_cap"] = int(os.environ["RCAP"])
    if os.environ.get("SPEC"):
        kw["spec_resident"] = int(os.environ["SPEC"])
    if os.environ.get("MAXRES"):
        kw["max_resident"] = int(os.environ["MAXRES"])
    s = Scheduler(wl, pol, pol.thresholds, **kw)
    if pol.kind != W.FCFS and not pol.thresholds:
        s.thresholds()
    out = torch.empty((L.NF, R), dtype=torch.int64, device="cuda")
    run_rows(s, wl.seed, 10**6, R, T, out)  # warm-up
    torch.cuda.synchronize()
    ts = []
    for k in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_rows(s, wl.seed, k * R, R, T, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rs = int(out[L.F["request_steps"]].sum())
    st = int((out[L.F["status"]] != 0).sum())
    li = s.launch_info()
    print(f"{wl_name} {W.POLICY_NAMES[pol.kind]:6s} ms={min(ts):8.3f} rs/s={rs/min(ts)*1e3:.3e} status!=0:{st} "
          f"wpb={li['warps_per_block']} bps={li['blocks_per_sm']} spec={li['spec_resident']} safe={li['max_resident']} "
          f"smem={li['shared_bytes']} fb={li['fallback_grid']} eng={li.get('engine', 0)} retries={li.get('last_retries', -1)}")
