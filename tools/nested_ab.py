"""A/B timing of the Nested engines on the bench workloads (CUDA events, best of 3).
env: CONFIGS=engine:capf,... (default seg:1.5,seg:3,member:0)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
from paper_2504_11320_b200 import Scheduler
from paper_2504_11320_b200.sim import run_rows

SEG10 = [50 * k for k in range(1, 11)]
WLS = [("C1", W.C1, [16], [1], 16384, None, {}),
       ("C3a", W.C3A, [20, 40, 80, 160], None, 10000, None, {}),
       ("C3a_tv", W.c3a_time_varying(), [20, 40, 80, 160], [11, 11, 10, 7], 10000, None, {}),
       ("C3b", W.C3B, SEG10, None, 10000, None, {})]
WLS += [(f"C4_{i}", W.c4(i), [100, 200, 300], None, 2000, None, {}) for i in range(5)]
WLS += [("C5", W.c5(55.0), SEG10, None, 2048, float(os.environ.get("C5T", "1818.2")),
         dict(max_resident=4096, restart_cap=2_000_000_000))]
only = os.environ.get("WLS")
for cfg in os.environ.get("CONFIGS", "seg:1.5,seg:3,member:0").split(","):
    eng, capf = cfg.split(":")
    os.environ["WAITSIM_ENGINE"] = eng
    os.environ["WAITSIM_SEG_CAP"] = capf
    for name, wl, seg, thr, R, T, kw in WLS:
        if only and name not in only.split(","):
            continue
        kw = dict(kw)
        if eng == "seg" and "max_resident" in kw and os.environ.get("SEGMAXRES") == "0":
            kw.pop("max_resident")
        s = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg), thr, **kw)
        if thr is None:
            s.thresholds()
        T = wl.horizon_s if T is None else T
        out = torch.empty((26, R), dtype=torch.int64, device="cuda")
        run_rows(s, wl.seed, 10 ** 6, R, T, out)
        torch.cuda.synchronize()
        ts = []
        for k in range(2 if name == "C5" else 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run_rows(s, wl.seed, k * R, R, T, out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        bad = int((out[23] != 0).sum())
        info = s.launch_info()
        s.close()
        rs = int(out[7].sum())
        print(f"{cfg:10s} {name:7s} {min(ts):10.2f} ms  {rs / min(ts) / 1e6:8.3e} req-steps/s  status!=0 {bad:4d}  "
              f"eng {info['engine']} warps/SM {info['blocks_per_sm'] * info['warps_per_block']} "
              f"spec {info['spec_resident']} smem/blk {info['shared_bytes']}", flush=True)
