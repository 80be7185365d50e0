# source-level ncu of C2 FCFS and C4 rho=0.95 WAIT (ring engine v2) + row stats
python - <<'PY' > gpurun_out/c4stats.log 2>&1
import sys; sys.path.insert(0, '.')
import numpy as np, workloads as W, oracle
from paper_2504_11320_b200 import Scheduler
for i in (2, 4):
    for eng in ("ring", "member"):
        import os; os.environ["WAITSIM_ENGINE"] = eng
        s = Scheduler(W.c4(i), W.Policy(W.WAIT)); s.thresholds()
        r = s.run_host(W.c4(i).seed, 0, 512, 20.0)
        f = lambda k: r[oracle.F[k]].astype(np.float64).mean()
        print(i, eng, s.launch_info()["engine"], "batches", f("batches"), "evict", f("evictions"), "rs", f("request_steps"), "arr", f("arrivals"), "status", int((r[oracle.F["status"]]!=0).sum()))
        s.close()
PY
WL=C4_4 POLS=wait REPS=2000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_r2b_c4w -f python tools/prof_run.py > gpurun_out/prof_r2b_c4w.log 2>&1; echo prof1=$?
WL=C2 POLS=fcfs timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_r2b_c2f -f python tools/prof_run.py > gpurun_out/prof_r2b_c2f.log 2>&1; echo prof2=$?
