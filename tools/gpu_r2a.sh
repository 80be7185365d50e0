# round-2 pass A: parity suite on the fixed build, source-level ncu of C2 (WAIT, FCFS) and C3a Nested
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
TAG=r2a_c2 NK=2 bash tools/gpu_srcprof.sh
WL=C3a POLS=nested timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_r2a_c3a -f python tools/prof_run.py > gpurun_out/prof_r2a_c3a.log 2>&1; echo prof3=$?
