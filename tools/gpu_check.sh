timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
rm -f gpurun_out/ab.log
for wl in C2 C3a C4_2 C3b; do WL=$wl timeout 300 python tools/time_run.py; done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
