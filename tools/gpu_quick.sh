# quick check: GPU parity suite (stop at first failure) + C2 / C4 timing
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
for w in ${WLS:-C2 C4_2 C4_4}; do WL=$w timeout 300 python tools/time_run.py; done
