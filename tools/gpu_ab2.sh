timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for wl in C2 C3a C4_2; do
LIB=$PWD/paper_2504_11320_b200/libsched_prev.so WL=$wl python tools/time_run.py 2>&1 | sed 's/^/prev /' | tail -4
WL=$wl python tools/time_run.py | sed 's/^/new  /'
done
