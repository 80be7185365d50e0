timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload walks --steps 3 --warmup 2 > gpurun_out/bench_walks.json 2>gpurun_out/bench_walks.err; echo walks=$?
cut -c1-900 gpurun_out/bench_walks.json; tail -3 gpurun_out/bench_walks.err
