# round-2 checks: parity suite, default bench, self-spawned 2-rank bench, C4 strong scaling
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench=$?
cut -c1-400 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 600 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/bench_n2.json 2>gpurun_out/bench_n2.err; echo bench2=$?
cut -c1-300 gpurun_out/bench_n2.json; grep -E "dist|bench" gpurun_out/bench_n2.err | head
timeout 900 python bench.py --workload C4 --total ${TOTAL:-20000} --steps 1 --warmup 3 > gpurun_out/bench_c4strong.json 2>gpurun_out/bench_c4strong.err; echo strong=$?
cut -c1-300 gpurun_out/bench_c4strong.json; tail -3 gpurun_out/bench_c4strong.err
