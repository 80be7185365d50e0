# end-of-session pass: parity suite + smoke, bench matrix (+ reference arm), C4 strong, --gpus 2
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
bash tools/gpu_bench_matrix.sh
timeout 900 python bench.py --workload C4 --total 100000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4strong.json 2>gpurun_out/bench_c4strong.err; echo strong=$?
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_gpus2.json 2> gpurun_out/bench_gpus2.err; echo gpus2=$?
