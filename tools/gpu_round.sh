# one round measurement pass on a fresh checkout: parity suite + smoke, then tools/gpu_measure_r2.sh (TAG)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
bash tools/gpu_measure_r2.sh
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_gpus2.json 2> gpurun_out/bench_gpus2.err; echo gpus2=$?
cut -c1-400 gpurun_out/bench_gpus2.json
