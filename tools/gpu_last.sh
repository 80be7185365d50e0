# last pass of the session: default bench (+ reference arm), C3a / C4 lines, ncu of the C2 kernels
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2>/dev/null; echo bench=$?
for w in C3a C4 C1; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2>/dev/null; echo $w=$?; done
TAG=r2e bash tools/gpu_ncu_c2.sh
