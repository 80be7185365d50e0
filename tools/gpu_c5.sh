timeout 1500 python bench.py --workload C5 --steps 3 --warmup 3 --reps 2048 --cpu-reps 4 > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err; echo rc=$?
cut -c1-1500 gpurun_out/bench_c5.jsonl; tail -3 gpurun_out/bench_c5.err
