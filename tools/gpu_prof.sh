set -x
ncu --version | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 2 -o gpurun_out/prof_r1 -f python tools/prof_run.py > gpurun_out/prof.log 2>&1; echo prof=$?
tail -5 gpurun_out/prof.log
