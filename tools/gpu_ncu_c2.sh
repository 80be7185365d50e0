# ncu launch list of the default bench + ncu --set full of the two C2 kernels (TAG)
TAG=${TAG:-r2d}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 3 -o gpurun_out/prof_$TAG -f python tools/prof_run.py > gpurun_out/prof_$TAG.log 2>&1; echo prof=$?
