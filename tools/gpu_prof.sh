TAG=${TAG:-r1d}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 2 -o gpurun_out/prof_$TAG -f python tools/prof_run.py > gpurun_out/prof_$TAG.log 2>&1; echo prof=$?
timeout 600 ncu --set full --clock-control none -k regex:walk_kernel -c 1 -o gpurun_out/prof_walks_$TAG -f python bench.py --workload walks --steps 1 --warmup 0 --reps 262144 > gpurun_out/prof_walks_$TAG.log 2>&1; echo profw=$?
