# round-2 measurement pass: bench matrix (+ reference arm), C4 strong-scaling sweep, ncu launch list of the
# default bench, ncu --set full of the C2 kernels, C3a Nested and C5 Nested (segment engine)
TAG=${TAG:-r2m}
bash tools/gpu_bench_matrix.sh
timeout 900 python bench.py --workload C4 --total 100000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4strong.json 2>gpurun_out/bench_c4strong.err; echo strong=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 3 -o gpurun_out/prof_$TAG -f python tools/prof_run.py > gpurun_out/prof_$TAG.log 2>&1; echo prof=$?
WL=C3a POLS=nested timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_${TAG}_c3a -f python tools/prof_run.py > gpurun_out/prof_${TAG}_c3a.log 2>&1; echo prof3=$?
WL=C5_55 POLS=nested REPS=2048 HORIZON=600 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_${TAG}_c5 -f python tools/prof_run.py > gpurun_out/prof_${TAG}_c5.log 2>&1; echo prof5=$?
