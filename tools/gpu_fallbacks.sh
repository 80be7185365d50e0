# launch list per workload: fallback launches (second sim_kernel of a policy) that take real time
for w in C2 C1 C3a C3a_tv C3b C4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sim_kernel --csv --log-file gpurun_out/fb_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo $w=$?
done
