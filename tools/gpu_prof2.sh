# ncu details (no source) of one policy under both engines: WL, POLS
for eng in member ring; do
WAITSIM_ENGINE=$eng timeout 900 ncu --section SpeedOfLight --section Occupancy --section WarpStateStats --section LaunchStats --metrics smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active --clock-control none -k regex:sim_kernel -c 1 -o gpurun_out/p2_$eng -f python tools/prof_run.py > gpurun_out/p2_$eng.log 2>&1; echo $eng=$?
done
