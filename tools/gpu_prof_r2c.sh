WL=C4_4 WAITSIM_ENGINE=member timeout 300 python tools/time_run.py 2>&1 | grep wait
WL=C4_4 POLS=wait REPS=2000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/prof_r2c_c4w -f python tools/prof_run.py > gpurun_out/prof_r2c_c4w.log 2>&1; echo prof1=$?
