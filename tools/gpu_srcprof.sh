# source-level ncu capture of the C2 WAIT and FCFS launches (one each)
TAG=${TAG:-r1e}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c ${NK:-2} -o gpurun_out/prof_$TAG -f python tools/prof_run.py > gpurun_out/prof_$TAG.log 2>&1; echo prof=$?
tail -3 gpurun_out/prof_$TAG.log
