# A/B with custom env per workload: LIBS, then lines of "WL REPS HORIZON POLS"
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log; }
while read wl reps hor pols; do
  [ -z "$wl" ] && continue
  for name in ${LIBS:-base cur}; do
    lib=paper_2504_11320_b200/libsched_$name.so; [ "$name" = cur ] && lib=paper_2504_11320_b200/libsched.so
    echo "== $name $wl" ; LIB=$lib WL=$wl REPS=$reps HORIZON=$hor POLS=$pols timeout 600 python tools/time_run.py 2>&1 | tail -3
  done
done <<< "$CASES"
