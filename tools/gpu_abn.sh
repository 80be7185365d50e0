# A/B: parity suite on the current build, then time each library on each workload
# env: LIBS="base new" (paper_2504_11320_b200/libsched_<name>.so; "cur" = libsched.so), WLS="C2 C3a C4_2"
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; }
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/ab.log
for wl in ${WLS:-C2 C3a C4_2}; do
  for name in ${LIBS:-base cur}; do
    lib=paper_2504_11320_b200/libsched_$name.so; [ "$name" = cur ] && lib=paper_2504_11320_b200/libsched.so
    echo "== $name $wl" >> gpurun_out/ab.log
    R=10000; [ "${wl:0:2}" = C5 ] && R=512
    REPS=${REPS:-$R} LIB=$lib WL=$wl timeout 300 python tools/time_run.py >> gpurun_out/ab.log 2>&1
  done
done
cat gpurun_out/ab.log
