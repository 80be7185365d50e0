for lib in paper_2504_11320_b200/libsched_mb1.so paper_2504_11320_b200/libsched_mb3.so; do
  echo "== $lib" >> gpurun_out/ab.log
  for wl in C2 C3a C4_2; do LIB=$lib WL=$wl timeout 300 python tools/time_run.py; done >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
