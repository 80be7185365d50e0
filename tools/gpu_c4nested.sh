# Nested speculative-capacity A/B over the memory regimes (C4 rho sweep, C3a, C5 short)
for n in base cur; do lib=paper_2504_11320_b200/libsched_$n.so; [ $n = cur ] && lib=paper_2504_11320_b200/libsched.so
  for i in 0 2 3 4; do echo "== $n C4_$i"; LIB=$lib WL=C4_$i REPS=2000 timeout 300 python tools/time_run.py | grep nested; done
  echo "== $n C3a"; LIB=$lib WL=C3a timeout 300 python tools/time_run.py | grep nested
  echo "== $n C5"; RCAP=1048576 MAXRES=4096 REPS=2048 HORIZON=1500 LIB=$lib WL=C5_55 timeout 600 python tools/time_run.py | grep nested
done
