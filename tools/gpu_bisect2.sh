for lib in paper_2504_11320_b200/libsched.so paper_2504_11320_b200/libsched_s11.so; do echo "== $lib"; LIB=$lib WL=C4_4 timeout 300 python tools/time_run.py | grep wait; done
