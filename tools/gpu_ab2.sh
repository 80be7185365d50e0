for i in 1 2; do
LIB=paper_2504_11320_b200/libsched_prev.so WL=C2 python tools/time_run.py
WL=C2 python tools/time_run.py
done
