# round-1 tree (abtree/) vs HEAD on the restart-heavy C5 workload
echo "== r1 C5"; (cd abtree && WL=C5 REPS=2048 HORIZON=${H5:-1818} MAXRES=4096 RCAP=1048576 timeout 600 python tools/time_run.py 2>&1 | tail -3)
echo "== r2 C5"; WL=C5 REPS=2048 HORIZON=${H5:-1818} MAXRES=4096 RCAP=2000000000 timeout 600 python tools/time_run.py 2>&1 | tail -3
echo "== r2 C5 member"; WAITSIM_ENGINE=member WL=C5 REPS=2048 HORIZON=${H5:-1818} MAXRES=4096 RCAP=2000000000 timeout 600 python tools/time_run.py 2>&1 | tail -3
