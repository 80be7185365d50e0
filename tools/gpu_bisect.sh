for c in $(ls abtree); do echo "== $c"; (cd abtree/$c && WL=C4_4 timeout 300 python tools/time_run.py | grep wait); done
echo "== HEAD"; WL=C4_4 timeout 300 python tools/time_run.py | grep wait
