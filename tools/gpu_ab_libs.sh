# A/B timing of library variants: LIBS="a.so b.so", WLS="C2 C4_2"
for lib in ${LIBS}; do for w in ${WLS:-C2}; do echo "== $lib $w"; LIB=$lib WL=$w timeout 300 python tools/time_run.py 2>&1 | grep -v nested; done; done
