python - <<'PY' > gpurun_out/zeta.json
import json
from paper_2504_11320_b200 import studies
res = {"strict": studies.zeta_sweep(zetas=(1, 2, 4, 8, 16, 32), reps=4096, slack=True),
       "equality": studies.zeta_sweep(zetas=(1, 2, 4, 8, 16, 32), reps=4096, slack=False)}
print(json.dumps(res))
PY
echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/zeta.json'))
for k,rows in d.items():
    print(k)
    for r in rows: print('  zeta=%3d gap=%.4f+-%.4f lat=%.4f ttft=%.4f evict=%d slack=%.2e thr=%s' % (r['zeta'], r['gap'], r['gap_se'], r['latency'], r['ttft'], r['evictions'], r['slack'], r['thresholds']))
"
timeout 600 python -m pytest tests/test_segment_study.py -m gpu -q 2>&1 | tail -2
