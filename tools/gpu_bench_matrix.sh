# bench line for every workload (1 GPU) -> gpurun_out/bench_matrix.jsonl
rm -f gpurun_out/bench_matrix.jsonl gpurun_out/bench_matrix.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2>> gpurun_out/bench_matrix.err
cat gpurun_out/bench_default.json >> gpurun_out/bench_matrix.jsonl
for w in C1 C3a C3a_tv C3b C4; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 >> gpurun_out/bench_matrix.jsonl 2>> gpurun_out/bench_matrix.err
done
timeout 1500 python bench.py --workload C5 --steps 2 --warmup 3 --cpu-reps 16 >> gpurun_out/bench_matrix.jsonl 2>> gpurun_out/bench_matrix.err
timeout 600 python bench.py --workload walks --steps 5 --warmup 2 >> gpurun_out/bench_matrix.jsonl 2>> gpurun_out/bench_matrix.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench_matrix.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_matrix.jsonl"):
    d = json.loads(l)
    print(d["config"].get("name", d["config"].get("workload")), f"{d['value']:.3e}", f"ms/step={d['ms_per_step']:.1f}", "frac=%.4f" % d["roofline"]["frac"],
          "cpu=%.2e" % d.get("cpu_baseline", {}).get("value", 0), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
cut -c1-300 gpurun_out/bench_reference.json
tail -5 gpurun_out/bench_matrix.err
