# bench line for every workload (1 GPU) -> gpurun_out/bench_matrix.jsonl
rm -f gpurun_out/bench_matrix.jsonl gpurun_out/bench_matrix.err
for w in C2 C1 C3a C3a_tv C3b C4; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 >> gpurun_out/bench_matrix.jsonl 2>> gpurun_out/bench_matrix.err
done
timeout 1200 python bench.py --workload C5 --steps 3 --warmup 3 --reps 2048 --cpu-reps 8 >> gpurun_out/bench_matrix.jsonl 2>> gpurun_out/bench_matrix.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_matrix.jsonl"):
    d = json.loads(l)
    print(d["config"]["name"], f"{d['value']:.3e}", f"ms/step={d['ms_per_step']:.1f}", "frac=%.3f" % d["roofline"]["frac"],
          "cpu=%.2e" % d.get("cpu_baseline", {}).get("value", 0), d["kernel_ms"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
tail -5 gpurun_out/bench_matrix.err
