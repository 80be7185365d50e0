"""Write the round's profiles/ summaries from a measurement pass (tools/gpu_measure_r2.sh).
usage: python tools/write_profiles.py TAG [ROUND_PREFIX=r2]"""
import collections
import csv
import json
import shutil
import subprocess
import sys

tag = sys.argv[1]
R = sys.argv[2] if len(sys.argv) > 2 else "r2"
G = "gpurun_out/"
# bench matrix
lines = [json.loads(l) for l in open(G + "bench_matrix.jsonl")]
shutil.copy(G + "bench_matrix.jsonl", f"profiles/{R}_bench_matrix.jsonl")
shutil.copy(G + "bench_reference.json", f"profiles/{R}_bench_reference.json")
shutil.copy(G + "bench_default.json", f"profiles/{R}_bench_c2_default.json")
ref = json.loads(open(G + "bench_reference.json").read().strip().splitlines()[-1])
out = [f"# {R} bench matrix (1 B200, `python bench.py --workload W`)", "",
       "Weak scaling, L2 flushed (256 MiB write) between timed steps; launches that each fill the GPU for >= 2 "
       "waves run back to back, others concurrently on separate streams; clocks 1965 MHz with no throttle "
       "reason on every line; `cpu` = the CPU oracle on the box's 16 host threads (bounded sample, "
       "`cpu_baseline`). Raw JSON lines: `%s_bench_matrix.jsonl`; reference arm (the oracle, C2): "
       "`%s_bench_reference.json` (%.2e request-steps/s)." % (R, R, ref["value"]), "",
       "| workload | value | unit | ms/step | e2e | roofline frac (alu, dominant launch alone) | dominant | "
       "per-launch ms | cpu oracle | GPU/CPU |", "|---|---|---|---|---|---|---|---|---|---|"]
for d in lines:
    name = d["config"].get("name", d["config"].get("workload"))
    cpu = d.get("cpu_baseline", {}).get("value", 0)
    km = ", ".join(f"{k} {v:.1f}" for k, v in (d.get("kernel_ms") or {}).items())
    out.append(f"| {name} | {d['value']:.3e} | {d['unit']} | {d['ms_per_step']:.1f} | {d['e2e']['value']:.3e} | "
               f"{d['roofline']['frac']:.4f} | {d['roofline'].get('kernel')} | {km} | {cpu:.2e} | "
               f"{(d['value'] / cpu if cpu else 0):.0f}x |")
open(f"profiles/{R}_bench_matrix.md", "w").write("\n".join(out) + "\n")
# launch list
rows = list(csv.reader(open(G + f"launches_{tag}.csv")))
h, agg, n = None, collections.OrderedDict(), collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k, v, u = d["Kernel Name"], float(d["Metric Value"]), d["Metric Unit"]
    v = v / 1e6 if u == "ns" else (v / 1e3 if u in ("us", "usecond") else v)
    agg[k] = agg.get(k, 0) + v
    n[k] += 1
tot = sum(agg.values())
o = [f"# ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (C2), {R}", "",
     "(cold-cache, serialised under ncu: compare shares, not absolutes; `sim_kernel<P, TRACE, RING, SEG>`: "
     "0 WAIT, 1 NESTED, 2 FCFS; RING=1 class-ring engine, SEG=1 segment engine; each FCFS step also has its "
     "speculative-capacity fallback launch, empty unless a replication overflowed)", "", "| share | total ms | launches | kernel |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    o.append(f"| {100 * v / tot:.2f}% | {v:.3f} | {n[k]} | `{k[:90]}` |")
open(f"profiles/{R}_launches_bench.md", "w").write("\n".join(o) + "\n")
shutil.copy(G + f"launches_{tag}.csv", f"profiles/{R}_launches_bench.csv")
# ncu full summary + traffic
subprocess.check_call([sys.executable, "tools/ncu_summary.py", G + f"prof_{tag}.ncu-rep", "/tmp/ncu_sum.md",
                       "/tmp/traffic.json"])
txt = open("/tmp/ncu_sum.md").read().splitlines()
txt[0] = (f"# ncu --set full summary, C2 bench launches (class-ring engine: sim_kernel<0,0,1,0> WAIT, "
          f"sim_kernel<2,0,1,0> FCFS + its empty fallback launch), {R} (`{G}prof_{tag}.ncu-rep`)")
open(f"profiles/{R}_ncu_full_c2.md", "w").write("\n".join(txt) + "\n")
t = json.load(open("profiles/traffic.json"))
new = json.load(open("/tmp/traffic.json"))
t["C2:wait"], t["C2:fcfs"] = new["wait"], new["fcfs"]
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(out))
