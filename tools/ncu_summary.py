"""Summarise an ncu --set full report: key metrics per kernel -> markdown + traffic json.

usage: python tools/ncu_summary.py rep.ncu-rep out.md [traffic.json]
"""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
traffic_path = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
idx = {n: i for i, n in enumerate(h)}
want = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__inst_executed.sum", "warp instructions executed"),
    ("sm__inst_issued.avg.per_cycle_active", "IPC (issued / active cycle, max 4)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue-slot utilisation %"),
    ("sm__warps_active.avg.per_cycle_active", "achieved warps / SM"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit: smem (blocks)"),
    ("launch__occupancy_limit_registers", "occupancy limit: registers (blocks)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "SIMT efficiency (threads / inst)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
stall_keys = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
lines = [f"# ncu summary of `{rep}`", ""]
traffic = {}
for r in rows[2:]:
    name = r[idx["Kernel Name"]]
    short = "wait" if "<(int)0" in name or "<0," in name else "nested" if "<(int)1" in name or "<1," in name else "fcfs"
    lines += [f"## {name}", "", "| metric | value |", "|---|---|"]
    for key, label in want:
        if key in idx:
            lines.append(f"| {label} (`{key}`) | {r[idx[key]]} {units[idx[key]]} |")
    st = []
    for k in stall_keys:
        try:
            st.append((float(r[idx[k]]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    lines += ["", "top stall reasons (avg warps stalled per issue-active cycle): " +
              ", ".join(f"{n} {v:.2f}" for v, n in st[:8]), ""]
    def num(key):
        v = float(r[idx[key]].replace(",", ""))
        u = units[idx[key]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    try:
        # one entry per policy: the longest launch (the main launch, not its
        # empty speculative-capacity fallback)
        dur = num("gpu__time_duration.sum")
        if short not in traffic or dur > traffic[short][1]:
            traffic[short] = (num("dram__bytes_read.sum") + num("dram__bytes_write.sum"), dur)
    except (KeyError, ValueError):
        pass
open(out, "w").write("\n".join(lines) + "\n")
if traffic_path:
    json.dump({k: v[0] for k, v in traffic.items()}, open(traffic_path, "w"), indent=1)
print("\n".join(lines))
