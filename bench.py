"""Benchmark of the hot path: batched WAIT / FCFS simulation of config C2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one pass of the whole path over one batch of synthetic input:
`sched_run` of R replications of config C2 (BASELINE.json configs[1]: two
prompt types at the paper's low-demand lengths/rates, M = 7B KV budget)
under WAIT (fluid-integer thresholds from `sched_thresholds`) AND under
FCFS (B = 1024), then the per-policy aggregate and its single NCCL
all-reduce.  Every step simulates fresh global replication indices.
Weak scaling: every rank runs R replications per step.
Metric (BASELINE.json): simulated request-steps per second, whole job.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated request-steps/sec (1/2/4/8 B200) + HBM GB/s vs peak; oracle ×speedup"
UNIT = "request-steps/s"
# algorithmic integer lane-ops per unit: request-step,
# arrival (generated at visibility and again at admission), batch
OPS_PER_REQUEST_STEP = 8
OPS_PER_ARRIVAL = 400
OPS_PER_BATCH = 100


def workload_desc(wl, reps):
    return {"workload": "C2: 2 prompt types (l,l',lambda)=(10,10,1000/s),(10,20,1000/s); "
                        "M=131072 tokens; d0=12ms, d1=0.35us/token; T=10 s; WAIT fluid-integer "
                        "thresholds + FCFS(vLLM new-first, B=1024)",
            "replications_per_gpu_per_step": reps, "horizon_s": wl.horizon_s,
            "policies": ["wait", "fcfs"]}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(wl, policies, reps, threads, min_wall=1.5, max_reps=1 << 15):
    """The oracle as it stands on the host cores, on a bounded sample: the
    replication count doubles until one pass takes >= min_wall seconds
    (>= 10-30 s of CPU work on a multi-core host).  Returns (rate, wall,
    request_steps, reps)."""
    import oracle
    while True:
        t0 = time.perf_counter()
        steps = 0
        for pol, thr in policies:
            rows = oracle.run(wl, pol, thr, n_reps=reps, rep_begin=0, n_threads=threads)
            steps += int(rows[oracle.F["request_steps"]].sum())
        dt = time.perf_counter() - t0
        if dt >= min_wall or reps >= max_reps:
            return steps / dt, dt, steps, reps
        reps *= 2


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm."""
    rank, world, _ = (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), 0)
    if rank != 0:
        return
    import workloads as W
    from oracle import fluid as fl
    wl = W.C2
    pols = [(W.Policy(W.WAIT), fl.wait_fluid_integer(wl)), (W.Policy(W.FCFS, B=1024), [0])]
    threads = os.cpu_count() or 1
    per_step = args.ref_reps
    import oracle
    for _ in range(args.warmup):
        oracle.run(wl, pols[0][0], pols[0][1], n_reps=min(per_step, threads), n_threads=threads)
    tot_steps, tot_t = 0, 0.0
    for k in range(args.steps):
        t0 = time.perf_counter()
        for pol, thr in pols:
            rows = oracle.run(wl, pol, thr, n_reps=per_step, rep_begin=k * per_step, n_threads=threads)
            tot_steps += int(rows[oracle.F["request_steps"]].sum())
        tot_t += time.perf_counter() - t0
    v = tot_steps / tot_t
    cfg = workload_desc(wl, per_step)
    cfg["sample"] = f"{per_step} replications per policy per step (bounded sample of C2)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded Philox Poisson traces)", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": cfg["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--reps", type=int, default=10_000)
    ap.add_argument("--ref-reps", type=int, default=64)
    ap.add_argument("--cpu-reps", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import workloads as W
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200.sim import AGG_INT, aggregate, run_rows

    rank, world, local = D.init()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    wl = W.C2
    R = args.reps
    s_wait = Scheduler(wl, W.Policy(W.WAIT), device=local)
    thr_rep = s_wait.thresholds()           # product's own setup (sched_thresholds)
    s_fcfs = Scheduler(wl, W.Policy(W.FCFS, B=1024), device=local)
    scheds = [("wait", s_wait), ("fcfs", s_fcfs)]
    rows = {n: torch.empty((len(__import__("paper_2504_11320_b200").FIELDS), R), dtype=torch.int64,
                           device=dev) for n, _ in scheds}
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device=dev)  # > 126 MB L2

    def step(k, evs=None):
        begin, n = D.rep_range(k, rank, world, R)
        aggs = []
        for i, (name, s) in enumerate(scheds):
            if evs is not None:
                evs[i].record(stream)
            run_rows(s, wl.seed, begin, n, wl.horizon_s, rows[name], stream)
            aggs.append(aggregate(rows[name], wl.horizon_s))
        if evs is not None:
            evs[len(scheds)].record(stream)
        packed = {"int": torch.cat([a["int"] for a in aggs]), "f64": torch.cat([a["f64"] for a in aggs])}
        return D.allreduce_aggregates(packed)  # S7: the one collective

    for k in range(args.warmup):
        step(10_000 + k)
    torch.cuda.synchronize()
    D.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_step, t_kern = [], {n: [] for n, _ in scheds}
    tot_int = None
    units = {n: {"request_steps": 0, "arrivals": 0, "batches": 0, "completed": 0} for n, _ in scheds}
    F_ = __import__("paper_2504_11320_b200").F
    for k in range(args.steps):
        flush.zero_()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(scheds) + 2)]
        agg = step(k, evs[:len(scheds) + 1])
        evs[-1].record(stream)
        torch.cuda.synchronize()
        t_step.append(evs[0].elapsed_time(evs[-1]) / 1e3)
        for i, (n, _) in enumerate(scheds):
            t_kern[n].append(evs[i].elapsed_time(evs[i + 1]) / 1e3)
            r = rows[n]
            for u in units[n]:
                units[n][u] += int(r[F_[u]].sum().item())
        tot_int = agg["int"] if tot_int is None else tot_int + agg["int"]
    torch.cuda.synchronize()
    D.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed = D.max_over_ranks(sum(t_step), dev)
    nI = len(AGG_INT)
    rs_idx = AGG_INT.index("request_steps")
    total_rs = int(sum(tot_int[i * nI + rs_idx].item() for i in range(len(scheds))))
    total_b = int(sum(tot_int[i * nI + AGG_INT.index("batches")].item() for i in range(len(scheds))))
    total_c = int(sum(tot_int[i * nI + AGG_INT.index("completed")].item() for i in range(len(scheds))))
    bad = int(sum(tot_int[i * nI + AGG_INT.index("status")].item() for i in range(len(scheds))))
    if bad:
        raise SystemExit(f"{bad} replications reported a capacity status != 0: not a valid run")
    value = total_rs / elapsed

    # e2e: the same metric through the host-buffer C-ABI call (D2H inside)
    out_host = {n: np.zeros((len(F_), R), dtype=np.uint64) for n, _ in scheds}
    torch.cuda.synchronize()
    D.barrier()
    t0 = time.perf_counter()
    e2e_rs = 0
    for k in range(args.steps):
        begin, n = D.rep_range(100 + k, rank, world, R)
        for name, s in scheds:
            s.run_host(wl.seed, begin, n, wl.horizon_s, out_host[name], stream.cuda_stream)
            e2e_rs += int(out_host[name][F_["request_steps"]].sum())
    e2e_t = D.max_over_ranks(time.perf_counter() - t0, dev)
    e2e_tot = torch.tensor([float(e2e_rs)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_tot)
    e2e_value = float(e2e_tot.item()) / e2e_t

    # roofline of the dominant kernel (alu/issue bound)
    dom = max(t_kern, key=lambda n: sum(t_kern[n]))
    u = units[dom]
    ops_per_launch = (OPS_PER_REQUEST_STEP * u["request_steps"] + OPS_PER_ARRIVAL * u["arrivals"]
                      + OPS_PER_BATCH * u["batches"]) / args.steps
    dur = sum(t_kern[dom]) / len(t_kern[dom])
    props = torch.cuda.get_device_properties(dev)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    sm_max = 1965.0
    if os.path.exists(peaks_path):
        sm_max = json.load(open(peaks_path)).get("sm_max_mhz", sm_max)
    peak_ops = props.multi_processor_count * 4 * 32 * sm_max * 1e6 / 1e12  # Tops/s
    achieved = ops_per_launch / dur / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded counter-based Philox Poisson traces, generated in-kernel)",
        "config": dict(workload_desc(wl, R), parallelism=f"dp{world} (replication sharding)",
                       l2="256 MiB buffer written between timed steps (L2 flush)",
                       wait_thresholds=thr_rep["thresholds"]),
        "batch_steps_per_s": total_b / elapsed, "requests_per_s": total_c / elapsed,
        "status_errors": bad,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": len(F_) * R * 8 * len(scheds),
                "note": "sched_run_host: launch + D2H of the metric rows + sync; inputs are seeds "
                        "(kernel arguments) so no H2D input bytes"},
        "gpu_launches": len(scheds) * args.steps,
        "roofline": {"bound": "alu", "kernel": f"sim_kernel<{dom}>", "achieved": achieved,
                     "peak": peak_ops, "unit": "Tops/s", "frac": achieved / peak_ops,
                     "traffic": traffic,
                     "ops_model": f"{OPS_PER_REQUEST_STEP}/request-step + {OPS_PER_ARRIVAL}/arrival "
                                  f"+ {OPS_PER_BATCH}/batch (integer lane-ops)",
                     "peak_basis": f"{props.multi_processor_count} SMs x 4 warp-instr/clk x 32 lanes x "
                                   f"{sm_max:.0f} MHz (MEASURED_PEAKS sm_max)"},
        "kernel_ms": {n: 1e3 * sum(v) / len(v) for n, v in t_kern.items()},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import workloads as W2
        from oracle import fluid as fl
        threads = os.cpu_count() or 1
        pols = [(W2.Policy(W2.WAIT), fl.wait_fluid_integer(wl)), (W2.Policy(W2.FCFS, B=1024), [0])]
        v, dt, n, nr = cpu_baseline(wl, pols, args.cpu_reps, threads)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": f"C2 full horizon, {nr} replications x 2 policies "
                                          f"({n} request-steps, {dt:.2f} s wall on {threads} threads)"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
