"""Benchmark of the hot path: the batched WAIT / Nested WAIT / FCFS simulation.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C2|C1|C3a|C3b|C4|C5|C3a_tv|walks] [--reps R]
    python bench.py --workload C4 --total 100000 [--gpus N]   (strong scaling)

`--gpus N` without a torchrun environment launches the N ranks itself
(torch.distributed.run, one process per GPU; gloo host reduce when the box
has fewer than N GPUs); under torchrun WORLD_SIZE must equal N.

A step = one pass of the whole path over one batch of synthetic input: for
every policy of the workload, one `sched_run` (C ABI) of R replications
(fresh global replication indices every step), the per-policy aggregate,
and the single NCCL all-reduce of the aggregates.  Weak scaling: every rank
runs R replications per policy per step.  The default workload is C2
(BASELINE.json configs[1]: two prompt types at the paper's low-demand
lengths/rates, 7B KV budget, WAIT vs FCFS, 10^4 replications on 1 B200).
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
# arrival (Philox + -ln U + marks + scan share, generated at visibility and
# regenerated at admission in the worst case), batch
OPS_PER_REQUEST_STEP = 8
OPS_PER_ARRIVAL = 400
OPS_PER_BATCH = 100
OPS_PER_EVICTION = 60   # LIFO victim (freed-KV scan share), restart record, FIFO re-rank


class StepIndex:
    """Replication-index steps of one run: timed steps 0..K-1 come first;
    every other launch (warm-up, e2e, solo timing) takes the next unused
    index, so no two launches share replications.  Replication indices are
    (step * world + rank) * R + i and must stay below 2^32 (sched_run)."""

    def __init__(self, steps: int, world: int, per_rank: int):
        self.next, self.world, self.R = steps, world, per_rank
        self.check(steps - 1)

    def check(self, k: int):
        if (k * self.world + self.world) * self.R > 1 << 32:
            raise SystemExit(f"step {k} x {self.world} ranks x {self.R} replications exceeds the 2^32 "
                             f"replication index space")

    def take(self) -> int:
        k = self.next
        self.check(k)
        self.next += 1
        return k


def peaks():
    """(SM max MHz, HBM GB/s, source) from MEASURED_PEAKS.json, else the
    B200_PROFILING.md fallbacks."""
    sm_max, hbm, src = 1965.0, 7700.0, "B200_PROFILING.md nominal (fallback)"
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        d = json.load(open(pp))
        sm_max, hbm = float(d.get("sm_max_mhz", sm_max)), float(d.get("hbm_gbs", hbm))
        src = "MEASURED_PEAKS.json"
    return sm_max, hbm, src


def roofline(u, dur, n_sm, traffic_key, kernel, out_bytes):
    """Issue-slot roofline of one launch: algorithmic integer
    lane-ops of its own metric rows u over its CUDA-event duration, against
    SMs x 4 warp-instr/clk x 32 lanes x max clock.  `frac` counts each
    arrival twice (generated at visibility, regenerated at admission),
    `frac_arrival_once` once.  HBM: ncu DRAM bytes of this launch
    (profiles/traffic.json) and the algorithmic bytes (metric rows written)
    over the same duration, against the measured copy bandwidth."""
    sm_max, hbm_peak, src = peaks()
    peak_ops = n_sm * 4 * 32 * sm_max * 1e6 / 1e12  # Tops/s
    base = (OPS_PER_REQUEST_STEP * u["request_steps"] + OPS_PER_BATCH * u["batches"]
            + OPS_PER_EVICTION * u["evictions"])
    ach2 = (base + OPS_PER_ARRIVAL * u["arrivals"]) / dur / 1e12
    ach1 = (base + OPS_PER_ARRIVAL // 2 * u["arrivals"]) / dur / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(traffic_key)
    hbm = {"algorithmic_bytes": out_bytes, "algorithmic_gbs": out_bytes / dur / 1e9,
           "ncu_dram_bytes": traffic, "achieved_gbs": (traffic / dur / 1e9) if traffic else None,
           "peak_gbs": hbm_peak, "frac": (traffic / dur / 1e9 / hbm_peak) if traffic else None,
           "note": "bytes per launch: metric rows written (algorithmic; arrivals are generated in-kernel) and "
                   "ncu dram__bytes_read+write of the same launch (profiles/traffic.json); the path is "
                   "issue/latency bound, not HBM bound (DESIGN.md §5.1)"}
    return {"bound": "alu", "kernel": kernel, "achieved": ach2, "peak": peak_ops, "unit": "Tops/s",
            "frac": ach2 / peak_ops, "frac_arrival_once": ach1 / peak_ops, "traffic": traffic,
            "ops_model": f"{OPS_PER_REQUEST_STEP}/request-step + {OPS_PER_ARRIVAL}/arrival (frac; "
                         f"{OPS_PER_ARRIVAL // 2} in frac_arrival_once) + {OPS_PER_BATCH}/batch + "
                         f"{OPS_PER_EVICTION}/eviction (integer lane-ops, DESIGN.md §5.4)",
            "peak_basis": f"{n_sm} SMs x 4 warp-instr/clk x 32 lanes x {sm_max:.0f} MHz ({src})",
            "hbm": hbm}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def nested_block(dev, rank, world, n_sm, flush, reps=10_000, launches=3):
    """C3a Nested WAIT (strict thresholds from sched_thresholds), 10^4
    replications per launch: request-steps/s, kernel ms and the roofline."""
    import torch
    import paper_2504_11320_b200 as pkg
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200.sim import run_rows
    _, pol, thr, wl = expand("C3a")[0][0]
    s = Scheduler(wl, pol, thr, device=dev.index)
    if thr is None:
        s.thresholds()  # the product's own setup (sched_thresholds) installs them
    rows = torch.empty((pkg.NF, reps), dtype=torch.int64, device=dev)
    st = torch.cuda.Stream(dev)
    run_rows(s, wl.seed, *D.rep_range(0, rank, world, reps), wl.horizon_s, rows, st)  # warm-up
    torch.cuda.synchronize()
    ms, tot_rs = [], 0
    keys = ("request_steps", "arrivals", "batches", "completed", "evictions")
    for k in range(1, launches + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run_rows(s, wl.seed, *D.rep_range(k, rank, world, reps), wl.horizon_s, rows, st)
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        u = {key: int(rows[pkg.F[key]].sum().item()) for key in keys}
        assert int((rows[pkg.F["status"]] != 0).sum().item()) == 0
        tot_rs += u["request_steps"]
    t = D.max_over_ranks(sum(ms) / 1e3, dev)
    roof = roofline(u, ms[-1] / 1e3, n_sm, "C3a:nested", "sim_kernel<nested>", pkg.NF * 8 * reps)
    li = s.launch_info()
    s.close()
    return {"workload": "C3a: Nested WAIT strict thresholds, 4 types l'=(20,40,80,160), rho=0.5, T=60 s",
            "value": D.sum_over_ranks(float(tot_rs), dev) / t, "unit": UNIT,
            "replications_per_launch_per_gpu": reps, "kernel_ms": sum(ms) / len(ms),
            "frac": roof["frac"], "frac_arrival_once": roof["frac_arrival_once"], "traffic": roof["traffic"],
            "engine": li["engine"], "warps_per_sm": li["blocks_per_sm"] * li["warps_per_block"]}


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_spawn(args) -> int:
    """--gpus N with no torchrun environment: launch the N ranks here (one
    process per GPU, torch.distributed.run on 127.0.0.1).  On a box with
    fewer than N GPUs the ranks share them and reduce over gloo on the host
    (WAITSIM_DIST_BACKEND=gloo); the JSON line says so."""
    import torch
    env = dict(os.environ)
    ngpu = torch.cuda.device_count()
    if ngpu < args.gpus:
        env["WAITSIM_DIST_BACKEND"] = "gloo"
        env["WAITSIM_SHARED_GPUS"] = str(ngpu)
        print(f"[bench] {args.gpus} ranks on {ngpu} GPU(s): gloo host reduce", file=sys.stderr, flush=True)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd, env=env)
    if rc:
        raise SystemExit(rc)
    return 0


def registry(name: str):
    """(workload, [(label, Policy, thresholds or None = setup recipe)], reps, text)."""
    import workloads as W
    seg10 = [50 * k for k in range(1, 11)]
    if name == "C2":
        return (W.C2, [("wait", W.Policy(W.WAIT), None), ("fcfs", W.Policy(W.FCFS, B=1024), None)],
                10_000, "C2: 2 prompt types (l,l',lambda)=(10,10,1000/s),(10,20,1000/s); M=131072 tokens; "
                        "d0=12ms, d1=0.35us/token; T=10 s; WAIT fluid-integer thresholds + FCFS(vLLM "
                        "new-first, B=1024)")
    if name == "C1":
        return (W.C1, [("wait", W.Policy(W.WAIT), None), ("fcfs", W.Policy(W.FCFS, B=32), None),
                       ("nested", W.Policy(W.NESTED, seg_end=[16]), [1])],
                16_384, "C1: 1 type (8,16,74/s), M=256, T=27.0 s; WAIT n=1, FCFS B=32, Nested 1 segment")
    if name == "C3a":
        return (W.C3A, [("nested", W.Policy(W.NESTED, seg_end=[20, 40, 80, 160]), None),
                        ("fcfs", W.Policy(W.FCFS, B=1024), None)],
                10_000, "C3a: 4 types l=10, l'=(20,40,80,160), rates 1:2:4:8 (rho=0.5), M=131072, "
                        "T=60 s; Nested WAIT strict thresholds + FCFS B=1024")
    if name == "C3a_tv":
        return (W.c3a_time_varying(), [("nested", W.Policy(W.NESTED, seg_end=[20, 40, 80, 160]),
                                        [11, 11, 10, 7]),
                                       ("fcfs", W.Policy(W.FCFS, B=1024), None)],
                10_000, "C3a with time-varying rates x(0.5,1,1.5,1) over 4x15 s (PAPER.md:1882); "
                        "Nested WAIT (11,11,10,7) + FCFS B=1024")
    if name == "C3b":
        return (W.C3B, [("nested", W.Policy(W.NESTED, seg_end=seg10), None),
                        ("fcfs", W.Policy(W.FCFS, B=2048), None)],
                10_000, "C3b: geometric l' on [1,500], l=60, rho=0.3, M=524288, T=60 s; Nested L=10 + "
                        "FCFS B=2048")
    if name == "C4":
        pols = []
        for i in range(5):
            pols += [(f"wait@{W.C4_RHO[i]}", W.Policy(W.WAIT), None, W.c4(i)),
                     (f"nested@{W.C4_RHO[i]}", W.Policy(W.NESTED, seg_end=[100, 200, 300]), None, W.c4(i)),
                     (f"fcfs@{W.C4_RHO[i]}", W.Policy(W.FCFS, B=1024), None, W.c4(i))]
        return (None, pols, 2_000, "C4: heavy-traffic sweep, 3 types l=20, l'=(100,200,300), rates 3:2:1, "
                                   "rho in {0.5,0.7,0.8,0.9,0.95} x {WAIT, Nested, FCFS}, T=20 s")
    if name == "C5":
        return (W.c5(55.0), [("nested", W.Policy(W.NESTED, seg_end=seg10), None),
                             ("fcfs", W.Policy(W.FCFS, B=1024), None)],
                2_048, "C5: chat-shaped marks (bins 23:11:8:7:6:4:3:2:1:1, prefill mean 60), 10^6 "
                       "arrivals per trace (QPS 55, T=18182 s); Nested L=10 strict thresholds (M^pi > M: "
                       "LIFO-eviction regime) + FCFS B=1024")
    raise SystemExit(f"unknown workload {name}")


# per-workload handle options (capacities sized for the long overloaded C5 traces)
# C5 Nested (strict thresholds, M^pi > M) thrashes: nearly every waiting
# prompt is an evicted restart, ~1e6 per trace by the horizon, so its pool
# holds ~2048 x 1e6 entries at the end (20 B each)
SCHED_KW = {"C5": dict(max_resident=4096, restart_cap=2_000_000_000)}


def expand(name):
    wl, pols, reps, text = registry(name)
    out = []
    for p in pols:
        out.append(p if len(p) == 4 else (p[0], p[1], p[2], wl))
    return out, reps, text


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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


def oracle_thresholds(wl, pol, thr):
    """Thresholds for the oracle legs: the given ones, else the oracle's own recipe."""
    import workloads as W
    from oracle import fluid as fl
    if thr is not None:
        return thr
    if pol.kind == W.WAIT:
        return fl.wait_fluid_integer(wl)
    if pol.kind == W.NESTED:
        return fl.nested_strict(wl, pol.seg_end)
    return [0]


def cpu_baseline(pols, reps, threads, min_wall=1.5, max_reps=1 << 15):
    """The oracle as it stands on the host cores, on a bounded sample: the
    replication count doubles until one pass takes >= min_wall seconds.
    Returns (rate, wall, request_steps, reps per policy)."""
    import oracle
    thr = [oracle_thresholds(wl, pol, t) for _, pol, t, wl in pols]
    while True:
        t0 = time.perf_counter()
        steps = 0
        for (_, pol, _, wl), th in zip(pols, thr):
            rows = oracle.run(wl, pol, th, n_reps=reps, rep_begin=0, n_threads=threads)
            steps += int(rows[oracle.F["request_steps"]].sum())
        dt = time.perf_counter() - t0
        if dt >= min_wall or reps >= max_reps:
            return steps / dt, dt, steps, reps
        reps *= 2


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm."""
    if int(os.environ.get("RANK", 0)) != 0:
        return
    import oracle
    pols, _, text = expand(args.workload)
    thr = [oracle_thresholds(wl, pol, t) for _, pol, t, wl in pols]
    threads = os.cpu_count() or 1
    per_step = args.ref_reps
    for _ in range(args.warmup):
        _, pol, _, wl = pols[0]
        oracle.run(wl, pol, thr[0], n_reps=min(per_step, threads), n_threads=threads)
    tot_steps, tot_t = 0, 0.0
    for k in range(args.steps):
        t0 = time.perf_counter()
        for (_, pol, _, wl), th in zip(pols, thr):
            rows = oracle.run(wl, pol, th, n_reps=per_step, rep_begin=k * per_step, n_threads=threads)
            tot_steps += int(rows[oracle.F["request_steps"]].sum())
        tot_t += time.perf_counter() - t0
    v = tot_steps / tot_t
    sample = f"{per_step} replications per policy per step (bounded sample of {args.workload})"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded Philox Poisson traces)",
        "config": {"workload": text, "name": args.workload, "replications_per_policy_per_step": per_step,
                   "sample": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def bench_walks(args):
    """--workload walks: the appendix random-walk chains (NEXT(4)) through
    sched_walks; metric = simulated walk-steps per second (weak scaling)."""
    import torch
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200._lib import WALK_FIELDS, walks, walks_device
    rank, world, local = D.init()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    N = args.reps or (1 << 20)
    B = 1000
    cases = [dict(kind=0, n=8, mu=8.0), dict(kind=1, n=6, n_prev=10, p=0.5)]
    out = torch.empty((len(WALK_FIELDS), N), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(k):
        for j, c in enumerate(cases):
            walks_device(c["kind"], c["n"], B, N, seed=0x2504113200000011,
                         out_ptr=out.data_ptr(), walk_begin=(k * world + rank) * N,
                         mu=c.get("mu", 0.0), n_prev=c.get("n_prev", 0), p=c.get("p", 0.0),
                         stream_ptr=stream.cuda_stream)

    # warm-up walks use indices after the timed ones (K..K+W-1): walk_begin
    # = (k * world + rank) * N stays small at any world size
    for k in range(args.warmup):
        step(args.steps + k)
    torch.cuda.synchronize()
    D.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for k in range(args.steps):
        step(k)
    b.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clk = clocks.stop()
    el = D.max_over_ranks(a.elapsed_time(b) / 1e3, dev)
    steps_total = world * args.steps * len(cases) * N * B
    value = steps_total / el
    # per walk-step: Philox 10 rounds (~100 lane-ops) + pmf inversion (~4 ops
    # per unit of the mean arrivals + 8) + the chain and coupled updates (~20)
    ops = sum(100 + 8 + 4 * (c.get("mu") or c["n_prev"] * c["p"]) + 20 for c in cases) / len(cases)
    props = torch.cuda.get_device_properties(dev)
    sm_max = 1965.0
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        sm_max = float(json.load(open(pp)).get("sm_max_mhz", sm_max))
    peak = props.multi_processor_count * 128 * sm_max * 1e6 / 1e12
    ach = value * ops / 1e12
    # e2e: the host-buffer call (launch + D2H + sync), after one untimed call,
    # best of three (a single cold call measured host setup, not the path)
    walks(0, 8, B, min(N, 65536), seed=1, mu=8.0, device=local)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        walks(0, 8, B, min(N, 65536), seed=1, mu=8.0, device=local)
        ts.append(time.perf_counter() - t0)
    e2e = min(N, 65536) * B / min(ts)
    line = {"metric": "simulated walk-steps/sec (appendix random-walk chains, NEXT(4))",
            "value": value, "unit": "walk-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic (Philox draws)", "config": {"workload": "walks", "walks_per_case": N,
                                                          "steps_per_walk": B, "cases": cases},
            "e2e": {"value": e2e, "unit": "walk-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": len(WALK_FIELDS) * 8 * min(N, 65536)},
            "gpu_launches": len(cases) * args.steps,
            "roofline": {"bound": "alu", "kernel": "walk_kernel", "achieved": ach, "peak": peak,
                         "unit": "Tops/s", "frac": ach / peak, "traffic": None,
                         "ops_model": f"{ops:.0f} lane-ops per walk-step"},
            "clocks": clk}
    if rank == 0:
        print(json.dumps(line))


def bench_strong(args):
    """--workload C4 --total R: STRONG scaling of the heavy-traffic sweep
    (BASELINE.json configs[3]): 5 rho x {WAIT, Nested,
    FCFS} x R replications per point, a fixed total sharded over the ranks
    (rank g runs the g-th contiguous share of EVERY point, so the 10-100x
    cost spread across rho and policies is split evenly); the 1-GPU run does
    the whole total.  One step = the whole sweep on fresh replication
    indices; value = request-steps of all ranks / max-over-ranks device time."""
    import numpy as np
    import torch

    import paper_2504_11320_b200 as pkg
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200.sim import aggregate, run_rows

    if args.workload != "C4":
        raise SystemExit("--total (strong scaling) is defined for the C4 sweep")
    rank, world, local = D.init()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    pols, _, text = expand("C4")
    R = args.total
    if R < world:
        raise SystemExit("--total must be >= the number of ranks")
    begin0, n = D.shard(R, rank, world)
    scheds = []
    for label, pol, thr, wl in pols:
        s = Scheduler(wl, pol, thr, device=local)
        if thr is None and pol.kind in (pkg.WAIT, pkg.NESTED):
            s.thresholds()  # the product's own setup (sched_thresholds) installs them
        scheds.append((label, s, wl))
    rows = {lb: torch.empty((pkg.NF, max(n, 1)), dtype=torch.int64, device=dev) for lb, _, _ in scheds}
    stream = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(dev) for _ in scheds]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device=dev)
    if (args.steps + args.warmup + 1) * R > 1 << 32:
        raise SystemExit("replication index space (2^32) exceeded")

    def sweep(k, reps, with_agg=True):
        """One sweep: every point's share of replications [k R, (k+1) R)."""
        b, m = D.shard(reps, rank, world)
        st = torch.cuda.Event(enable_timing=True)
        st.record(stream)
        ends = []
        for i, (lb, s, wl) in enumerate(scheds):
            streams[i].wait_event(st)
            if m:
                run_rows(s, wl.seed, k * R + b, m, wl.horizon_s, rows[lb][:, :m], streams[i])
            e = torch.cuda.Event(enable_timing=True)
            e.record(streams[i])
            ends.append(e)
        for e in ends:
            stream.wait_event(e)
        agg = None
        if with_agg:
            aggs = [aggregate(rows[lb][:, :m], wl.horizon_s) for lb, _, wl in scheds]
            agg = D.allreduce_aggregates({"int": torch.cat([a["int"] for a in aggs]),
                                          "f64": torch.cat([a["f64"] for a in aggs])})
        en = torch.cuda.Event(enable_timing=True)
        en.record(stream)
        return st, ends, en, agg, m

    for k in range(args.warmup):  # warm-up sweeps on a small share (code paths, allocations)
        sweep(args.steps + k, min(R, 256 * world), with_agg=False)
    torch.cuda.synchronize()
    D.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_sweep, t_kern, req = [], {lb: [] for lb, _, _ in scheds}, 0
    from paper_2504_11320_b200.sim import AGG_INT
    for k in range(args.steps):
        flush.zero_()
        st, ends, en, agg, m = sweep(k, R)
        torch.cuda.synchronize()
        t_sweep.append(st.elapsed_time(en) / 1e3)
        for (lb, _, _), e in zip(scheds, ends):
            t_kern[lb].append(st.elapsed_time(e) / 1e3)
        if agg is not None:
            ints = agg["int"].view(len(scheds), len(AGG_INT))
            if int(ints[:, AGG_INT.index("status")].sum()):
                raise SystemExit("a replication reported a capacity status != 0: not a valid run")
            req = req + int(ints[:, AGG_INT.index("request_steps")].sum())
    torch.cuda.synchronize()
    D.barrier()
    clk = clocks.stop()
    elapsed = D.max_over_ranks(sum(t_sweep), dev)
    value = req / elapsed
    # e2e: one sweep through the host-buffer C-ABI call (D2H of the rows inside)
    out_host = torch.empty((pkg.NF, max(n, 1)), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    D.barrier()
    t0 = time.perf_counter()
    e2e_rs = 0
    for lb, s, wl in scheds:
        if n:
            s.run_host(wl.seed, (args.steps + args.warmup) * R + begin0, n, wl.horizon_s, out_host,
                       stream.cuda_stream)
            e2e_rs += int(out_host[pkg.F["request_steps"]].sum())
    e2e_t = D.max_over_ranks(time.perf_counter() - t0, dev)
    e2e_value = D.sum_over_ranks(float(e2e_rs), dev) / e2e_t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded counter-based Philox Poisson traces, generated in-kernel)",
        "config": {"workload": text + f"; strong scaling: {R} replications per (rho, policy) point in total, "
                                      f"rank g runs share g of every point", "name": "C4-strong",
                   "replications_per_point_total": R, "points": [lb for lb, _, _ in scheds],
                   "parallelism": f"dp{world} (replication sharding, fixed total)",
                   "l2": "256 MiB buffer written between timed sweeps (L2 flush)",
                   "warmup": f"{args.warmup} sweeps of {min(R, 256 * world)} replications per point"},
        "sweep_s": elapsed / args.steps,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": pkg.NF * 8 * n * len(scheds),
                "note": "one sweep through sched_run_host (launch + D2H of the rows + sync per point)"},
        "gpu_launches": sum(2 + (1 if s.launch_info()["fallback_grid"] else 0) for _, s, _ in scheds) * args.steps,
        "kernel_ms_to_end": {lb: 1e3 * sum(v) / len(v) for lb, v in t_kern.items()},
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line))
    for _, s, _ in scheds:
        s.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--reps", type=int, default=0, help="replications per policy per GPU per step")
    ap.add_argument("--ref-reps", type=int, default=64)
    ap.add_argument("--cpu-reps", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", default="auto", choices=["auto", "serial", "concurrent"],
                    help="policy launches on one stream or one stream each (auto: serial when each fills >= 2 waves)")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3a Nested block of the default line")
    ap.add_argument("--total", type=int, default=0,
                    help="strong scaling (C4): replications per (rho, policy) point, sharded over ranks")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_spawn(args)
    world_env = int(os.environ.get("WORLD_SIZE", 1))
    if world_env != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_env}: one rank per GPU expected")
    if args.workload == "walks":
        return bench_walks(args)
    if args.total:
        return bench_strong(args)

    import numpy as np
    import torch

    import paper_2504_11320_b200 as pkg
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200.sim import AGG_INT, aggregate, run_rows

    rank, world, local = D.init()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    pols, reps_default, text = expand(args.workload)
    R = args.reps or reps_default
    scheds, thr_used = [], {}
    for label, pol, thr, wl in pols:
        s = Scheduler(wl, pol, thr, device=local, **SCHED_KW.get(args.workload, {}))
        if thr is None and pol.kind in (pkg.WAIT, pkg.NESTED):
            thr_used[label] = s.thresholds()["thresholds"]  # product's own setup (sched_thresholds)
        scheds.append((label, s, wl))
    rows = {n: torch.empty((pkg.NF, R), dtype=torch.int64, device=dev) for n, _, _ in scheds}
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device=dev)  # > 126 MB L2
    F_ = pkg.F

    # every policy's launch on its own stream, so independent launches share
    # the GPU (a C4 sweep point alone does not fill 148 SMs); launches that
    # each fill the GPU for >= 2 waves run back to back on one stream instead
    # (concurrent persistent grids only fragment each other's occupancy)
    def waves(s, n):
        li = s.launch_info()
        return n / max(1, li["grid"] * li["warps_per_block"])
    n_local = D.rep_range(0, rank, world, R)[1]
    serial = all(waves(s, n_local) >= 2.0 for _, s, _ in scheds)
    if args.streams != "auto":
        serial = args.streams == "serial"
    pstreams = [torch.cuda.Stream(dev)] * len(scheds) if serial else [torch.cuda.Stream(dev) for _ in scheds]

    def step(k, ev_start=None, ev_ends=None, ev_begins=None):
        begin, n = D.rep_range(k, rank, world, R)
        start = ev_start or torch.cuda.Event()
        start.record(stream)
        ends = ev_ends or [torch.cuda.Event() for _ in scheds]
        for i, (name, s, wl) in enumerate(scheds):
            pstreams[i].wait_event(start)
            if ev_begins:
                ev_begins[i].record(pstreams[i])
            run_rows(s, wl.seed, begin, n, wl.horizon_s, rows[name], pstreams[i])
            ends[i].record(pstreams[i])
        for e in ends:
            stream.wait_event(e)
        aggs = [aggregate(rows[name], wl.horizon_s) for name, _, wl in scheds]
        packed = {"int": torch.cat([a["int"] for a in aggs]), "f64": torch.cat([a["f64"] for a in aggs])}
        return D.allreduce_aggregates(packed)  # S7: the one collective

    # step indices: timed 0..K-1, warm-up K..K+W-1, then the e2e and solo
    # launches; replication indices (step*world + rank)*R + i stay < 2^32
    idx = StepIndex(args.steps, world, R)
    for k in range(args.warmup):
        step(idx.take())
    torch.cuda.synchronize()
    D.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_step, t_kern = [], {n: [] for n, _, _ in scheds}
    tot_int = None
    units = {n: {"request_steps": 0, "arrivals": 0, "batches": 0, "completed": 0, "evictions": 0}
             for n, _, _ in scheds}
    for k in range(args.steps):
        flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in scheds]
        begins = [torch.cuda.Event(enable_timing=True) for _ in scheds]
        ev1 = torch.cuda.Event(enable_timing=True)
        agg = step(k, ev0, ends, begins)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_step.append(ev0.elapsed_time(ev1) / 1e3)
        for i, (n, _, _) in enumerate(scheds):
            t_kern[n].append(begins[i].elapsed_time(ends[i]) / 1e3)  # this launch: begin -> end
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

    def tot(field):
        return int(sum(tot_int[i * nI + AGG_INT.index(field)].item() for i in range(len(scheds))))

    bad = tot("status")
    if bad:
        raise SystemExit(f"{bad} replications reported a capacity status != 0: not a valid run")
    value = tot("request_steps") / elapsed

    # e2e: the same metric through the host-buffer C-ABI call (D2H inside)
    # pinned host rows (the D2H of each step's result lands here)
    out_host = {n: torch.empty((pkg.NF, R), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
                for n, _, _ in scheds}
    for name, s, wl in scheds:  # untimed: the handle's host-path staging buffer is allocated once
        b0, n0 = D.rep_range(idx.take(), rank, world, R)
        s.run_host(wl.seed, b0, n0, wl.horizon_s, out_host[name], stream.cuda_stream)
    torch.cuda.synchronize()
    D.barrier()
    t0 = time.perf_counter()
    e2e_rs = 0
    e2e_steps = max(1, min(args.steps, 3))
    for k in range(e2e_steps):
        begin, n = D.rep_range(idx.take(), rank, world, R)
        for name, s, wl in scheds:
            s.run_host(wl.seed, begin, n, wl.horizon_s, out_host[name], stream.cuda_stream)
            e2e_rs += int(out_host[name][F_["request_steps"]].sum())
    e2e_t = D.max_over_ranks(time.perf_counter() - t0, dev)
    e2e_value = D.sum_over_ranks(float(e2e_rs), dev) / e2e_t

    # roofline of the dominant kernel (alu/issue bound),
    # timed alone (no concurrent launches) on its own stream
    # dominant = the launch with the largest device time in the timed steps
    dom = max(t_kern, key=lambda n: sum(t_kern[n]))
    di = [n for n, _, _ in scheds].index(dom)
    _, s_dom, wl_dom = scheds[di]
    solo = []
    for k in range(3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        begin, n = D.rep_range(idx.take(), rank, world, R)
        a.record(pstreams[di])
        run_rows(s_dom, wl_dom.seed, begin, n, wl_dom.horizon_s, rows[dom], pstreams[di])
        b.record(pstreams[di])
        torch.cuda.synchronize()
        solo.append((a.elapsed_time(b) / 1e3, {u: int(rows[dom][F_[u]].sum().item()) for u in units[dom]}))
    dur, u = solo[-1]
    props = torch.cuda.get_device_properties(dev)
    roof = roofline(u, dur, props.multi_processor_count, f"{args.workload}:{dom}", f"sim_kernel<{dom}>",
                    out_bytes=pkg.NF * 8 * R)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded counter-based Philox Poisson traces, generated in-kernel)",
        "config": {"workload": text, "name": args.workload, "replications_per_policy_per_gpu_per_step": R,
                   "policies": [n for n, _, _ in scheds], "parallelism": f"dp{world} (replication sharding)",
                   "l2": "256 MiB buffer written between timed steps (L2 flush)",
                   "thresholds_from_sched_thresholds": thr_used},
        "batch_steps_per_s": tot("batches") / elapsed, "requests_per_s": tot("completed") / elapsed,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": pkg.NF * R * 8 * len(scheds),
                "note": "sched_run_host: launch + D2H of the metric rows + sync; the step's inputs are "
                        "seeds and replication indices (kernel arguments), so no H2D input bytes"},
        # per policy and step: the simulation, its fallback launch (if any), sched_aggregate
        "gpu_launches": sum(2 + (1 if s.launch_info()["fallback_grid"] else 0) for _, s, _ in scheds)
        * args.steps,
        "roofline": roof,
        "hbm": roof.pop("hbm"),
        "kernel_ms": {n: 1e3 * sum(v) / len(v) for n, v in t_kern.items()},
        "kernel_ms_note": "per policy: that launch's begin -> end (" + (
            "launches run back to back on one stream: each fills the GPU for >= 2 waves" if serial else
            "launches run concurrently on separate streams") + "); roofline uses the dominant launch timed alone",
        "dominant_alone_ms": 1e3 * dur,
        "clocks": clk,
    }
    if args.workload == "C2" and not args.no_extra:
        # the Nested WAIT kernel on the paper's nested synthetic (C3a), so the
        # default line carries a Nested number too (the C2 headline above is
        # unchanged); same replication sharding, timed alone
        line["nested_c3a"] = nested_block(dev, rank, world, props.multi_processor_count, flush)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, n, nr = cpu_baseline(pols, args.cpu_reps, threads)
        v1, dt1, n1, nr1 = cpu_baseline(pols, 8, 1, min_wall=1.0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": f"{args.workload}, {nr} replications per policy "
                                          f"({n} request-steps, {dt:.2f} s wall on {threads} threads)",
                                "cpu_model": cpu_model(), "one_core": {
                                    "value": v1, "unit": UNIT, "cores": 1,
                                    "sample": f"{nr1} replications per policy ({n1} request-steps, {dt1:.2f} s)"}}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
