"""ctypes binding of libsched (include/sched.h): argument marshalling only.

Every step of the simulation runs in the CUDA kernel behind the C ABI; this
module only converts Python values to the C structs and back.  It raises if
the shared library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsched.so")

WAIT, NESTED, FCFS, FCFS_ONGOING = 0, 1, 2, 3
ERRORS = {-1: "SCHED_E_INVALID", -2: "SCHED_E_UNSTABLE", -3: "SCHED_E_INFEASIBLE",
          -4: "SCHED_E_UNSATISFIABLE", -5: "SCHED_E_CUDA", -6: "SCHED_E_CAPACITY"}

FIELDS = [
    "arrivals", "admitted", "completed", "completed_after_T", "completed_tokens",
    "first_tokens", "batches", "request_steps", "prefill_steps", "evictions",
    "busy_ticks", "idle_ticks", "lat_lo", "lat_hi", "ttft_lo", "ttft_hi",
    "soj_lo", "soj_hi", "completion_batch_idx", "max_kv_peak", "final_waiting",
    "final_resident", "traj_hash", "status", "now_stop", "sum_waiting",
]
NF = len(FIELDS)
F = {n: i for i, n in enumerate(FIELDS)}

# every symbol include/sched.h declares
EXPORTS = ["sched_create", "sched_thresholds", "sched_run", "sched_run_host", "sched_aggregate",
           "sched_run_trace", "sched_get_launch_info", "sched_get_status", "sched_restart_pool_stats",
           "sched_walks", "sched_walks_host", "sched_destroy", "sched_last_error"]
WALK_FIELDS = ["W_B", "stuck", "sumW", "maxW", "Wt_B", "viol", "sumX", "maxS", "minS", "S_B"]
WF = {n: i for i, n in enumerate(WALK_FIELDS)}


class SchedError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class SchedConfig(C.Structure):
    _fields_ = [
        ("K", C.c_uint32), ("lambda_", C.POINTER(C.c_double)),
        ("l_off", C.POINTER(C.c_uint32)), ("l_val", C.POINTER(C.c_uint16)),
        ("l_w", C.POINTER(C.c_uint64)),
        ("lp_off", C.POINTER(C.c_uint32)), ("lp_val", C.POINTER(C.c_uint16)),
        ("lp_w", C.POINTER(C.c_uint64)),
        ("d0_s", C.c_double), ("d1_s", C.c_double), ("M", C.c_int64),
        ("policy", C.c_int32), ("n_thr", C.c_uint32), ("thresholds", C.POINTER(C.c_uint32)),
        ("n_seg", C.c_uint32), ("seg_end", C.POINTER(C.c_uint16)),
        ("B", C.c_uint32), ("tok_budget", C.c_uint32), ("max_resident", C.c_uint32),
        ("restart_cap", C.c_uint32),
        ("rf_off", C.POINTER(C.c_uint32)), ("rf_t", C.POINTER(C.c_double)),
        ("rf_rate", C.POINTER(C.c_double)),
        ("spec_resident", C.c_uint32), ("device", C.c_int32), ("tau_b0", C.c_int64),
    ]


class ThresholdReport(C.Structure):
    _fields_ = [
        ("rho", C.c_double), ("dT_star", C.c_double), ("M_star", C.c_double),
        ("thr_star", C.c_double), ("n_star", C.c_double * 32),
        ("n_thr", C.c_uint32), ("thresholds", C.c_uint32 * 32),
        ("dT_n", C.c_double), ("M_pi", C.c_double), ("M_pi_paper", C.c_double),
        ("feasible", C.c_int32), ("mem_exceeds_M", C.c_int32),
        ("p", C.c_double * 32), ("theta", C.c_double * 32), ("theta_lb", C.c_double * 32),
        ("budget_base", C.c_double), ("budget_queue", C.c_double),
        ("budget_hp", C.c_double), ("budget_total", C.c_double),
        ("tv_Lambda_pi", C.c_double), ("tv_p_star", C.c_double * 32), ("tv_feasible", C.c_int32),
    ]


class LaunchInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("grid", "block", "warps_per_block", "shared_bytes",
                                          "blocks_per_sm", "sm_count", "max_resident",
                                          "restart_cap", "spec_resident", "fallback_grid",
                                          "fallback_warps_per_block", "engine", "last_retries")]


_lib = None


def lib() -> C.CDLL:
    """Load libsched.so; raises (no fallback) if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.sched_last_error.restype = C.c_char_p
        L.sched_create.argtypes = [C.POINTER(C.c_void_p), C.POINTER(SchedConfig)]
        L.sched_thresholds.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double,
                                       C.POINTER(ThresholdReport)]
        L.sched_run.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                                C.c_void_p, C.c_void_p]
        L.sched_run_host.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                                     C.c_void_p, C.c_void_p]
        L.sched_run_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_uint32, C.c_double, C.c_void_p, C.c_void_p,
                                      C.c_int64, C.POINTER(C.c_int64)]
        L.sched_aggregate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_double, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        L.sched_get_launch_info.argtypes = [C.c_void_p, C.POINTER(LaunchInfo)]
        L.sched_restart_pool_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.sched_get_status.argtypes = [C.c_void_p, C.POINTER(C.c_uint32)]
        L.sched_destroy.argtypes = [C.c_void_p]
        L.sched_walks.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_int64, C.c_double,
                                  C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                  C.c_void_p]
        L.sched_walks_host.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_int64, C.c_double,
                                       C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                       C.c_int32]
        for name in ["sched_create", "sched_thresholds", "sched_run", "sched_run_host", "sched_aggregate",
                     "sched_run_trace", "sched_get_launch_info", "sched_restart_pool_stats",
                     "sched_get_status", "sched_walks", "sched_walks_host"]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise SchedError(rc, lib().sched_last_error().decode())


def _arr(data, dt):
    a = np.ascontiguousarray(np.asarray(data, dtype=dt))
    return a, a.ctypes.data_as(C.POINTER(np.ctypeslib.as_ctypes_type(dt)))


class Scheduler:
    """One simulated system + policy on one device (a libsched handle).

    `workload` is any object with lam, l_tab, lp_tab, d0_s, d1_s, M
    (e.g. workloads.Workload); `policy` has kind, seg_end, B, tok_budget.
    """

    def __init__(self, workload, policy, thresholds: Optional[Sequence[int]] = None,
                 device: int = 0, max_resident: int = 0, restart_cap: int = 0,
                 spec_resident: int = 0):
        keep = []
        cfg = SchedConfig()

        def tab(tables):
            off, vals, ws = [0], [], []
            for t in tables:
                for v, w in t:
                    vals.append(v)
                    ws.append(w)
                off.append(len(vals))
            return off, vals, ws

        loff, lval, lw = tab(workload.l_tab)
        poff, pval, pw = tab(workload.lp_tab)
        for name, data, dt in [("lambda_", workload.lam, np.float64), ("l_off", loff, np.uint32),
                               ("l_val", lval, np.uint16), ("l_w", lw, np.uint64),
                               ("lp_off", poff, np.uint32), ("lp_val", pval, np.uint16),
                               ("lp_w", pw, np.uint64)]:
            a, p = _arr(data, dt)
            keep.append(a)
            setattr(cfg, name, p)
        cfg.K = len(workload.lam)
        cfg.d0_s, cfg.d1_s, cfg.M = workload.d0_s, workload.d1_s, workload.M
        cfg.policy = policy.kind
        thr = list(thresholds) if thresholds is not None else list(policy.thresholds or [])
        if policy.kind in (FCFS, FCFS_ONGOING):
            thr = []
        a, p = _arr(thr or [0], np.uint32)
        keep.append(a)
        cfg.thresholds, cfg.n_thr = p, len(thr)
        seg = list(policy.seg_end or [])
        a, p = _arr(seg or [0], np.uint16)
        keep.append(a)
        cfg.seg_end, cfg.n_seg = p, len(seg)
        cfg.B, cfg.tok_budget = policy.B, policy.tok_budget
        cfg.max_resident, cfg.restart_cap, cfg.device = max_resident, restart_cap, device
        cfg.spec_resident = spec_resident
        cfg.tau_b0 = int(getattr(workload, "tau_b0", 0))
        rfs = getattr(workload, "rate_fn", None)
        if rfs:
            off, ts, rs = [0], [], []
            for pieces in rfs:
                for t0, r in (pieces or []):
                    ts.append(t0)
                    rs.append(r)
                off.append(len(ts))
            for name, data, dt in [("rf_off", off, np.uint32), ("rf_t", ts or [0.0], np.float64),
                                   ("rf_rate", rs or [0.0], np.float64)]:
                a, p = _arr(data, dt)
                keep.append(a)
                setattr(cfg, name, p)
        h = C.c_void_p()
        _check(lib().sched_create(C.byref(h), C.byref(cfg)))
        self._h = h
        self.workload, self.policy, self.device = workload, policy, device

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.sched_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
        self._h = None

    __del__ = close

    def thresholds(self, mode: int = 0, delta: float = 0.1, budget_B: float = 0.0,
                   allow_unstable: bool = False) -> dict:
        rep = ThresholdReport()
        rc = lib().sched_thresholds(self._h, mode, delta, budget_B, C.byref(rep))
        if rc != 0 and not (allow_unstable and rc == -2):
            _check(rc)
        n = rep.n_thr
        return dict(rho=rep.rho, dT_star=rep.dT_star, M_star=rep.M_star, thr_star=rep.thr_star,
                    n_star=list(rep.n_star[:len(self.workload.lam)]),
                    thresholds=list(rep.thresholds[:n]), dT_n=rep.dT_n, M_pi=rep.M_pi,
                    M_pi_paper=rep.M_pi_paper, feasible=bool(rep.feasible),
                    mem_exceeds_M=bool(rep.mem_exceeds_M), p=list(rep.p[:n]),
                    theta=list(rep.theta[:n]), theta_lb=list(rep.theta_lb[:n]),
                    budget=(rep.budget_base, rep.budget_queue, rep.budget_hp, rep.budget_total),
                    tv_Lambda_pi=rep.tv_Lambda_pi, tv_p_star=list(rep.tv_p_star[:n]),
                    tv_feasible=rep.tv_feasible, status=rc)

    def launch_info(self) -> dict:
        li = LaunchInfo()
        _check(lib().sched_get_launch_info(self._h, C.byref(li)))
        return {n: getattr(li, n) for n, _ in LaunchInfo._fields_}

    def status_mask(self) -> int:
        """Sticky status (bit s: a replication ended with status s since the
        previous call; cleared by the call)."""
        m = C.c_uint32(0)
        _check(lib().sched_get_status(self._h, C.byref(m)))
        return m.value

    def restart_pool(self) -> dict:
        """Restart pool capacity and high-water mark, in entries (20 B each)."""
        cap, hw = C.c_uint64(0), C.c_uint64(0)
        _check(lib().sched_restart_pool_stats(self._h, C.byref(cap), C.byref(hw)))
        return {"capacity_entries": cap.value, "high_water_entries": hw.value,
                "high_water_bytes": hw.value * 20}

    def run_device(self, seed: int, rep_begin: int, n_reps: int, horizon_s: float,
                   out_ptr: int, stream_ptr: int = 0):
        """Asynchronous launch; out_ptr = device pointer to NF * n_reps uint64."""
        _check(lib().sched_run(self._h, seed, rep_begin, n_reps, horizon_s,
                               C.c_void_p(out_ptr), C.c_void_p(stream_ptr)))

    def run_host(self, seed: int, rep_begin: int, n_reps: int, horizon_s: float,
                 out: Optional[np.ndarray] = None, stream_ptr: int = 0) -> np.ndarray:
        """Rows [NF, n_reps] (uint64) through a host buffer (H2D/D2H inside)."""
        if out is None:
            out = np.zeros((NF, n_reps), dtype=np.uint64)
        # sched_run_host writes NF * n_reps uint64 through this pointer
        if out.dtype != np.uint64 or out.shape != (NF, n_reps) or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous uint64 array of shape {(NF, n_reps)}")
        _check(lib().sched_run_host(self._h, seed, rep_begin, n_reps, horizon_s,
                                    out.ctypes.data, C.c_void_p(stream_ptr)))
        return out

    def run_trace(self, traces, horizon_s: float, log_cap: int = 0):
        """traces: per replication [(t_tick, class, l, l')] sorted by (t, class)."""
        flat = [a for tr in traces for a in tr]
        off = np.cumsum([0] + [len(tr) for tr in traces]).astype(np.int64)
        t = np.array([a[0] for a in flat] or [0], dtype=np.int64)
        c = np.array([a[1] for a in flat] or [0], dtype=np.int32)
        l = np.array([a[2] for a in flat] or [1], dtype=np.int32)
        lp = np.array([a[3] for a in flat] or [1], dtype=np.int32)
        out = np.zeros((NF, len(traces)), dtype=np.uint64)
        log = np.zeros((max(log_cap, 1), 7), dtype=np.int64)
        n = C.c_int64(0)
        _check(lib().sched_run_trace(self._h, t.ctypes.data, c.ctypes.data, l.ctypes.data,
                                     lp.ctypes.data, off.ctypes.data, len(traces), horizon_s,
                                     out.ctypes.data, log.ctypes.data if log_cap else None,
                                     log_cap, C.byref(n)))
        return out, log[: n.value]


def u128(rows: np.ndarray, name: str):
    lo = rows[F[name + "_lo"]]
    hi = rows[F[name + "_hi"]]
    return [int(h) << 64 | int(x) for x, h in zip(lo, hi)]


def walks(kind: int, n: int, B: int, n_walks: int, seed: int, walk_begin: int = 0,
          mu: float = 0.0, n_prev: int = 0, p: float = 0.0, device: int = 0) -> np.ndarray:
    """Appendix random-walk chains on the GPU (C ABI sched_walks_host):
    field-major int64 [len(WALK_FIELDS), n_walks]."""
    out = np.zeros((len(WALK_FIELDS), n_walks), dtype=np.int64)
    _check(lib().sched_walks_host(kind, n, mu, n_prev, p, seed, walk_begin, n_walks, B,
                                  out.ctypes.data, device))
    return out


def aggregate_device(rows_ptr: int, ld: int, n_reps: int, horizon_s: float, out_int_ptr: int,
                     out_f64_ptr: int, stream_ptr: int = 0):
    """sched_aggregate: asynchronous device-side sums of one run's rows."""
    _check(lib().sched_aggregate(C.c_void_p(rows_ptr), ld, n_reps, horizon_s, C.c_void_p(out_int_ptr),
                                 C.c_void_p(out_f64_ptr), C.c_void_p(stream_ptr)))


def walks_device(kind: int, n: int, B: int, n_walks: int, seed: int, out_ptr: int,
                 walk_begin: int = 0, mu: float = 0.0, n_prev: int = 0, p: float = 0.0,
                 stream_ptr: int = 0):
    """Asynchronous launch into a device buffer of len(WALK_FIELDS) * n_walks int64."""
    _check(lib().sched_walks(kind, n, mu, n_prev, p, seed, walk_begin, n_walks, B,
                             C.c_void_p(out_ptr), C.c_void_p(stream_ptr)))
