"""CPU oracle for the WAIT / Nested WAIT / FCFS simulation -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this package.  The product path
(paper_2504_11320_b200/) never imports it and shares no code with it.

* des_oracle.cpp / liboracle.so -- the sequential discrete-event simulator
  (DESIGN.md §4), loaded through ctypes.
* fluid.py -- the host-side setup math (fluid equilibrium, thresholds, theta,
  memory budget) in exact rational arithmetic.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "des_oracle.cpp")
_SRC_WALKS = os.path.join(_HERE, "walks_oracle.cpp")

FIELDS = [
    "arrivals", "admitted", "completed", "completed_after_T", "completed_tokens",
    "first_tokens", "batches", "request_steps", "prefill_steps", "evictions",
    "busy_ticks", "idle_ticks", "lat_lo", "lat_hi", "ttft_lo", "ttft_hi",
    "soj_lo", "soj_hi", "completion_batch_idx", "max_kv_peak", "final_waiting",
    "final_resident", "traj_hash", "status", "now_stop", "sum_waiting",
]
NF = len(FIELDS)
F = {n: i for i, n in enumerate(FIELDS)}

WAIT, NESTED, FCFS, FCFS_ONGOING = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(_SRC_WALKS),
            os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", _SO, _SRC, _SRC_WALKS, "-lpthread"])
    return _SO


class _Cfg(C.Structure):
    _fields_ = [
        ("K", C.c_int32), ("lam", C.POINTER(C.c_double)),
        ("l_off", C.POINTER(C.c_int32)), ("l_val", C.POINTER(C.c_uint16)),
        ("l_w", C.POINTER(C.c_uint64)),
        ("lp_off", C.POINTER(C.c_int32)), ("lp_val", C.POINTER(C.c_uint16)),
        ("lp_w", C.POINTER(C.c_uint64)),
        ("d0_s", C.c_double), ("d1_s", C.c_double), ("M", C.c_int64),
        ("policy", C.c_int32), ("n_thr", C.c_int32), ("thr", C.POINTER(C.c_uint32)),
        ("n_seg", C.c_int32), ("seg_end", C.POINTER(C.c_uint16)),
        ("B", C.c_uint32), ("tok_budget", C.c_uint32), ("horizon_s", C.c_double),
        ("rf_off", C.POINTER(C.c_int32)), ("rf_t", C.POINTER(C.c_double)),
        ("rf_rate", C.POINTER(C.c_double)), ("tau_b0", C.c_int64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_exp_from_bits.restype = C.c_double
        _lib.orc_exp_from_bits.argtypes = [C.c_uint32, C.c_uint32]
        _lib.orc_run.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.c_uint64, C.c_int64,
                                 C.c_void_p, C.c_int32]
        _lib.orc_run_trace.restype = C.c_int64
        _lib.orc_run_trace.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_int64]
        _lib.orc_walks.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_int64, C.c_double,
                                   C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]
        _lib.orc_gen_arrivals.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.c_uint32,
                                          C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    return _lib


def _arr(a, dt):
    a = np.ascontiguousarray(np.asarray(a, dtype=dt))
    return a, a.ctypes.data_as(C.POINTER(np.ctypeslib.as_ctypes_type(dt)))


class Config:
    """ctypes view of (workload, policy, thresholds); keeps its arrays alive."""

    def __init__(self, wl, policy, thresholds: Optional[Sequence[int]] = None,
                 horizon_s: Optional[float] = None):
        keep = []

        def tab(tables):
            off, vals, ws = [0], [], []
            for t in tables:
                for v, w in t:
                    vals.append(v)
                    ws.append(w)
                off.append(len(vals))
            return off, vals, ws

        loff, lval, lw = tab(wl.l_tab)
        poff, pval, pw = tab(wl.lp_tab)
        cfg = _Cfg()
        cfg.K = wl.K
        for name, data, dt in [("lam", wl.lam, np.float64), ("l_off", loff, np.int32),
                               ("l_val", lval, np.uint16), ("l_w", lw, np.uint64),
                               ("lp_off", poff, np.int32), ("lp_val", pval, np.uint16),
                               ("lp_w", pw, np.uint64)]:
            a, p = _arr(data, dt)
            keep.append(a)
            setattr(cfg, name, p)
        cfg.d0_s, cfg.d1_s, cfg.M = wl.d0_s, wl.d1_s, wl.M
        cfg.policy = policy.kind
        thr = list(thresholds if thresholds is not None else policy.thresholds)
        a, p = _arr(thr, np.uint32)
        keep.append(a)
        cfg.thr, cfg.n_thr = p, len(thr)
        seg = list(policy.seg_end or [])
        a, p = _arr(seg if seg else [0], np.uint16)
        keep.append(a)
        cfg.seg_end, cfg.n_seg = p, len(seg)
        cfg.B, cfg.tok_budget = policy.B, policy.tok_budget
        cfg.horizon_s = wl.horizon_s if horizon_s is None else horizon_s
        cfg.tau_b0 = int(getattr(wl, "tau_b0", 0))
        rfs = getattr(wl, "rate_fn", None)
        if rfs:
            off, ts, rs = [0], [], []
            for pieces in rfs:
                for t0, r in (pieces or []):
                    ts.append(t0)
                    rs.append(r)
                off.append(len(ts))
            for name, data, dt in [("rf_off", off, np.int32), ("rf_t", ts or [0.0], np.float64),
                                   ("rf_rate", rs or [0.0], np.float64)]:
                a, p = _arr(data, dt)
                keep.append(a)
                setattr(cfg, name, p)
        self.cfg, self._keep = cfg, keep


def run(wl, policy, thresholds=None, n_reps: int = 1, rep_begin: int = 0,
        n_threads: int = 1, seed: Optional[int] = None, horizon_s=None) -> np.ndarray:
    """Per-replication metric rows, field-major uint64 array [NF, n_reps]."""
    cfg = Config(wl, policy, thresholds, horizon_s)
    out = np.zeros((NF, n_reps), dtype=np.uint64)
    lib().orc_run(C.byref(cfg.cfg), wl.seed if seed is None else seed, rep_begin, n_reps,
                  out.ctypes.data, n_threads)
    return out


def run_trace(wl, policy, thresholds, traces: Sequence[Sequence[Tuple[int, int, int, int]]],
              log_cap: int = 0, horizon_s=None):
    """Explicit traces [(t_tick, class, l, l')] per replication.

    Returns (rows [NF, n], log [n_batches, 7] of replication 0)."""
    cfg = Config(wl, policy, thresholds, horizon_s)
    flat = [a for tr in traces for a in tr]
    off = np.cumsum([0] + [len(tr) for tr in traces]).astype(np.int64)
    t = np.array([a[0] for a in flat] or [0], dtype=np.int64)
    c = np.array([a[1] for a in flat] or [0], dtype=np.int32)
    l = np.array([a[2] for a in flat] or [1], dtype=np.int32)
    lp = np.array([a[3] for a in flat] or [1], dtype=np.int32)
    out = np.zeros((NF, len(traces)), dtype=np.uint64)
    log = np.zeros((max(log_cap, 1), 7), dtype=np.int64)
    n = lib().orc_run_trace(C.byref(cfg.cfg), t.ctypes.data, c.ctypes.data, l.ctypes.data,
                            lp.ctypes.data, off.ctypes.data, len(traces), out.ctypes.data,
                            log.ctypes.data if log_cap else None, log_cap)
    return out, log[:n]


def gen_arrivals(wl, r: int, c: int, n: int, seed: Optional[int] = None):
    """First n arrivals of class c in replication r: (t ticks, l, l')."""
    from workloads import Policy
    cfg = Config(wl, Policy(FCFS, thresholds=[0], B=1), [0])
    t = np.zeros(n, np.int64)
    l = np.zeros(n, np.int32)
    lp = np.zeros(n, np.int32)
    rc = lib().orc_gen_arrivals(C.byref(cfg.cfg), wl.seed if seed is None else seed, r, c,
                                n, t.ctypes.data, l.ctypes.data, lp.ctypes.data)
    if rc != 0:
        raise ValueError("class has rate 0")
    return t, l, lp


def philox(ctr, key):
    out = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), out)
    return list(out)


def exp_from_bits(x0: int, x1: int) -> float:
    return lib().orc_exp_from_bits(x0, x1)


def u128(rows: np.ndarray, name: str) -> List[int]:
    lo = rows[F[name + "_lo"]].astype(object)
    hi = rows[F[name + "_hi"]].astype(object)
    return [int(h) << 64 | int(x) for x, h in zip(lo, hi)]


WALK_FIELDS = ["W_B", "stuck", "sumW", "maxW", "Wt_B", "viol", "sumX", "maxS", "minS", "S_B"]
WF = {n: i for i, n in enumerate(WALK_FIELDS)}


def walks(kind: int, n: int, B: int, n_walks: int, seed: int, walk_begin: int = 0,
          mu: float = 0.0, n_prev: int = 0, p: float = 0.0) -> np.ndarray:
    """Appendix random-walk chains, field-major [10, n_walks]."""
    out = np.zeros((len(WALK_FIELDS), n_walks), dtype=np.int64)
    lib().orc_walks(kind, n, mu, n_prev, p, seed, walk_begin, n_walks, B, out.ctypes.data)
    return out
