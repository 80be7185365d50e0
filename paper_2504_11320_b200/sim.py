"""torch plumbing around libsched: device output buffers, streams, aggregation.

PyTorch only provides device memory and streams here; the simulation itself
is the CUDA kernel behind `Scheduler.run_device` (C ABI `sched_run`).
"""
from __future__ import annotations

from typing import Dict

import numpy as np
import torch

from ._lib import NF, F, Scheduler

TPS = 1e12  # ticks per second


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("CUDA device required: libsched has no CPU fallback")


def run_rows(s: Scheduler, seed: int, rep_begin: int, n_reps: int, horizon_s: float,
             out: torch.Tensor = None, stream: torch.cuda.Stream = None) -> torch.Tensor:
    """Launch on `stream` (default: current); returns the device tensor
    [NF, n_reps] (int64 view of the uint64 rows).  Asynchronous."""
    require_cuda()
    if out is None:
        out = torch.empty((NF, n_reps), dtype=torch.int64, device=f"cuda:{s.device}")
    assert out.is_cuda and out.dtype == torch.int64 and out.shape == (NF, n_reps)
    st = stream if stream is not None else torch.cuda.current_stream(s.device)
    s.run_device(seed, rep_begin, n_reps, horizon_s, out.data_ptr(), st.cuda_stream)
    return out


# per-(policy) aggregate vector for the cross-GPU reduce:
# integer counters summed exactly, tick sums as float64 seconds
AGG_INT = ["arrivals", "admitted", "completed", "completed_after_T", "completed_tokens",
           "first_tokens", "batches", "request_steps", "prefill_steps", "evictions",
           "final_waiting", "final_resident", "status"]
AGG_F64 = ["lat", "ttft", "soj", "busy", "lat_sq", "thr_sq"]


def aggregate(rows: torch.Tensor, horizon_s: float, stream: torch.cuda.Stream = None) -> Dict[str, torch.Tensor]:
    """Sums over replications of one rows tensor [NF, n] (small vectors).
    Device rows: one libsched kernel (sched_aggregate, asynchronous on
    `stream`).  Host rows (the CPU process-group tests feed oracle rows): the
    same definition in torch ops."""
    if rows.is_cuda:
        from ._lib import aggregate_device
        assert rows.dtype == torch.int64 and rows.shape[0] == NF and rows.stride(1) == 1
        out_i = torch.empty(len(AGG_INT), dtype=torch.int64, device=rows.device)
        out_f = torch.empty(len(AGG_F64), dtype=torch.float64, device=rows.device)
        st = stream if stream is not None else torch.cuda.current_stream(rows.device)
        aggregate_device(rows.data_ptr(), rows.stride(0), rows.shape[1], horizon_s, out_i.data_ptr(),
                         out_f.data_ptr(), st.cuda_stream)
        return {"int": out_i, "f64": out_f}
    r = rows
    # status: the NUMBER of replications with a nonzero status (1 resident
    # overflow, 2 restart overflow), not the sum of the codes
    ints = torch.stack([(r[F[k]] != 0).sum() if k == "status" else r[F[k]].sum() for k in AGG_INT])
    two64 = 18446744073709551616.0

    def t128(name):
        lo = r[F[name + "_lo"]].double()
        lo = torch.where(lo < 0, lo + two64, lo)
        return (lo + r[F[name + "_hi"]].double() * two64) / TPS

    lat = t128("lat")
    comp = r[F["completed"]].double().clamp_min(1)
    mean_lat = lat / comp
    thr = r[F["completed_tokens"]].double() / horizon_s
    f64 = torch.stack([lat.sum(), t128("ttft").sum(), t128("soj").sum(),
                       r[F["busy_ticks"]].double().sum() / TPS,
                       (mean_lat ** 2).sum(), (thr ** 2).sum()])
    return {"int": ints, "f64": f64}
