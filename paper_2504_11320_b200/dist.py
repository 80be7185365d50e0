"""Replication sharding over ranks and the single cross-GPU reduce.

Replications are independent, so ranks never exchange simulation state: rank
g of G simulates its own contiguous range of GLOBAL replication indices (the
Philox counter carries the global index, so every row is identical whatever
G is).  The only collective is one all-reduce(SUM) of a small per-policy
aggregate vector (integer counters + float64 second sums) over NCCL.
"""
from __future__ import annotations

import os
import sys
from typing import Dict, Tuple

import torch
import torch.distributed as dist


def env_rank() -> Tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = None) -> Tuple[int, int, int]:
    """Process group for the single metric all-reduce: NCCL (one process
    per GPU) by default; WAITSIM_DIST_BACKEND=gloo runs the same code with a
    host-side reduce (used to exercise N>1 on fewer GPUs).  Returns (rank,
    world, device index)."""
    rank, world, local = env_rank()
    backend = backend or os.environ.get("WAITSIM_DIST_BACKEND")
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            # NCCL logs its communicator init (rank / nranks / transport) on
            # stderr, so a launcher can see how many ranks took part
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
        print(f"[dist] rank {dist.get_rank()}/{dist.get_world_size()} backend={dist.get_backend()} "
              f"device=cuda:{local}", file=sys.stderr, flush=True)
    return rank, world, local


def _host_reduce() -> bool:
    return dist.get_backend() == "gloo"


def _all_reduce(t: torch.Tensor, op=None) -> torch.Tensor:
    op = op if op is not None else dist.ReduceOp.SUM
    if t.is_cuda and _host_reduce():
        h = t.cpu()
        dist.all_reduce(h, op=op)
        return h.to(t.device)
    dist.all_reduce(t, op=op)
    return t


def rep_range(step: int, rank: int, world: int, per_rank: int) -> Tuple[int, int]:
    """(rep_begin, n_reps) of `rank` at `step`: disjoint, contiguous ranges;
    the union over ranks of one step is [step*world*per_rank, (step+1)*world*per_rank)."""
    return (step * world + rank) * per_rank, per_rank


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Split `total` replications into `world` contiguous near-equal ranges."""
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def allreduce_aggregates(agg: Dict[str, torch.Tensor]) -> Dict[str, torch.Tensor]:
    """THE collective: one all-reduce(SUM) of the packed aggregate vector.
    Integer counters travel as float64, exact while every sum stays below
    2^53 (request steps of a C2 step on 8 GPUs are ~2.6e10)."""
    if not (dist.is_available() and dist.is_initialized()):
        return agg
    ints, f64 = agg["int"], agg["f64"]
    buf = _all_reduce(torch.cat([ints.to(torch.float64), f64]))
    n = ints.numel()
    return {"int": buf[:n].round().to(torch.int64), "f64": buf[n:]}


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    return float(_all_reduce(t, dist.ReduceOp.MAX).item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    return float(_all_reduce(t).item())


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
