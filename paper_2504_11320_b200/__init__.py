"""B200-native batched WAIT / Nested WAIT / FCFS simulator (arXiv 2504.11320).

The hot path lives in libsched.so (include/sched.h, csrc/); this package is
the thin Python layer above it: `_lib` (ctypes marshalling), `sim` (torch
device buffers and streams), `dist` (sharding over ranks + the single NCCL
all-reduce of metric sums).
"""
from ._lib import (EXPORTS, F, FIELDS, FCFS, FCFS_ONGOING, NESTED, NF, WAIT, SchedError,
                   Scheduler, lib, u128)

__all__ = ["Scheduler", "SchedError", "lib", "F", "FIELDS", "NF", "EXPORTS", "WAIT",
           "NESTED", "FCFS", "FCFS_ONGOING", "u128"]
