"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host logic:
replication sharding is disjoint and complete, and the single all-reduce of
the per-policy aggregate vector equals the aggregate of the unsharded run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2504_11320_b200 import dist as D
from paper_2504_11320_b200.sim import aggregate


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, R, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    r, w, _ = D.init(backend="gloo")
    assert (r, w) == (rank, world)
    begin, n = D.rep_range(3, rank, world, R)
    rows = oracle.run(W.C1, W.Policy(W.WAIT), [1], n_reps=n, rep_begin=begin)  # stand-in rows
    agg = aggregate(torch.from_numpy(rows.view(np.int64)), W.C1.horizon_s)
    red = D.allreduce_aggregates(agg)
    mx = D.max_over_ranks(float(rank) + 0.5)
    q.put((rank, begin, n, red["int"].tolist(), red["f64"].tolist(), mx))
    dist.destroy_process_group()


def test_sharded_allreduce_matches_unsharded():
    world, R = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    ranges = [(b, n) for _, b, n, _, _, _ in res]
    assert ranges == [(3 * world * R, R), (3 * world * R + R, R)]   # disjoint, contiguous
    full = oracle.run(W.C1, W.Policy(W.WAIT), [1], n_reps=world * R, rep_begin=3 * world * R)
    ref = aggregate(torch.from_numpy(full.view(np.int64)), W.C1.horizon_s)
    for _, _, _, ints, f64, mx in res:
        assert ints == ref["int"].tolist()                          # exact integer sums
        assert np.allclose(f64, ref["f64"].numpy(), rtol=1e-12)
        assert mx == world - 0.5                                      # max over ranks


def test_shard_helper_covers_range():
    for total in [1, 7, 10_000]:
        for world in [1, 2, 4, 8]:
            spans = [D.shard(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == total
            for (b0, n0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + n0 == b1
