"""The S7 cross-GPU reduce on DEVICE tensors (-m gpu): per-policy aggregates of
GPU rows (sim.aggregate) through the single all-reduce (dist.allreduce_
aggregates) equal the aggregate of the unsharded oracle rows.

* one rank over NCCL (the real communicator, world size 1 on this box);
* two ranks sharing cuda:0 over gloo (the host-reduce path bench.py takes
  when a box has fewer GPUs than ranks), each simulating its shard.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu

POL, THR, R, T = W.Policy(W.WAIT), [16, 16], 64, 1.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ref(begin, n):
    from paper_2504_11320_b200.sim import aggregate
    rows = oracle.run(W.C2, POL, THR, n_reps=n, rep_begin=begin, n_threads=8, horizon_s=T)
    return aggregate(torch.from_numpy(rows.view(np.int64)), T)


def _gpu_agg(rank, world, dev):
    from paper_2504_11320_b200 import Scheduler
    from paper_2504_11320_b200 import dist as D
    from paper_2504_11320_b200.sim import aggregate, run_rows
    begin, n = D.rep_range(5, rank, world, R)
    s = Scheduler(W.C2, POL, THR, device=dev)
    rows = run_rows(s, W.C2.seed, begin, n, T)
    agg = aggregate(rows, T)
    assert agg["int"].is_cuda
    red = D.allreduce_aggregates(agg)
    torch.cuda.synchronize()
    s.close()
    return red


def test_nccl_single_rank_allreduce_on_device():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2504_11320_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        red = _gpu_agg(0, 1, 0)
        assert red["int"].is_cuda and red["f64"].is_cuda
        ref = _ref(5 * R, R)
        assert red["int"].cpu().tolist() == ref["int"].tolist()
        assert np.allclose(red["f64"].cpu().numpy(), ref["f64"].numpy(), rtol=1e-12)
        assert D.max_over_ranks(2.5, torch.device("cuda:0")) == 2.5
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2504_11320_b200 import dist as D
    D.init(backend="gloo")
    red = _gpu_agg(rank, world, 0)
    q.put((rank, red["int"].cpu().tolist(), red["f64"].cpu().tolist()))
    dist.destroy_process_group()


def test_two_ranks_gloo_on_device_tensors():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _ref(5 * world * R, world * R)
    for _, ints, f64 in res:
        assert ints == ref["int"].tolist()
        assert np.allclose(f64, ref["f64"].numpy(), rtol=1e-12)


def test_aggregate_kernel_matches_definition_on_slices():
    """sched_aggregate on a column slice (row stride > n_reps) of random rows,
    some with a nonzero status: integer sums exact, float sums within 1e-12
    relative of the torch definition on the same rows (host)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2504_11320_b200.sim import NF, F, aggregate
    g = np.random.default_rng(7)
    full = g.integers(0, 1 << 40, size=(NF, 4096), dtype=np.int64)
    for f in ("lat_hi", "ttft_hi", "soj_hi"):
        full[F[f]] = g.integers(0, 3, size=4096)
    full[F["status"]] = g.integers(0, 3, size=4096) * (g.random(4096) < 0.1)
    full[F["completed"], :7] = 0  # mean latency divides by max(completed, 1)
    dev = torch.from_numpy(full).cuda()
    for lo, n in [(0, 1), (5, 300), (100, 3996)]:
        got = aggregate(dev[:, lo:lo + n], 10.0)
        torch.cuda.synchronize()
        ref = aggregate(torch.from_numpy(np.ascontiguousarray(full[:, lo:lo + n])), 10.0)
        assert got["int"].cpu().tolist() == ref["int"].tolist(), (lo, n)
        assert np.allclose(got["f64"].cpu().numpy(), ref["f64"].numpy(), rtol=1e-12, atol=0), (lo, n)
