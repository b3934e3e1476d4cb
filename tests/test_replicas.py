"""Multi-GPU host logic on CPU: bench.py's replica aggregation (max-over-ranks
device time, whole-job value) with torch.distributed gloo, world_size 2.

The path does not shard: N GPUs run N independent
replicas, so the only cross-rank step is this reduction."""

import os
import socket
import sys

import pytest

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local_ms = [10.0, 25.0][rank]  # rank 1 is the slow replica
        value, max_ms = bench.replica_aggregate(local_ms, cells_per_rank=1000, steps=4, dist=dist)
        q.put((rank, value, max_ms))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_replica_aggregate_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=10) for _ in range(2))
    for rank, value, max_ms in got:
        assert max_ms == pytest.approx(25.0)  # max over ranks, on every rank
        assert value == pytest.approx(2 * 1000 * 4 / 25e-3)  # whole-job cells / max time


def test_replica_aggregate_single():
    import bench

    value, max_ms = bench.replica_aggregate(8.0, cells_per_rank=500, steps=2)
    assert max_ms == 8.0 and value == pytest.approx(500 * 2 / 8e-3)
