"""N>1 host logic on CPU: replicas timed by the slowest rank (gloo, world_size 2).

bench.py runs one independent solve per GPU (the reference's GS order forbids
sharding one solve); the only collectives are the barrier and the
max-over-ranks reduction of the device time, exercised here with gloo.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = 10.0 + 5.0 * rank   # rank 1 is the slow replica
    ms = bench.max_over_ranks(local_ms, dist, "cpu")
    dist.barrier()
    out[rank] = (ms, bench.replica_value(world, 1000, 6, ms))
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1]
    ms, value = out[0]
    assert ms == 15.0
    assert value == pytest.approx(2 * 1000 * 6 / 0.015)


def test_single_process_identity():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.replica_value(1, 67081, 6, 10.0) == pytest.approx(67081 * 6 / 0.01)
