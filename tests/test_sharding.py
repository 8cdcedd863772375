"""Multi-rank host logic on CPU (gloo, world_size 2): instance sharding and the max-over-ranks timing."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2403_15913_b200.sharding import max_over_ranks, per_unit_ms, shard


def test_shard_partitions():
    for total in (1, 7, 64):
        for world in (1, 2, 3, 8):
            got = [list(shard(total, world, r)) for r in range(world)]
            flat = [i for g in got for i in g]
            assert flat == list(range(total))
            assert max(map(len, got)) - min(map(len, got)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(shard(64, world, rank))
    ms = 10.0 + rank  # rank 1 is the slowest
    m = max_over_ranks(ms)
    out[rank] = (mine[0], len(mine), m, per_unit_ms(m, steps=5, units_per_step=len(mine) * world))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][:2] == (0, 32) and out[1][:2] == (32, 32)
    assert out[0][2] == out[1][2] == 11.0
    assert out[0][3] == pytest.approx(11.0 / (5 * 64))
