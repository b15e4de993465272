"""Multi-rank plumbing on CPU (world_size 2, gloo): scenario partition
matches the reference (executor.cpp:7-19) and the host-staged all-reduce used
by the sharded solver (paper_2301_04869_b200/distributed.py) combines ranks
with sum / max / min in place."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_04869_b200 import _native as nat
from paper_2301_04869_b200.distributed import gloo_allreduce


def test_partition_matches_reference_rule():
    assert nat.partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert nat.partition(256, 8) == [(32 * g, 32 * (g + 1)) for g in range(8)]
    assert nat.partition(5, 5) == [(g, g + 1) for g in range(5)]
    with pytest.raises(nat.BipmError):
        nat.partition(3, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = gloo_allreduce()
    a = np.array([1.0 + rank, -2.0 * rank, 3.0])
    fn(a, 0)
    b = np.array([float(rank), -float(rank)])
    fn(b, 1)
    c = np.array([float(rank) + 0.5])
    fn(c, 2)
    out[rank] = np.concatenate([a, b, c]).tolist()
    dist.destroy_process_group()


def test_host_allreduce_two_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == [3.0, -2.0, 6.0, 1.0, 0.0, 0.5]
