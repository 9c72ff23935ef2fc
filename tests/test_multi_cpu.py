"""Multi-process sharding of design points (world_size 2, gloo, CPU).

The GPU path runs one process per GPU with NCCL; the only collective is the
all-gather of result rows (paper_2604_17550_b200/sweep.py: shard, gather_rows).
Here the evaluator is replaced by a deterministic function of the point index
so the partition and the gather are checked without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_17550_b200.sweep import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fake_rows(idx):
    idx = np.asarray(idx, np.int64)
    return np.stack([idx * 7 + k for k in range(6)], axis=1), (idx % 3 == 0).astype(np.int32) * 3


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    from paper_2604_17550_b200.sweep import gather_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard(n, world, rank)
        rows, status = _fake_rows(range(a, b))
        st, full = gather_rows(status, rows, n, world, rank)
        want_rows, want_status = _fake_rows(range(n))
        q.put((rank, bool((full == want_rows).all() and (st == want_status).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 7, 4096])
def test_gather_rows_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    results = dict(q.get(timeout=5) for _ in procs)
    assert results == {0: True, 1: True}


@pytest.mark.parametrize("n,world", [(4096, 8), (10, 3), (2, 4), (0, 2)])
def test_shard_partitions_points(n, world):
    seen = []
    for r in range(world):
        a, b = shard(n, world, r)
        assert 0 <= a <= b <= n
        seen.extend(range(a, b))
    assert seen == list(range(n))
