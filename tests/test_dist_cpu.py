"""Multi-process (world_size 2, gloo, CPU) checks of the request-sharding host logic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2305_17423_b200 import dist as D


def test_shard_requests_balanced_and_complete():
    g = np.random.default_rng(0)
    costs = [int(c) for c in g.integers(100, 5000, 64)]
    for ws in (1, 2, 4, 8):
        shards = D.shard_requests(costs, ws)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(64))
        loads = [sum(costs[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(costs)
        assert D.shard_requests(costs, ws) == shards  # deterministic


def test_request_cost_counts_tiles_and_pixels():
    b = np.zeros((8, 8), bool)
    b[1, 1] = True
    assert D.request_cost(b) == 4 + 1
    b[:] = True
    assert D.request_cost(b) == 16 * 4 + 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    costs = [400, 100, 900, 250, 50]
    shards = D.shard_requests(costs, ws)
    local = {i: np.full((1, 4, 8, 8), float(i), np.float32) for i in shards[rank]}
    out = D.gather_results(local, ws)
    mx = D.max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((sorted(out), [float(out[k][0, 0, 0, 0]) for k in sorted(out)], mx))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_and_max_over_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys, vals, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert keys == [0, 1, 2, 3, 4] and vals == [0.0, 1.0, 2.0, 3.0, 4.0] and mx == 2.0
