"""Multi-rank host logic on CPU (gloo, world_size 2): the image sharding the
bench and carve_batch use (whole images per GPU, no collective
on the data path), max-over-ranks timing, and result assembly. The per-image
work here is the CPU oracle (test infrastructure) standing in for one GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partitions_exactly():
    for n in (1, 7, 8, 1024, 1025):
        for world in (1, 2, 3, 4, 8):
            spans = [bench.shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    lo, hi = bench.shard(n, world, rank)
    port_ = oracle.port()
    outs = {k: port_.carve(port_.make_test_image(24, 16, k), 18) for k in range(lo, hi)}
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks timing, as bench.py does
    gathered = [None] * world
    dist.all_gather_object(gathered, {k: v.tobytes() for k, v in outs.items()})
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        q.put((float(t.item()), merged))
    dist.destroy_process_group()


def test_two_rank_batch_matches_single_rank():
    n, world = 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    assert sorted(merged) == list(range(n))
    port_ = oracle.port()
    for k in range(n):
        want = port_.carve(port_.make_test_image(24, 16, k), 18)
        assert merged[k] == want.tobytes()
